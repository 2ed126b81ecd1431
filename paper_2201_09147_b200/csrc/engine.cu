// Engine kernels: ray generation, the compacting multiscale trace loop, fused normals +
// shading, and the batch-evaluation kernels of the API path.
//
// This translation unit is compiled with -fmad=false and uses explicit _rn intrinsics for
// every host-visible float/double operation, so the tracer, ray and shading arithmetic
// restates the reference's -ffp-contract=off C++ exactly (proj/CMakeLists.txt:15).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include <nvtx3/nvToolsExt.h>

#include "engine.cuh"
#include "mlp_simt.cuh"
#include "mlp_tc.cuh"
#include "device_ops.cuh"

namespace nsdf_b200 {

// ---------------------------------------------------------------------------------------
// Workspace
// ---------------------------------------------------------------------------------------
Workspace::~Workspace() {
  if (base) cudaFree(base);
  if (host_pinned) cudaFreeHost(host_pinned);
}

cudaError_t Workspace::reserve(size_t need) {
  if (need <= bytes) return cudaSuccess;
  if (base) cudaFree(base);
  base = nullptr;
  bytes = 0;
  size_t grow = need + need / 4;
  cudaError_t e = cudaMalloc(&base, grow);
  if (e == cudaSuccess) bytes = grow;
  return e;
}

cudaError_t Workspace::reserve_host(size_t need) {
  if (need <= host_bytes) return cudaSuccess;
  if (host_pinned) cudaFreeHost(host_pinned);
  host_pinned = nullptr;
  host_bytes = 0;
  cudaError_t e = cudaMallocHost(&host_pinned, need);
  if (e == cudaSuccess) host_bytes = need;
  return e;
}

cudaEvent_t Profiler::begin(cudaStream_t s) {
  if (!on) return nullptr;
  cudaEvent_t e;
  if (pool.empty()) {
    cudaEventCreate(&e);
  } else {
    e = pool.back();
    pool.pop_back();
  }
  cudaEventRecord(e, s);
  return e;
}

void Profiler::end(int kind, cudaEvent_t a, cudaStream_t s) {
  if (!on || !a) return;
  cudaEvent_t b = begin(s);
  pending.push_back({kind, a, b});
}

void Profiler::collect() {
  for (const Span& sp : pending) {
    cudaEventSynchronize(sp.b);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, sp.a, sp.b);
    if (sp.kind < NSDF_MAX_LEVELS) {
      acc.level_ms[sp.kind] += ms;
    } else if (sp.kind == kNormals) {
      acc.normals_ms += ms;
    } else {
      acc.frame_ms += ms;
      acc.frames++;
    }
    pool.push_back(sp.a);
    pool.push_back(sp.b);
  }
  pending.clear();
}

void Profiler::reset() {
  collect();
  acc = nsdf_profile{};
}

Profiler::~Profiler() {
  for (const Span& sp : pending) {
    cudaEventDestroy(sp.a);
    cudaEventDestroy(sp.b);
  }
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

size_t frame_workspace_bytes(int n_rays, int n_counters) {
  const size_t n = size_t(std::max(n_rays, 1));
  size_t b = 0;
  b += 7 * align_up(n * 4, 256);                    // px py pz t dx dy dz
  b += align_up(n * kMaxLevels * 2, 256);    // iters
  b += 2 * align_up(n * 4, 256);                    // level_reached, final_dist
  b += align_up(n, 256);                            // hit
  b += align_up(n * 4, 256);                        // pixel
  b += 4 * align_up(n * 4, 256);                    // 3 lists + fallback list
  b += align_up(size_t(n_counters) * 4, 256);
  return b;
}

FrameBuffers carve_frame(void* base, int n_rays, int n_counters) {
  const size_t n = size_t(std::max(n_rays, 1));
  char* p = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += align_up(bytes, 256);
    return r;
  };
  FrameBuffers fb;
  fb.st.cap = int(n);
  fb.st.n_pix = int(n);  // callers with a camera set the frame's W*H
  fb.st.px = reinterpret_cast<float*>(take(n * 4));
  fb.st.py = reinterpret_cast<float*>(take(n * 4));
  fb.st.pz = reinterpret_cast<float*>(take(n * 4));
  fb.st.t = reinterpret_cast<float*>(take(n * 4));
  fb.st.dx = reinterpret_cast<float*>(take(n * 4));
  fb.st.dy = reinterpret_cast<float*>(take(n * 4));
  fb.st.dz = reinterpret_cast<float*>(take(n * 4));
  fb.st.iters = reinterpret_cast<uint16_t*>(take(n * kMaxLevels * 2));
  fb.st.level_reached = reinterpret_cast<int*>(take(n * 4));
  fb.st.final_dist = reinterpret_cast<float*>(take(n * 4));
  fb.st.hit = reinterpret_cast<uint8_t*>(take(n));
  fb.st.pixel = reinterpret_cast<int*>(take(n * 4));
  for (int i = 0; i < 3; ++i) fb.list[i] = reinterpret_cast<int*>(take(n * 4));
  fb.fallback_list = reinterpret_cast<int*>(take(n * 4));
  fb.counters = reinterpret_cast<int*>(take(size_t(n_counters) * 4));
  fb.n_counters = n_counters;
  return fb;
}

int normal_tile_terms(Mode m) {
  static const int forced = [] {
    const char* e = getenv("NSDF_NORMAL_TERMS");
    return e ? atoi(e) : 0;
  }();
  if (m == Mode::Fp16Low) return 1;
  return forced == 3 ? 3 : 1;
}

int device_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
    cudaGetLastError();
    sms = 148;
  }
  return sms;
}

static int num_sms() { return device_sms(); }

namespace {
// The SMEM opt-in is ONE value per (device, kernel): raised to the largest size any launch
// needed so far (a smaller request must not lower it under another caller's cached size).
struct KernelCfgEntry {
  size_t configured = 0;
  std::map<std::pair<int, size_t>, KernelCfg> by_launch;  // (threads, smem)
};
std::mutex g_cfg_mu;
std::map<std::pair<int, const void*>, KernelCfgEntry> g_cfg_cache;
}  // namespace

void reset_kernel_cfg() {
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  g_cfg_cache.clear();
}

KernelCfg kernel_cfg(const void* kernel, int threads, size_t smem, bool max_carveout) {
  int dev = 0;
  cudaGetDevice(&dev);
  using Entry = KernelCfgEntry;
  auto& cache = g_cfg_cache;
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  Entry& e = cache[{dev, kernel}];
  KernelCfg k;
  if (smem > e.configured) {
    k.err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (k.err != cudaSuccess) {
      cudaGetLastError();
      return k;
    }
    if (max_carveout) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    e.configured = smem;
  }
  auto it = e.by_launch.find({threads, smem});
  if (it != e.by_launch.end()) return it->second;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k.occupancy, kernel, threads, smem) != cudaSuccess) k.occupancy = 1;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess) k.regs = fa.numRegs;
  cudaGetLastError();
  k.sms = device_sms();
  e.by_launch.emplace(std::make_pair(threads, smem), k);
  return k;
}

// ---------------------------------------------------------------------------------------
// Rays: generate_rays (camera.cpp:20-43), per pixel in double without contraction.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void pixel_ray(const CamBasis& c, int px, int py, float d[3]) {
  const double v = __ddiv_rn(__dadd_rn(double(py), 0.5), double(c.height));
  const double sy = __dmul_rn(__dsub_rn(1.0, __dmul_rn(2.0, v)), c.half_h);
  const double u = __ddiv_rn(__dadd_rn(double(px), 0.5), double(c.width));
  const double sx = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0), c.half_w);
  double e[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) e[i] = __dadd_rn(__dadd_rn(c.fwd[i], __dmul_rn(c.right[i], sx)), __dmul_rn(c.up[i], sy));
  const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(e[0], e[0]), __dmul_rn(e[1], e[1])), __dmul_rn(e[2], e[2])));
#pragma unroll
  for (int i = 0; i < 3; ++i) d[i] = n > 0 ? __double2float_rn(__ddiv_rn(e[i], n)) : 0.0f;
}

__global__ void rays_kernel(CamBasis c, int tile_size, int tile_rank, int tile_world, const int* owners,
                            RayState st, int* n_slots) {
  const int npix = c.width * c.height;
  const int tiles_x = (c.width + tile_size - 1) / tile_size;
  // Whole warps iterate together so warp_append sees full masks.
  for (int base = blockIdx.x * blockDim.x; base < npix; base += gridDim.x * blockDim.x) {
    const int pix = base + threadIdx.x;
    const bool inside = pix < npix;
    const int px = inside ? pix % c.width : 0, py = inside ? pix / c.width : 0;
    bool own = inside;
    if (tile_world > 1 && inside) {
      const int tile = (py / tile_size) * tiles_x + px / tile_size;
      own = (owners ? owners[tile] : tile % tile_world) == tile_rank;
    }
    int slot = pix;
    if (tile_world > 1) {
      const unsigned mask = __ballot_sync(0xffffffffu, own);
      const int lane = threadIdx.x & 31;
      int b = 0;
      if (mask) {
        if (lane == __ffs(mask) - 1) b = atomicAdd(n_slots, __popc(mask));
        b = __shfl_sync(0xffffffffu, b, __ffs(mask) - 1);
      }
      slot = b + __popc(mask & ((1u << lane) - 1u));
    }
    if (!own || !in_bounds(slot, st.cap, kChkSlot)) continue;
    float d[3];
    pixel_ray(c, px, py, d);
    st.px[slot] = c.origin[0];
    st.py[slot] = c.origin[1];
    st.pz[slot] = c.origin[2];
    st.dx[slot] = d[0];
    st.dy[slot] = d[1];
    st.dz[slot] = d[2];
    st.pixel[slot] = pix;
  }
}

void launch_generate_rays(const CamBasis& cb, int tile_size, int tile_rank, int tile_world, const int* owners,
                          RayState st, int* n_slots_dev, cudaStream_t s) {
  const int npix = cb.width * cb.height;
  const int blocks = std::min((npix + 255) / 256, num_sms() * 8);
  rays_kernel<<<std::max(blocks, 1), 256, 0, s>>>(cb, tile_size, tile_rank, tile_world, owners, st, n_slots_dev);
}

__global__ void rays_to_host_kernel(RayState st, int n, float* rays6) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float* r = rays6 + size_t(6) * i;
    r[0] = st.px[i];
    r[1] = st.py[i];
    r[2] = st.pz[i];
    r[3] = st.dx[i];
    r[4] = st.dy[i];
    r[5] = st.dz[i];
  }
}

void launch_rays_to_host_layout(const RayState& st, int n, float* rays6, cudaStream_t s) {
  if (n <= 0) return;
  rays_to_host_kernel<<<std::min((n + 255) / 256, num_sms() * 8), 256, 0, s>>>(st, n, rays6);
}

__global__ void init_from_rays_kernel(const float* rays6, int n, RayState st) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float* r = rays6 + size_t(6) * i;
    st.px[i] = r[0];
    st.py[i] = r[1];
    st.pz[i] = r[2];
    st.dx[i] = r[3];
    st.dy[i] = r[4];
    st.dz[i] = r[5];
    st.pixel[i] = i;
  }
}

void launch_init_state_from_rays(const float* rays6, int n, RayState st, cudaStream_t s) {
  if (n <= 0) return;
  init_from_rays_kernel<<<std::min((n + 255) / 256, num_sms() * 8), 256, 0, s>>>(rays6, n, st);
}

void launch_reset_state(RayState st, int n, cudaStream_t s) {
  if (n <= 0) return;
  cudaMemsetAsync(st.t, 0, size_t(n) * 4, s);
  cudaMemsetAsync(st.iters, 0, size_t(n) * kMaxLevels * 2, s);
  cudaMemsetAsync(st.level_reached, 0xff, size_t(n) * 4, s);
  cudaMemsetAsync(st.final_dist, 0, size_t(n) * 4, s);
  cudaMemsetAsync(st.hit, 0, size_t(n), s);
}

// ---------------------------------------------------------------------------------------
// Field tile: MLP (FFMA oracle tile) or analytic member.
// ---------------------------------------------------------------------------------------
template <bool kGrad, int kT>
__device__ __forceinline__ void field_tile(const DevField& f, const float* pts, float* bufA, float* bufB,
                                           float* vals) {
  if (f.kind == kFieldMlp) {
    simt_mlp_tile<kGrad, kT>(f.net, pts, bufA, bufB, vals);
    return;
  }
  constexpr int kRays = kGrad ? kTileCols / 4 : kTileCols;
  for (int col = threadIdx.x; col < kTileCols; col += kT) {
    const int ray = kGrad ? col / 4 : col, chain = kGrad ? col % 4 : 0;
    const double x = pts[ray], y = pts[kRays + ray], z = pts[2 * kRays + ray];
    if (chain == 0) {
      vals[col] = __double2float_rn(analytic_eval(f, x, y, z));
    } else {
      double g[3];
      analytic_grad(f, x, y, z, g);
      vals[col] = __double2float_rn(g[chain - 1]);
    }
  }
  __syncthreads();
}

static size_t field_smem(const DevField& f) {
  const int w = f.kind == kFieldMlp ? f.net.max_width : 4;
  return simt_tile_smem_bytes(w) + (4 * kTileCols + kTileCols + kTileCols) * sizeof(float);
}

template <typename K>
static int blocks_for(K kernel, int threads, size_t smem) {
  const KernelCfg k = kernel_cfg(reinterpret_cast<const void*>(kernel), threads, smem);
  return (k.sms > 0 ? k.sms : num_sms()) * std::max(k.occupancy, 1);
}

// CTA size of the FFMA tiles: 256 threads (16 row groups x 16 column groups) for nets up to
// 128 wide; 1024 for 256-wide nets, whose 128 KB activation tile allows one CTA per SM —
// four times the warps to hide the weight loads (oracle mode 2.5x faster on 256x3 levels;
// narrower nets keep 256, where 1024 threads would leave row groups idle).
static bool wide_tile(const DevField& f) { return f.kind == kFieldMlp && f.net.max_width >= 256; }

// ---------------------------------------------------------------------------------------
// Trace iteration (trace_level body, trace.cpp:46-82) for one compacted active list.
// ---------------------------------------------------------------------------------------
template <int kT>
__global__ void __launch_bounds__(kT) trace_iter_simt(IterArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int W = a.lv.field.kind == kFieldMlp ? max(a.lv.field.net.max_width, 4) : 4;
  float* bufA = smem;
  float* bufB = bufA + W * kTileCols;
  float* pts = bufB + W * kTileCols;
  float* vals = pts + 4 * kTileCols;
  int* slots = reinterpret_cast<int*>(vals + kTileCols);
  const int n = *a.in_count;
  const int tid = threadIdx.x;
  for (int base = blockIdx.x * kTileCols; base < n; base += gridDim.x * kTileCols) {
    const int cnt = min(kTileCols, n - base);
    if (tid < kTileCols) {
      int slot = tid < cnt && in_bounds(base + tid, a.st.cap, kChkListRead) ? a.in_list[base + tid] : -1;
      if (slot >= 0 && !in_bounds(slot, a.st.cap, kChkSlot)) slot = -1;
      slots[tid] = slot;
      pts[tid] = slot >= 0 ? a.st.px[slot] : 0.0f;
      pts[kTileCols + tid] = slot >= 0 ? a.st.py[slot] : 0.0f;
      pts[2 * kTileCols + tid] = slot >= 0 ? a.st.pz[slot] : 0.0f;
      pts[3 * kTileCols + tid] = a.lv.time;
    }
    __syncthreads();
    field_tile<false, kT>(a.lv.field, pts, bufA, bufB, vals);
    if (tid < kTileCols) {
      const int slot = slots[tid];
      bool conv = false, cont = false;
      if (slot >= 0) trace_update(a, slot, vals[tid], conv, cont);
      warp_append(conv, slot, a.adv_list, a.adv_count, a.st.cap);
      warp_append(cont, slot, a.next_list, a.next_count, a.st.cap);
    }
    __syncthreads();
  }
}

__global__ void iota_kernel(int* list, const int* n) {
  const int cnt = *n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) list[i] = i;
}

TraceResult run_trace(Mode mode, const std::vector<LevelDesc>& levels, float eps, float t_max,
                      FrameBuffers& fb, int n_max, const int* n_slots_dev, cudaStream_t s, Profiler* prof) {
  TraceResult res;
  int cur = 0, nxt = 1, adv = 2;
  iota_kernel<<<std::max(1, std::min((n_max + 255) / 256, num_sms() * 8)), 256, 0, s>>>(fb.list[cur], n_slots_dev);
  res.launches++;
  const int* level_in_count = n_slots_dev;
  int coff = 1;  // counters[0] holds the slot count
  for (const LevelDesc& lv : levels) {
    // per level: [adv count, claim cursor, evaluations, iteration list sizes...]
    int* adv_count = fb.counters + coff;
    int* cursor = fb.counters + coff + 1;
    int* evals = fb.counters + coff + 2;
    int* refine_count = fb.counters + coff + 3;
    int* refine_cursor = fb.counters + coff + 4;
    int* it_counts = fb.counters + coff + 5;
    res.counter_layout_base.push_back(coff);
    coff += 5 + lv.budget;
    IterArgs a;
    a.lv = lv;
    a.eps = eps;
    a.t_max = t_max;
    a.st = fb.st;
    a.adv_list = fb.list[adv];
    a.adv_count = adv_count;
    const int* in_list = fb.list[cur];
    const int* in_count = level_in_count;
    int ping = cur, pong = nxt;
    cudaEvent_t ev = prof ? prof->begin(s) : nullptr;
    char range[32];
    snprintf(range, sizeof range, "nsdf level %d", lv.level);
    nvtxRangePushA(range);
    // fast mode: ONE persistent launch per level (rows refilled from the input list)
    TcLaunch tl = TcLaunch::kDeclined;
    // An E4M3 final level parks near-threshold stop decisions on the free list (fb.list[nxt]:
    // the persistent path does not ping-pong) and finishes them in a resume launch with the
    // fp16 correction terms: a flipped stop decision moves the hit by one ~eps_stop step (a
    // flipped hand-off between levels only shifts where the next level starts)
    const bool refine = lv.final_level && mode_tc(mode) && mode_terms(mode) == 3 && lv.field.kind == kFieldMlp &&
                        tc_supported(lv.field.net) && tc_uses_e4m3(lv.field.net);
    if (mode_tc(mode) && lv.field.kind == kFieldMlp && tc_supported(lv.field.net))
      tl = tc_trace_level(mode_terms(mode), lv, eps, t_max, in_list, in_count, cursor, evals, fb.list[adv], adv_count,
                          fb.st, n_max, s, refine ? fb.list[nxt] : nullptr, refine ? refine_count : nullptr);
    if (tl == TcLaunch::kRan && refine) {
      tl = tc_trace_level(mode_terms(mode), lv, eps, t_max, fb.list[nxt], refine_count, refine_cursor, evals,
                          fb.list[adv], adv_count, fb.st, n_max, s, nullptr, nullptr, /*resume=*/true);
      res.launches++;
    }
    if (tl == TcLaunch::kFailed) {  // no silent FFMA fallback: the frame fails
      nvtxRangePop();
      res.error = tc_last_error();
      res.failed_level = lv.level;
      return res;
    }
    const bool persistent = tl == TcLaunch::kRan;
    res.persistent.push_back(persistent ? 1 : 0);
    if (persistent) res.launches++;
    for (int iter = 0; !persistent && iter < lv.budget; ++iter) {
      a.iter = iter;
      a.in_list = in_list;
      a.in_count = in_count;
      a.next_list = fb.list[pong];
      a.next_count = it_counts + iter;
      {
        const size_t smem = field_smem(lv.field) + kTileCols * sizeof(int);
        const bool wide = wide_tile(lv.field);
        const int blocks = wide ? blocks_for(trace_iter_simt<1024>, 1024, smem) : blocks_for(trace_iter_simt<256>, 256, smem);
        const int grid = std::max(1, std::min(blocks, (n_max + kTileCols - 1) / kTileCols));
        if (wide)
          trace_iter_simt<1024><<<grid, 1024, smem, s>>>(a);
        else
          trace_iter_simt<256><<<grid, 256, smem, s>>>(a);
      }
      res.launches++;
      in_list = fb.list[pong];
      in_count = it_counts + iter;
      std::swap(ping, pong);
    }
    nvtxRangePop();
    if (prof) {
      prof->end(lv.level, ev, s);
      prof->acc.trace_launches += persistent ? 1 : lv.budget;
    }
    // The advanced list feeds the next level; the other two lists are free again.
    level_in_count = adv_count;
    const int new_cur = adv;
    adv = cur;
    cur = new_cur;
    (void)ping;
  }
  res.hit_list = fb.list[cur];
  res.hit_count = const_cast<int*>(level_in_count);
  return res;
}

__global__ void mark_hits_kernel(const int* list, const int* count, RayState st) {
  const int n = *count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (in_bounds(list[i], st.cap, kChkSlot)) st.hit[list[i]] = 1;
}

void launch_mark_hits(const int* list, const int* count, int n_max, RayState st, cudaStream_t s) {
  mark_hits_kernel<<<std::max(1, std::min((n_max + 255) / 256, num_sms() * 8)), 256, 0, s>>>(list, count, st);
}

__global__ void write_records_kernel(RayState st, int n, nsdf_hit_record* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    nsdf_hit_record r;
    r.hit = st.hit[i];
    r.point[0] = st.px[i];
    r.point[1] = st.py[i];
    r.point[2] = st.pz[i];
    r.t = st.t[i];
    r.level_reached = st.level_reached[i];
#pragma unroll
    for (int j = 0; j < NSDF_MAX_LEVELS; ++j) r.iterations_used[j] = st.iters[size_t(i) * kMaxLevels + j];
    r.final_distance = st.final_dist[i];
    out[st.pixel ? st.pixel[i] : i] = r;
  }
}

void launch_write_records(const RayState& st, int n, nsdf_hit_record* out, cudaStream_t s) {
  if (n <= 0) return;
  write_records_kernel<<<std::min((n + 255) / 256, num_sms() * 8), 256, 0, s>>>(st, n, out);
}

// ---------------------------------------------------------------------------------------
// Shading (shade.cpp:44-93) and the framebuffer.
// ---------------------------------------------------------------------------------------
__global__ void fb_background_kernel(RayState st, const int* n_slots, ShadeParams sp, float* rgb, float* depth,
                                     uint8_t* mask) {
  const int n = *n_slots;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int p = st.pixel[i];
    if (!in_bounds(p, st.n_pix, kChkPixel)) continue;
    rgb[size_t(3) * p + 0] = sp.background[0];
    rgb[size_t(3) * p + 1] = sp.background[1];
    rgb[size_t(3) * p + 2] = sp.background[2];
    depth[p] = 0.0f;
    mask[p] = 0;
  }
}

__global__ void pack_owned_kernel(RayState st, const int* n_slots, const float* rgb, const float* depth,
                                  const uint8_t* mask, float* p_rgb, float* p_depth, uint8_t* p_mask, int* p_pixel) {
  const int n = *n_slots;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int p = st.pixel[i];
    p_rgb[size_t(3) * i + 0] = rgb[size_t(3) * p + 0];
    p_rgb[size_t(3) * i + 1] = rgb[size_t(3) * p + 1];
    p_rgb[size_t(3) * i + 2] = rgb[size_t(3) * p + 2];
    p_depth[i] = depth[p];
    p_mask[i] = mask[p];
    p_pixel[i] = p;
  }
}

void launch_pack_owned(const RayState& st, const int* n_slots_dev, int n_max, const float* rgb, const float* depth,
                       const uint8_t* mask, float* p_rgb, float* p_depth, uint8_t* p_mask, int* p_pixel,
                       cudaStream_t s) {
  pack_owned_kernel<<<std::max(1, std::min((n_max + 255) / 256, num_sms() * 8)), 256, 0, s>>>(
      st, n_slots_dev, rgb, depth, mask, p_rgb, p_depth, p_mask, p_pixel);
}

// Inverse of pack_owned on the framebuffer's device (render_multi without peer access):
// the packed pixels of one context, copied over by a peer memcpy, land at their pixels.
__global__ void scatter_packed_kernel(const int* count, const float* p_rgb, const float* p_depth, const uint8_t* p_mask,
                                      const int* p_pixel, float* rgb, float* depth, uint8_t* mask) {
  const int n = *count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const size_t p = size_t(p_pixel[i]);
    rgb[3 * p + 0] = p_rgb[size_t(3) * i + 0];
    rgb[3 * p + 1] = p_rgb[size_t(3) * i + 1];
    rgb[3 * p + 2] = p_rgb[size_t(3) * i + 2];
    depth[p] = p_depth[i];
    mask[p] = p_mask[i];
  }
}

void launch_scatter_packed(const int* count_dev, int n_max, const float* p_rgb, const float* p_depth,
                           const uint8_t* p_mask, const int* p_pixel, float* rgb, float* depth, uint8_t* mask,
                           cudaStream_t s) {
  scatter_packed_kernel<<<std::max(1, std::min((n_max + 255) / 256, num_sms() * 8)), 256, 0, s>>>(
      count_dev, p_rgb, p_depth, p_mask, p_pixel, rgb, depth, mask);
}

void launch_fb_background(const RayState& st, const int* n_slots_dev, int n_max, const ShadeParams& sp, float* rgb,
                          float* depth, uint8_t* mask, cudaStream_t s) {
  fb_background_kernel<<<std::max(1, std::min((n_max + 255) / 256, num_sms() * 8)), 256, 0, s>>>(st, n_slots_dev, sp,
                                                                                                  rgb, depth, mask);
}

struct NormalArgs {
  DevField field;
  float time;
  const int* list;
  const int* count;
  RayState st;
  ShadeParams sp;
  int defer_fallback;
  int* fb_list;
  int* fb_count;
  float* rgb;
  float* depth;
  uint8_t* mask;
};

__device__ __forceinline__ void write_pixel(const NormalArgs& a, int slot, const float n[3]) {
  float c[3];
  const float px = a.st.px[slot], py = a.st.py[slot], pz = a.st.pz[slot];
  shade_point(a.sp, px, py, pz, n[0], n[1], n[2], c);
  const int p = a.st.pixel[slot];
  if (!in_bounds(p, a.st.n_pix, kChkPixel)) return;
  a.rgb[size_t(3) * p + 0] = c[0];
  a.rgb[size_t(3) * p + 1] = c[1];
  a.rgb[size_t(3) * p + 2] = c[2];
  a.depth[p] = a.st.t[slot];
  a.mask[p] = 1;
}

template <int kT>
__global__ void __launch_bounds__(kT) normals_shade_simt(NormalArgs a) {
  extern __shared__ __align__(16) float smem[];
  constexpr int kRays = kTileCols / 4;
  const int W = a.field.kind == kFieldMlp ? max(a.field.net.max_width, 4) : 4;
  float* bufA = smem;
  float* bufB = bufA + W * kTileCols;
  float* pts = bufB + W * kTileCols;
  float* vals = pts + 4 * kTileCols;
  int* slots = reinterpret_cast<int*>(vals + kTileCols);
  const int n = *a.count;
  const int tid = threadIdx.x;
  for (int base = blockIdx.x * kRays; base < n; base += gridDim.x * kRays) {
    const int cnt = min(kRays, n - base);
    if (tid < kRays) {
      int slot = tid < cnt && in_bounds(base + tid, a.st.cap, kChkListRead) ? a.list[base + tid] : -1;
      if (slot >= 0 && !in_bounds(slot, a.st.cap, kChkSlot)) slot = -1;
      slots[tid] = slot;
      pts[tid] = slot >= 0 ? a.st.px[slot] : 0.0f;
      pts[kRays + tid] = slot >= 0 ? a.st.py[slot] : 0.0f;
      pts[2 * kRays + tid] = slot >= 0 ? a.st.pz[slot] : 0.0f;
      pts[3 * kRays + tid] = a.time;
    }
    __syncthreads();
    field_tile<true, kT>(a.field, pts, bufA, bufB, vals);
    if (tid < 32) {
      const int slot = tid < kRays ? slots[tid] : -1;
      bool defer = false;
      if (slot >= 0) {
        float nrm[3];
        if (!normalize_normal(vals[4 * tid + 1], vals[4 * tid + 2], vals[4 * tid + 3], nrm)) {
          nrm[0] = 0.0f;
          nrm[1] = 1.0f;
          nrm[2] = 0.0f;
          defer = a.defer_fallback != 0;
        }
        if (!defer) write_pixel(a, slot, nrm);
      }
      warp_append(defer, slot, a.fb_list, a.fb_count, a.st.cap);
    }
    __syncthreads();
  }
}

int launch_normals_shade(Mode mode, const DevField& nf, float time, const int* list, const int* count, int n_max,
                         const RayState& st, const ShadeParams& sp, bool defer_fallback, int* fb_list, int* fb_count,
                         float* rgb, float* depth, uint8_t* mask, cudaStream_t s) {
  NormalArgs a{nf, time, list, count, st, sp, defer_fallback ? 1 : 0, fb_list, fb_count, rgb, depth, mask};
  if (mode_tc(mode) && nf.kind == kFieldMlp && tc_supported(nf.net)) {
    const TcLaunch r = tc_normals_shade(normal_tile_terms(mode), nf, time, list, count, n_max, st, sp, defer_fallback,
                                        fb_list, fb_count, rgb, depth, mask, s);
    if (r == TcLaunch::kRan) return NSDF_PATH_TCGEN05;
    if (r == TcLaunch::kFailed) return -1;  // tc_last_error() holds the CUDA error
  }
  const size_t smem = field_smem(nf) + kTileCols * sizeof(int);
  if (wide_tile(nf)) {
    const int grid = std::max(1, std::min(blocks_for(normals_shade_simt<1024>, 1024, smem), (n_max + 15) / 16));
    normals_shade_simt<1024><<<grid, 1024, smem, s>>>(a);
  } else {
    const int grid = std::max(1, std::min(blocks_for(normals_shade_simt<256>, 256, smem), (n_max + 15) / 16));
    normals_shade_simt<256><<<grid, 256, smem, s>>>(a);
  }
  return NSDF_PATH_SIMT;
}

// ---------------------------------------------------------------------------------------
// API-path batch kernels.
// ---------------------------------------------------------------------------------------
template <bool kGrad, int kT>
__global__ void __launch_bounds__(kT) eval_simt(DevField f, const float* pts_g, int rows, int k, float time,
                                                      float* out, float* grad, double delta, const float* fallback,
                                                      unsigned long long* counts, int normal_map) {
  extern __shared__ __align__(16) float smem[];
  constexpr int kRays = kGrad ? kTileCols / 4 : kTileCols;
  const int W = f.kind == kFieldMlp ? max(f.net.max_width, 4) : 4;
  float* bufA = smem;
  float* bufB = bufA + W * kTileCols;
  float* pts = bufB + W * kTileCols;
  float* vals = pts + 4 * kTileCols;
  const int tid = threadIdx.x;
  for (int base = blockIdx.x * kRays; base < k; base += gridDim.x * kRays) {
    if (tid < kRays) {
      const int col = base + tid;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        pts[r * kRays + tid] = col < k ? (r < rows ? pts_g[size_t(r) * k + col] : time) : 0.0f;
    }
    __syncthreads();
    field_tile<kGrad, kT>(f, pts, bufA, bufB, vals);
    if (!kGrad) {
      if (tid < kRays && base + tid < k) out[base + tid] = vals[tid];
    } else if (tid < 32) {
      const int col = base + tid;
      const bool valid = tid < kRays && col < k;
      bool outside = false, fell_back = false;
      if (valid) {
        if (!normal_map) {
          if (out) out[col] = vals[4 * tid];
          if (grad)
            for (int c = 0; c < 3; ++c) grad[size_t(c) * k + col] = vals[4 * tid + 1 + c];
        } else {
          outside = fabs(double(vals[4 * tid])) > delta;
          float nrm[3];
          if (!normalize_normal(vals[4 * tid + 1], vals[4 * tid + 2], vals[4 * tid + 3], nrm)) {
            fell_back = true;
            if (fallback) {
              for (int c = 0; c < 3; ++c) nrm[c] = fallback[size_t(c) * k + col];
            } else {
              nrm[0] = 0.0f;
              nrm[1] = 1.0f;
              nrm[2] = 0.0f;
            }
          }
          for (int c = 0; c < 3; ++c) grad[size_t(c) * k + col] = nrm[c];
        }
      }
      if (normal_map) {
        const unsigned mo = __ballot_sync(0xffffffffu, outside), mf = __ballot_sync(0xffffffffu, fell_back);
        if (tid == 0 && (mo | mf)) {
          atomicAdd(counts + 0, (unsigned long long)__popc(mo));
          atomicAdd(counts + 1, (unsigned long long)__popc(mf));
        }
      }
    }
    __syncthreads();
  }
}

template <bool kGrad>
static void launch_eval_impl(const DevField& f, const float* pts, int rows, int k, float time, float* out, float* grad,
                             double delta, const float* fallback, unsigned long long* counts, int normal_map,
                             cudaStream_t s) {
  const size_t smem = field_smem(f);
  constexpr int kRays = kGrad ? kTileCols / 4 : kTileCols;
  if (wide_tile(f)) {
    const int grid = std::max(1, std::min(blocks_for(eval_simt<kGrad, 1024>, 1024, smem), (k + kRays - 1) / kRays));
    eval_simt<kGrad, 1024><<<grid, 1024, smem, s>>>(f, pts, rows, k, time, out, grad, delta, fallback, counts,
                                                    normal_map);
  } else {
    const int grid = std::max(1, std::min(blocks_for(eval_simt<kGrad, 256>, 256, smem), (k + kRays - 1) / kRays));
    eval_simt<kGrad, 256><<<grid, 256, smem, s>>>(f, pts, rows, k, time, out, grad, delta, fallback, counts,
                                                  normal_map);
  }
}

cudaError_t launch_eval(Mode mode, const DevField& f, const float* pts, int rows, int k, float time, float* out,
                        float* grad, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  if (mode_tc(mode) && f.kind == kFieldMlp && tc_supported(f.net)) {
    const TcLaunch r = tc_eval(mode_terms(mode), f, pts, rows, k, time, out, grad, s);
    if (r == TcLaunch::kRan) return cudaSuccess;
    if (r == TcLaunch::kFailed) return tc_last_error();
  }
  if (grad)
    launch_eval_impl<true>(f, pts, rows, k, time, out, grad, 0.0, nullptr, nullptr, 0, s);
  else
    launch_eval_impl<false>(f, pts, rows, k, time, out, nullptr, 0.0, nullptr, nullptr, 0, s);
  return cudaGetLastError();
}

cudaError_t launch_normal_map(Mode mode, const DevField& f, const float* pts, int k, float time, double delta,
                              const float* fallback, float* normals, unsigned long long* counts, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  if (mode_tc(mode) && f.kind == kFieldMlp && tc_supported(f.net)) {
    const TcLaunch r = tc_normal_map(mode_terms(mode), f, pts, k, time, delta, fallback, normals, counts, s);
    if (r == TcLaunch::kRan) return cudaSuccess;
    if (r == TcLaunch::kFailed) return tc_last_error();
  }
  launch_eval_impl<true>(f, pts, 3, k, time, nullptr, normals, delta, fallback, counts, 1, s);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Per-vertex mesh normal mapping (shading::map_normals_to_mesh, mesh.cpp:122-156): the
// vertices (double) cast to float points, the fine field's value + gradient by the batch
// kernels, then this gate: |value| > delta -> violator (normal kept); |g| < 1e-8 (double
// norm of the float gradient) -> fallback (kept); else normal = g / |g| in double
// (Vec3::norm / operator/, separately rounded).
// ---------------------------------------------------------------------------------------
__global__ void cast_vertices_kernel(const double* v, int k, float* pts) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    pts[j] = __double2float_rn(v[3 * size_t(j) + 0]);
    pts[size_t(k) + j] = __double2float_rn(v[3 * size_t(j) + 1]);
    pts[2 * size_t(k) + j] = __double2float_rn(v[3 * size_t(j) + 2]);
  }
}

__global__ void mesh_map_kernel(const float* vals, const float* grads, int k, double delta, double* normals,
                                unsigned long long* counts) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    int what = 0;  // 0 mapped, 1 violator, 2 fallback
    if (fabs(double(vals[j])) > delta) {
      what = 1;
    } else {
      const double gx = grads[j], gy = grads[size_t(k) + j], gz = grads[2 * size_t(k) + j];
      const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz)));
      if (n < 1e-8) {
        what = 2;
      } else {
        normals[3 * size_t(j) + 0] = __ddiv_rn(gx, n);
        normals[3 * size_t(j) + 1] = __ddiv_rn(gy, n);
        normals[3 * size_t(j) + 2] = __ddiv_rn(gz, n);
      }
    }
    const unsigned lanes = __activemask();
    for (int w = 0; w < 3; ++w) {
      const unsigned m = __ballot_sync(lanes, what == w);
      if (m && (threadIdx.x & 31) == __ffs(lanes) - 1) atomicAdd(counts + w, (unsigned long long)__popc(m));
    }
  }
}

cudaError_t launch_map_mesh_normals(Mode mode, const DevField& f, float time, const double* vertices, int k,
                                    double delta, float* pts, float* vals, float* grads, double* normals,
                                    unsigned long long* counts, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  const int grid = std::max(1, std::min((k + 255) / 256, num_sms() * 8));
  cast_vertices_kernel<<<grid, 256, 0, s>>>(vertices, k, pts);
  if (cudaError_t e = launch_eval(mode, f, pts, 3, k, time, vals, grads, s)) return e;
  mesh_map_kernel<<<grid, 256, 0, s>>>(vals, grads, k, delta, normals, counts);
  return cudaGetLastError();
}

__global__ void shade_kernel(const float* pts, const float* nrm, int k, ShadeParams sp, float* rgb) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    float c[3];
    shade_point(sp, pts[j], pts[size_t(k) + j], pts[size_t(2) * k + j], nrm[j], nrm[size_t(k) + j],
                nrm[size_t(2) * k + j], c);
    for (int i = 0; i < 3; ++i) rgb[size_t(i) * k + j] = c[i];
  }
}

void launch_shade(const float* pts, const float* normals, int k, const ShadeParams& sp, float* rgb, cudaStream_t s) {
  if (k <= 0) return;
  shade_kernel<<<std::min((k + 255) / 256, num_sms() * 8), 256, 0, s>>>(pts, normals, k, sp, rgb);
}

// ---------------------------------------------------------------------------------------
// Mesh G-buffer (config 4).  Triangles are staged through shared memory in blocks of 256;
// each thread keeps its pixel's nearest positive hit.
// ---------------------------------------------------------------------------------------
__global__ void raycast_mesh_kernel(CamBasis c, const float* __restrict__ tv, int n_tri, float* pos, uint8_t* mask) {
  __shared__ float tri[256 * 9];
  const int npix = c.width * c.height;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  float d[3] = {0, 0, 1};
  if (pix < npix) pixel_ray(c, pix % c.width, pix / c.width, d);
  const float ox = c.origin[0], oy = c.origin[1], oz = c.origin[2];
  float best = 3.0e38f;
  for (int base = 0; base < n_tri; base += 256) {
    const int cnt = min(256, n_tri - base);
    __syncthreads();
    for (int i = threadIdx.x; i < cnt * 9; i += blockDim.x) tri[i] = tv[size_t(base) * 9 + i];
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {
      const float* t = tri + k * 9;
      const float e1x = t[3] - t[0], e1y = t[4] - t[1], e1z = t[5] - t[2];
      const float e2x = t[6] - t[0], e2y = t[7] - t[1], e2z = t[8] - t[2];
      const float px = d[1] * e2z - d[2] * e2y, py = d[2] * e2x - d[0] * e2z, pz = d[0] * e2y - d[1] * e2x;
      const float det = e1x * px + e1y * py + e1z * pz;
      if (fabsf(det) < 1e-12f) continue;
      const float inv = 1.0f / det;
      const float sx = ox - t[0], sy = oy - t[1], sz = oz - t[2];
      const float u = (sx * px + sy * py + sz * pz) * inv;
      if (u < 0.0f || u > 1.0f) continue;
      const float qx = sy * e1z - sz * e1y, qy = sz * e1x - sx * e1z, qz = sx * e1y - sy * e1x;
      const float v = (d[0] * qx + d[1] * qy + d[2] * qz) * inv;
      if (v < 0.0f || u + v > 1.0f) continue;
      const float tt = (e2x * qx + e2y * qy + e2z * qz) * inv;
      if (tt > 1e-6f && tt < best) best = tt;
    }
  }
  if (pix >= npix) return;
  const bool hit = best < 3.0e38f;
  mask[pix] = hit ? 1 : 0;
  pos[pix] = hit ? ox + best * d[0] : 0.0f;
  pos[size_t(npix) + pix] = hit ? oy + best * d[1] : 0.0f;
  pos[size_t(2) * npix + pix] = hit ? oz + best * d[2] : 0.0f;
}

void launch_raycast_mesh(const CamBasis& cb, const float* tri_verts, int n_tri, float* positions, uint8_t* mask,
                         cudaStream_t s) {
  const int npix = cb.width * cb.height;
  raycast_mesh_kernel<<<(npix + 255) / 256, 256, 0, s>>>(cb, tri_verts, n_tri, positions, mask);
}

// Positive control of the checked build: one deliberate out-of-bounds index (-1 of 1).
__global__ void check_selftest_kernel() {
  if (threadIdx.x == 0 && blockIdx.x == 0) (void)in_bounds(-1, 1, kChkSlot);
}

cudaError_t launch_check_selftest(cudaStream_t s) {
  check_selftest_kernel<<<1, 32, 0, s>>>();
  return cudaGetLastError();
}

cudaError_t check_report_engine(CheckRecord* out, bool reset) {
#if NSDF_CHECKED
  if (cudaError_t e = cudaMemcpyFromSymbol(out, g_check, sizeof(CheckRecord))) return e;
  if (reset) {
    const CheckRecord zero{};
    return cudaMemcpyToSymbol(g_check, &zero, sizeof(CheckRecord));
  }
  return cudaSuccess;
#else
  (void)reset;
  *out = CheckRecord{};
  return cudaSuccess;
#endif
}

}  // namespace nsdf_b200
