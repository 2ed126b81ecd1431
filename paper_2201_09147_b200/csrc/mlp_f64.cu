// FP64 SIREN evaluator: the certification path.
//
// The reference certifies nestings in double precision (estimate_sup_diff / verify_nesting /
// sample_near_surface, nesting.cpp:131-361, all through Field::eval_batch/grad_batch on
// Matrix<double>, i.e. mlp::forward_batch<double> / gradient_batch<double>).  This kernel
// restates that arithmetic bit for bit on the device:
//   - every output is acc = bias (value chain) or 0 (gradient chains), then
//     acc = fma(W[i,kk], x[kk], acc) for kk ascending (gemm_f64_avx2 panels and tail,
//     kernels_avx2.cpp:89-150) — each thread owns whole outputs, so no chain is split;
//   - sin(omega*x) / omega*cos(omega*x) via the double Cephes scheme with every operation
//     separately rounded (sincos_poly_avx2_d, kernels_avx2.cpp:284-333; constants
//     sincos_poly.hpp:26-40); the quadrant uses the lanes' 32-bit truncation (cvttpd);
//   - Alg. 2 chains (mlp.cpp:104-167): G0_c = W0[i,c]*dphi, G_i = gemm(W_i, G)*dphi,
//     grad_c = Wn . G_c from 0.
// This TU is compiled with -fmad=false; the explicit __fma_rn are the only fused ops.
//
// Tile: 16 activation columns (16 points, or 4 points x 4 chains), activations resident in
// shared memory as two ping-pong buffers [max_width][16] of doubles (64 KB at width 256, so
// three CTAs share an SM); per hidden layer pass a thread owns 4 output rows x 4 columns
// (rb = tid/4, cb = tid%4).
#include <algorithm>

#include <cstdio>
#include <cstdlib>

#include "common_f64.cuh"
#include "engine.cuh"

namespace nsdf_b200 {

namespace {

constexpr int kCols64 = 16;
constexpr int kThreads64 = 256;

// value -> s; derivative -> dphi = omega*cos (sine_f64_avx2, kernels_avx2.cpp:336-352)
__device__ __forceinline__ void activate_d(const DevNet& n, double z, double& s, double& dphi) {
  if (n.activation == NSDF_ACT_SINE) {
    double c;
    sincos_ref_d(__dmul_rn(n.omega_d, z), s, c);
    dphi = __dmul_rn(n.omega_d, c);
  } else {
    s = z;
    dphi = 1.0;
  }
}

template <bool kGrad>
__device__ void f64_input_layer(const DevNet& n, const double* __restrict__ pts, double* __restrict__ out) {
  constexpr int kRays = kGrad ? kCols64 / 4 : kCols64;
  const int M = n.rows[0], K = n.cols[0];
  const double* __restrict__ w = n.w64[0];
  const double* __restrict__ b = n.b64[0];
  for (int idx = threadIdx.x; idx < M * kRays; idx += kThreads64) {
    const int r = idx / kRays, ray = idx - r * kRays;
    double z = __ldg(b + r);
    for (int kk = 0; kk < K; ++kk) z = __fma_rn(__ldg(w + r * K + kk), pts[kk * kRays + ray], z);
    double s, dphi;
    activate_d(n, z, s, dphi);
    if (kGrad) {
      double* o = out + r * kCols64 + ray * 4;
      o[0] = s;
      o[1] = __dmul_rn(__ldg(w + r * K + 0), dphi);  // scale_rows: W0[i,c] * dphi
      o[2] = __dmul_rn(__ldg(w + r * K + 1), dphi);
      o[3] = __dmul_rn(__ldg(w + r * K + 2), dphi);
    } else {
      out[r * kCols64 + ray] = s;
    }
  }
}

template <bool kGrad>
__device__ void f64_hidden_layer(const DevNet& n, int l, const double* __restrict__ in, double* __restrict__ out) {
  const int M = n.rows[l], K = n.cols[l], Mp = n.rows_pad[l];
  const double* __restrict__ wt = n.wt64[l];
  const double* __restrict__ b = n.b64[l];
  const int cb = threadIdx.x & 3, rb = threadIdx.x >> 2;
  const int c0 = cb * 4;
  for (int r0 = rb * 4; r0 < M; r0 += 256) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double bi = r0 + i < M ? __ldg(b + r0 + i) : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = (!kGrad || j == 0) ? bi : 0.0;
    }
    const double* __restrict__ wp = wt + r0;
    const double* __restrict__ xp = in + c0;
#pragma unroll 2
    for (int kk = 0; kk < K; ++kk) {
      const double2 w01 = __ldg(reinterpret_cast<const double2*>(wp + size_t(kk) * Mp));
      const double2 w23 = __ldg(reinterpret_cast<const double2*>(wp + size_t(kk) * Mp + 2));
      const double2 x01 = *reinterpret_cast<const double2*>(xp + kk * kCols64);
      const double2 x23 = *reinterpret_cast<const double2*>(xp + kk * kCols64 + 2);
      const double wv[4] = {w01.x, w01.y, w23.x, w23.y};
      const double xv[4] = {x01.x, x01.y, x23.x, x23.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(wv[i], xv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (r0 + i >= M) break;
      double* o = out + (r0 + i) * kCols64 + c0;
      if (kGrad) {
        double s, dphi;
        activate_d(n, acc[i][0], s, dphi);
        o[0] = s;
        o[1] = __dmul_rn(acc[i][1], dphi);  // hadamard(gemm, dphi)
        o[2] = __dmul_rn(acc[i][2], dphi);
        o[3] = __dmul_rn(acc[i][3], dphi);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double s, dphi;
          activate_d(n, acc[i][j], s, dphi);
          o[j] = s;
        }
      }
    }
  }
}

// pts_g: rows x k (row-major, one point per column); a 3-row batch for a 4-input net gets
// the constant `time` row (with_time_row, field.cpp:213-220).  out: k; grad: 3 x k.
template <bool kGrad>
__global__ void __launch_bounds__(kThreads64) eval_f64_kernel(DevNet n, const double* __restrict__ pts_g, int rows,
                                                              int k, double time, double* out, double* grad) {
  extern __shared__ __align__(16) double smem64[];
  constexpr int kRays = kGrad ? kCols64 / 4 : kCols64;
  const int W = max(n.max_width, 4);
  double* bufA = smem64;
  double* bufB = bufA + W * kCols64;
  double* pts = bufB + W * kCols64;
  const int L = n.n_layers;
  const int tid = threadIdx.x;
  for (int base = blockIdx.x * kRays; base < k; base += gridDim.x * kRays) {
    if (tid < kRays) {
      const int col = base + tid;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        pts[r * kRays + tid] = col < k ? (r < rows ? pts_g[size_t(r) * k + col] : time) : 0.0;
    }
    __syncthreads();
    const double* fin;
    if (L == 1) {
      fin = nullptr;  // affine network (mlp.cpp:115-126): handled below
    } else {
      f64_input_layer<kGrad>(n, pts, bufA);
      __syncthreads();
      double* in = bufA;
      double* o = bufB;
      for (int l = 1; l + 1 < L; ++l) {
        f64_hidden_layer<kGrad>(n, l, in, o);
        __syncthreads();
        double* t = in;
        in = o;
        o = t;
      }
      fin = in;
    }
    // output layer: value from the bias, tangents from 0 (gemm without bias)
    for (int col = tid; col < kCols64; col += kThreads64) {
      const int ray = kGrad ? col >> 2 : col, chain = kGrad ? col & 3 : 0;
      const int g = base + ray;
      if (ray >= kRays || g >= k) continue;
      double acc;
      if (L == 1) {
        if (chain == 0) {
          acc = __ldg(n.b64[0]);
          for (int kk = 0; kk < n.cols[0]; ++kk) acc = __fma_rn(__ldg(n.w64[0] + kk), pts[kk * kRays + ray], acc);
        } else {
          acc = __ldg(n.w64[0] + chain - 1);  // the gradient is the weight row
        }
      } else {
        const int K = n.cols[L - 1];
        const double* __restrict__ w = n.w64[L - 1];
        acc = chain == 0 ? __ldg(n.b64[L - 1]) : 0.0;
        for (int kk = 0; kk < K; ++kk) acc = __fma_rn(__ldg(w + kk), fin[kk * kCols64 + col], acc);
      }
      if (chain == 0) {
        if (out) out[g] = acc;
      } else if (grad) {
        grad[size_t(chain - 1) * k + g] = acc;
      }
    }
    __syncthreads();
  }
}

template <bool kGrad>
cudaError_t launch_f64(const DevNet& n, const double* pts, int rows, int k, double time, double* out, double* grad,
                cudaStream_t s) {
  const int W = std::max(n.max_width, 4);
  const size_t smem = size_t(2) * W * kCols64 * sizeof(double) + 4 * kCols64 * sizeof(double);
  const KernelCfg kc = kernel_cfg(reinterpret_cast<const void*>(eval_f64_kernel<kGrad>), kThreads64, smem);
  if (kc.err != cudaSuccess) return kc.err;
  const int sms = kc.sms;
  const int per_sm = std::max(1, int((228 * 1024) / (smem + 1024)));
  constexpr int kRays = kGrad ? kCols64 / 4 : kCols64;
  const int grid = std::max(1, std::min(sms * std::min(per_sm, 4), (k + kRays - 1) / kRays));
  if (getenv("NSDF_DEBUG_LAUNCH"))
    fprintf(stderr, "launch_f64<%d> W=%d smem=%zu grid=%d sms=%d occ=%d pending=%s\n", int(kGrad), W, smem, grid, sms,
            kc.occupancy, cudaGetErrorString(cudaPeekAtLastError()));
  eval_f64_kernel<kGrad><<<grid, kThreads64, smem, s>>>(n, pts, rows, k, time, out, grad);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_eval_f64(const DevNet& n, const double* pts, int rows, int k, double time, double* out,
                            double* grad, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  return grad ? launch_f64<true>(n, pts, rows, k, time, out, grad, s)
              : launch_f64<false>(n, pts, rows, k, time, out, nullptr, s);
}

// ---------------------------------------------------------------------------------------
// Certification on the device: the Newton projection of
// sample_near_surface (nesting.cpp:98-127) with the points resident, and the FP64 analytic
// members so that every bound field evaluates here.
// ---------------------------------------------------------------------------------------
namespace {

__global__ void analytic_f64_kernel(DevField f, const double* pts, int k, double* out, double* grad) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    const double x = pts[j], y = pts[size_t(k) + j], z = pts[2 * size_t(k) + j];
    if (out) out[j] = analytic_eval(f, x, y, z);
    if (grad) {
      double g[3];
      analytic_grad(f, x, y, z, g);
      for (int r = 0; r < 3; ++r) grad[size_t(r) * k + j] = g[r];
    }
  }
}

int grid_for(int k) { return std::max(1, std::min((k + 255) / 256, 148 * 8)); }

// Vec3 array (x y z per point) -> 3 x k rows
__global__ void aos_to_rows_kernel(const double* v, int k, double* p) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    for (int r = 0; r < 3; ++r) p[size_t(r) * k + j] = v[3 * size_t(j) + r];
}

// p -= (f / |g|^2) g where |g|^2 >= 1e-16 (separately rounded, left to right)
__global__ void newton_kernel(double* p, const double* f, const double* g, int k) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    const double gx = g[j], gy = g[size_t(k) + j], gz = g[2 * size_t(k) + j];
    const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz));
    if (n2 < 1e-16) continue;
    const double s = __ddiv_rn(f[j], n2);
    p[j] = __dsub_rn(p[j], __dmul_rn(s, gx));
    p[size_t(k) + j] = __dsub_rn(p[size_t(k) + j], __dmul_rn(s, gy));
    p[2 * size_t(k) + j] = __dsub_rn(p[2 * size_t(k) + j], __dmul_rn(s, gz));
  }
}

constexpr int kScanBlock = 1024;

// per 1024-point block: number of kept points (|f| <= tol)
__global__ void keep_count_kernel(const double* f, int k, double tol, int* block_counts) {
  const int j = blockIdx.x * kScanBlock + threadIdx.x;
  const bool keep = j < k && fabs(f[j]) <= tol;
  const int n = __syncthreads_count(keep);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = n;
}

// exclusive scan of the block counts (<= 1024 blocks, one CTA); total -> counts[n_blocks]
__global__ void scan_counts_kernel(int* counts, int n_blocks) {
  __shared__ int sh[kScanBlock];
  const int i = threadIdx.x;
  const int v = i < n_blocks ? counts[i] : 0;
  sh[i] = v;
  __syncthreads();
  for (int o = 1; o < kScanBlock; o <<= 1) {
    const int add = i >= o ? sh[i - o] : 0;
    __syncthreads();
    sh[i] += add;
    __syncthreads();
  }
  if (i < n_blocks) counts[i] = sh[i] - v;
  if (i == kScanBlock - 1) counts[n_blocks] = sh[i];
}

// kept points and their gradients, in input order, as Vec3 arrays
__global__ void keep_scatter_kernel(const double* p, const double* f, const double* g, int k, double tol,
                                    const int* offsets, double* kept, double* kept_g) {
  __shared__ int warp_base[kScanBlock / 32];
  const int j = blockIdx.x * kScanBlock + threadIdx.x;
  const bool keep = j < k && fabs(f[j]) <= tol;
  const unsigned m = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_base[w] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < kScanBlock / 32; ++i) {
      const int c = warp_base[i];
      warp_base[i] = run;
      run += c;
    }
  }
  __syncthreads();
  if (!keep) return;
  const size_t o = size_t(offsets[blockIdx.x] + warp_base[w] + __popc(m & ((1u << lane) - 1u)));
  for (int r = 0; r < 3; ++r) {
    kept[3 * o + r] = p[size_t(r) * k + j];
    kept_g[3 * o + r] = g[size_t(r) * k + j];
  }
}

}  // namespace

cudaError_t launch_eval_field_f64(const DevField& f, const double* pts, int rows, int k, double time, double* out,
                                  double* grad, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  if (f.kind == kFieldMlp) return launch_eval_f64(f.net, pts, rows, k, time, out, grad, s);
  analytic_f64_kernel<<<grid_for(k), 256, 0, s>>>(f, pts, k, out, grad);
  return cudaGetLastError();
}

size_t projection_workspace_doubles(int k) { return size_t(k) * 16 + 2 * (size_t(k) / kScanBlock + 2); }

cudaError_t launch_project_to_surface(const DevField& f, double time, const double* cand, int k, double keep_tol,
                                      int steps, double* ws, double* kept, double* kept_g, int* d_count,
                                      cudaStream_t s) {
  if (k <= 0) return cudaMemsetAsync(d_count, 0, sizeof(int), s);
  double* p = ws;
  double* fv = p + 3 * size_t(k);
  double* g = fv + size_t(k);
  int* counts = reinterpret_cast<int*>(g + 3 * size_t(k));
  const int n_blocks = (k + kScanBlock - 1) / kScanBlock;
  if (n_blocks > kScanBlock) return cudaErrorInvalidValue;  // batches are <= 2^20 points
  aos_to_rows_kernel<<<grid_for(k), 256, 0, s>>>(cand, k, p);
  for (int step = 0; step < steps; ++step) {
    if (cudaError_t e = launch_eval_field_f64(f, p, 3, k, time, fv, g, s)) return e;
    newton_kernel<<<grid_for(k), 256, 0, s>>>(p, fv, g, k);
  }
  if (cudaError_t e = launch_eval_field_f64(f, p, 3, k, time, fv, g, s)) return e;
  keep_count_kernel<<<n_blocks, kScanBlock, 0, s>>>(fv, k, keep_tol, counts);
  scan_counts_kernel<<<1, kScanBlock, 0, s>>>(counts, n_blocks);
  keep_scatter_kernel<<<n_blocks, kScanBlock, 0, s>>>(p, fv, g, k, keep_tol, counts, kept, kept_g);
  if (cudaError_t e = cudaMemcpyAsync(d_count, counts + n_blocks, sizeof(int), cudaMemcpyDeviceToDevice, s)) return e;
  return cudaGetLastError();
}

}  // namespace nsdf_b200
