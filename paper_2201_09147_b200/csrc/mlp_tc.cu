// tcgen05 fast path of the SIREN evaluator (north_star subsystems 1-3).
//
// A CTA evaluates tiles of 128 TMEM lanes: 128 rays (forward) or 32 rays x 4 chains (value +
// 3 input tangents: the "width x 4" analytic-normal tile).  Per tile:
//
//   layer 0              a K = 32 MMA: A0 (TMEM) = the point split into three fp16 parts (+
//                        ones for the bias), B0 = fp16 hi/lo parts of omega*W0 and omega*b0
//                        (built per CTA at launch) -> D0 = omega*(W0 p + b0) in TMEM
//   biases               hidden weights hold omega*W; one extra K = 16 MMA per hidden layer
//                        (constant ones block x 3-part omega*b) -> every accumulator is the
//                        sine argument in radians
//   hidden layers        D[128 x W] (fp32, TMEM) = A[128 x W] (fp16 hi/lo, TMEM: written in
//                        place over the previous layer's accumulator) . W_l^T (fp16
//                        hi/lo): tcgen05.mma.cta_group::1.kind::f16, M=128 N=W K=16, three
//                        terms per K step (split precision) — or, for 128/256-wide nets at
//                        omega0 <= 15, A_hi.W_hi in f16 + both corrections as one
//                        kind::f8f6f4 K=32 MMA (mlp_tc.cuh tc_split8) — issued by one thread; 256-wide
//                        layers as two N = 128 column blocks with their own completion
//                        barriers (the epilogue of block 0 runs under block 1's MMAs and the
//                        next layer follows without a drain); weights SMEM-resident (64-wide)
//                        or streamed in (N-block, K chunk) pieces of W*32 halves through a
//                        2-3 stage cp.async.bulk ring by a producer warp (pre-arranged in the
//                        UMMA canonical layout at upload, so a piece is one contiguous copy)
//   K streaming          16-column block b belongs to column group b % groups; the MMA of
//                        layer m+1 consumes block rows as the epilogue of layer m writes them
//                        (kready mbarriers); accumulators alternate between two TMEM regions
//   epilogue             tcgen05.ld 32x32b.x16 (one block ahead) -> one FFMA forms
//                        omega*(z + b) in radians -> MUFU sine -> fp16 hi/lo -> tcgen05.st
//                        into the block's own columns = the next layer's A;
//                        tangent lanes multiply by omega*cos of their ray's value lane (warp
//                        shuffle); the last hidden layer folds in the 1 x W output layer
//   consumer             persistent trace (a whole level per launch, rows refilled from the
//                        level's list) | normal + shade + framebuffer | batch outputs
//
// Warp roles: warp 0 = MMA issuer (+ TMEM allocator), warp 1 = weight producer (streamed
// nets), then 4 epilogue warps per column group (warp w reads TMEM lanes 32*(w%4) .. +31).
// 64-wide nets run 4 CTAs per SM, 128-wide 2, 256-wide 1 (SMEM / TMEM / register bound).
//
// SMEM operand layout (K-major, SWIZZLE_NONE canonical): element (row r, k) of an R-row
// operand at ((k/8)*(R/8) + r/8)*64 + (r%8)*8 + k%8 halves, i.e. 8x16-byte core matrices;
// descriptor SBO = 128 B (next 8 rows), LBO = R*16 B (next 8 k).
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device_ops.cuh"
#include "mlp_tc.cuh"

namespace nsdf_b200 {

namespace {

constexpr int kRows = 128;   // TMEM lanes per tile
constexpr int kKC = 32;      // K elements per streamed weight chunk
constexpr int kMaxStages = 4;  // weight ring depth: tc_stages(W) (256-wide: 3 — 2 starves the
                               // N-block pipeline at layer boundaries, 4 gains nothing more;
                               // 128-wide: 3 — level 1.65 -> 1.57 ms, 4 the same)
#ifndef NSDF_TC_STAGES256
#define NSDF_TC_STAGES256 3
#endif
#ifndef NSDF_TC_STAGES128
#define NSDF_TC_STAGES128 3
#endif
__host__ __device__ constexpr int tc_stages(int W) { return W == 256 ? NSDF_TC_STAGES256 : (W == 128 ? NSDF_TC_STAGES128 : 2); }
static_assert(NSDF_TC_STAGES256 >= 2 && NSDF_TC_STAGES256 <= kMaxStages, "ring depth");
constexpr int kBlk = 16;     // columns per epilogue block = K per MMA step
constexpr int kMaxSub = 8;   // max blocks per column group per layer (kready barriers)
constexpr float kHalfPi = 1.5707963267948966f;
// debug timeline buffer (NSDF_TC_TIMELINE): tile marks of CTA 0, MMA issuer waits, tile
// count, then per CTA: globaltimer at start and end, tiles run
// Compiled in only with -DNSDF_TC_TIMELINE_BUILD=1 (build.py: env NSDF_TC_TIMELINE_BUILD=1):
// even never-taken instrumentation branches cost ~3% in the tile loops.
#ifndef NSDF_TC_TIMELINE_BUILD
#define NSDF_TC_TIMELINE_BUILD 0
#endif
constexpr bool kTimeline = NSDF_TC_TIMELINE_BUILD != 0;

constexpr int kDbgTiles = 65 * 16 + 64 * 4;
constexpr int kDbgCta = kDbgTiles + 8;
constexpr int kDbgMaxCta = 2048;
constexpr int kDbgTileT = kDbgCta + 5 * kDbgMaxCta;  // CTA 0: clock64 at each tile's start
constexpr int kDbgMaxTiles = 2048;
constexpr int kDbgSize = kDbgTileT + kDbgMaxTiles;
__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- PTX wrappers ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
// mbarrier wait: a plain try_wait loop (a runtime-selectable suspend-time hint variant
// cost 2.8% per frame: two loop bodies behind a branch at every wait).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t a = smem_addr(bar);
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// The MMA issuer runs as a whole converged warp (its operands stay warp-uniform, so they
// live in uniform registers); tcgen05.mma / commit are issued by one elected lane.  Issued
// from a single divergent lane instead, every MMA was wrapped in a uniformity loop.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Asynchronous 32x32b.x16 load: the registers are only valid after tmem_wait16 (which
// names them as outputs, so the compiler cannot read them earlier).
__device__ __forceinline__ void tmem_issue16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait16(uint32_t (&r)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]: the A operand read from tensor memory (128 lanes = rows,
// K packed two fp16 per 32-bit column, 8 columns per K = 16 step).
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// The same with E4M3 operands (kind::f8f6f4, K = 32 per instruction: four fp8 per 32-bit TMEM
// column, 8 columns), accumulating into the same FP32 accumulator as the f16 MMAs.
__device__ __forceinline__ void tc_mma_ts_f8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc));
}
// Four values -> four E4M3 bytes, the first in the lowest byte (K order within a column).
__device__ __forceinline__ uint32_t pack_e4m3x4(float a, float b, float c, float d) {
  const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
  const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(c, d), __NV_SATFINITE, __NV_E4M3);
  return lo | (hi << 16);
}
// Each lane writes 8 consecutive 32-bit columns of its own TMEM lane.
__device__ __forceinline__ void tmem_st8(uint32_t taddr, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3,
                                         uint32_t w4, uint32_t w5, uint32_t w6, uint32_t w7) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(w0),
               "r"(w1), "r"(w2), "r"(w3), "r"(w4), "r"(w5), "r"(w6), "r"(w7)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// UMMA shared-memory descriptor, K-major SWIZZLE_NONE (sm_100 version bit 46).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46);
}
// Instruction descriptor kind::f16: D f32, A/B f16, both K-major, M=128, N.
__host__ __device__ constexpr uint32_t umma_idesc(int n) {
  return (1u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(kRows >> 4) << 24);
}

// Offset (in halves) of element (row, k) in a 128-row canonical operand.
__device__ __forceinline__ int a_off(int row, int k) { return ((k >> 3) * (kRows / 8) + (row >> 3)) * 64 + (row & 7) * 8; }

// sin(omega * z) on the MUFU pipe: the argument is formed in radians by one FFMA
// (omega folded into the scale and the bias) and fed to sin.approx, which ptxas lowers to
// FMUL.RZ(x, 1/2pi) + MUFU.SIN: the hardware reduces the revolutions exactly, so the only
// error beyond the fp32 rounding of x itself (ulp(x) ~1e-5 rad at |x| ~ 150, shared by any
// fp32 reduction including the reference's Cody-Waite) is one RZ rounding of x/2pi.
// 3 issue slots per activation instead of 7 for an explicit turns reduction.
__device__ __forceinline__ float fast_sin(float x) { return __sinf(x); }

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// Low parts of a split-precision pair: fp16(x - float(fp16(x))).
// (one packed FFMA2: a - hi exactly, for both values of the pair)
__device__ __forceinline__ uint32_t pack_half2_lo(float a, float b, uint32_t hi) {
  const __half2 h = *reinterpret_cast<const __half2*>(&hi);
  const float2 d = __ffma2_rn(__half22float2(h), make_float2(-1.0f, -1.0f), make_float2(a, b));
  return pack_half2(d.x, d.y);
}

// ---- kernel parameters -------------------------------------------------------------------
enum TcOp : int { kOpTrace = 0, kOpNormals = 1, kOpEval = 2, kOpNormalMap = 3 };

struct TcNet {
  int n_layers, width, input_dim;
  float omega;
  const __half* wq;                 // hidden layers [h][hi | lo][W*W] of omega*W, canonical chunked layout
  const float* w0;                  // layer 0, row-major W x input_dim (fp32)
  const float* b;                   // biases, [n_layers-1][W] (fp32)
  const float* wout;                // output row (fp32), W
  float bout;
  float scale, inv_scale;           // 2^tc_shift and its inverse (hidden weights/biases scaled)
  int f8_mask;                      // DevNet::tc_f8_mask
};

struct TcArgs {
  TcNet net;
  int op;
  int terms;  // 3 = split-fp16 (A_hi.W_hi + A_lo.W_hi + A_hi.W_lo), 1 = plain fp16
  int claim_div;  // persistent trace: claim granularity = n / (grid * claim_div), clamped to [1, 32]
  int min_items;  // persistent trace: rays per active CTA at least this (fewer CTAs for short lists)
  // trace (persistent level)
  LevelDesc lv;
  float eps, t_max;
  const int* in_list;
  const int* in_count;
  int* adv_list;
  int* adv_count;
  int* cursor;   // claim cursor into in_list
  int* evals;    // evaluation counter
  // E4M3 final levels: a ray whose stop decision lies within kRefineBand of eps is parked
  // (state written back, the evaluation not counted) on refine_list; a second launch with
  // the fp16 correction terms resumes those rays (resume: iteration count from st.iters)
  int* refine_list;
  int* refine_count;
  int resume;
  RayState st;
  // normals
  float time;
  ShadeParams sp;
  int defer_fallback;
  int* fb_list;
  int* fb_count;
  float* rgb;
  float* depth;
  uint8_t* mask;
  // eval
  const float* pts;
  int rows, k;
  float* out;
  float* grad;
  // normal map (neural_normal_map semantics, shade.cpp:8-42)
  double delta;
  const float* fallback;
  unsigned long long* counts;
  long long* dbg;  // debug timeline (NSDF_TC_TIMELINE): CTA 0, epilogue thread 0
  int dbg_skip;    // first tile recorded (NSDF_TC_TIMELINE_SKIP)
};

// Layer 0 runs on the tensor cores as a K = 32 MMA: each row's A0 holds its point split
// into three fp16 parts plus ones for the bias, B0 the matching fp16 hi/lo parts of
// omega*W0 and a three-part omega*b0 (time folded in), so D0 = omega*(W0 p + b0) to ~2^-22.
//   k 0-2: p_hi  3-5: p_mid  6-8: p_lo  9: 1      (x W_hi, W_hi, W_hi, b_hi)
//   k 10-12: p_hi  13-15: p_mid  16: 1  17: 1     (x W_lo, W_lo, b_mid, b_lo)
// A tangent row c (normal tiles) holds ones at k = c and 10 + c, so its D0 = omega*W0[:, c].
constexpr int kK0 = 32;

// Dynamic shared-memory carve-up.  SWIZZLE_NONE operands need 16-byte alignment only.
struct TcSmem {
  __half* wst;          // resident hidden weights, or [tc_stages(W)] streamed weight chunks
  __half* b0;           // [W x 32] layer-0 B operand
  __half* bb;           // [L-2][W x 16] bias B operand of each hidden layer: omega*b in 3 fp16 parts
  __half* ones;         // [128 x 16] bias A operand: ones at k = 0..2 on value rows
  float* wout;          // [W]
  float* part;          // [3][kRows] partial output dots of column groups 1..3
  int* stage_buf;       // [kStageCap] staged compaction appends (persistent trace)
  int* stage_count;
  int* stage_base;      // flush base broadcast
  uint64_t* bars;       // full[kMaxStages], empty[kMaxStages], kready[kMaxSub], a0ready, tstart, dfull[2]
  uint32_t* tmem_base;
  int* done;            // persistent level: no more tiles
};
constexpr int kStageCap = 512;
// |f - eps| below which an E4M3 final level defers a ray's stop decision to the fp16-term
// resume launch: > 2x the largest E4M3-vs-fp16 difference of f measured on the fixtures
// (2.1e-5), so every stop at the evaluated point is decided as the fp16 terms would
constexpr float kRefineBand = 5e-5f;
constexpr int kNumBars = 2 * kMaxStages + kMaxSub + 4;  // full, empty, kready, a0ready, tstart, dfull[2]

__host__ __device__ inline size_t tc_weight_bytes(int W, int L, int terms, bool resident) {
  const int nw = terms == 3 ? 2 : 1;
  // resident: every hidden layer's [hi | lo] pair, as laid out in global memory
  return resident ? size_t(L - 2) * W * W * 2 * tc_parts(W) : size_t(tc_stages(W)) * W * kKC * 2 * nw;
}

__host__ __device__ inline size_t tc_smem_bytes(int W, int L, int terms, bool resident, bool persist) {
  size_t b = 0;
  b += tc_weight_bytes(W, L, terms, resident);
  b += size_t(W) * kK0 * 2;
  b += size_t(L - 2) * W * kBlk * 2 + size_t(kRows) * kBlk * 2;
  b += size_t(W) * 4;
  b += (W == 64 ? 0 : size_t(3) * kRows * 4);
  b += persist ? size_t(kStageCap) * 4 + 16 : 16;
  b += kNumBars * 8 + 32;
  return b + 128;  // alignment slack
}

__device__ inline TcSmem tc_carve(uint8_t* raw, int W, int L, int terms, bool resident, bool persist) {
  size_t off = 0;
  auto take = [&](size_t bytes, size_t align) {
    off = (off + align - 1) / align * align;
    uint8_t* p = raw + off;
    off += bytes;
    return p;
  };
  TcSmem s;
  s.wst = reinterpret_cast<__half*>(take(tc_weight_bytes(W, L, terms, resident), 128));
  s.b0 = reinterpret_cast<__half*>(take(size_t(W) * kK0 * 2, 128));
  s.bb = reinterpret_cast<__half*>(take(size_t(L - 2) * W * kBlk * 2, 128));
  s.ones = reinterpret_cast<__half*>(take(size_t(kRows) * kBlk * 2, 128));
  s.wout = reinterpret_cast<float*>(take(size_t(W) * 4, 16));
  s.part = reinterpret_cast<float*>(take(W == 64 ? 0 : size_t(3) * kRows * 4, 16));
  s.stage_buf = reinterpret_cast<int*>(take(persist ? size_t(kStageCap) * 4 : 0, 16));
  s.stage_count = reinterpret_cast<int*>(take(16, 16));
  s.stage_base = s.stage_count + 1;
  s.done = s.stage_count + 2;
  s.bars = reinterpret_cast<uint64_t*>(take(kNumBars * 8, 8));
  s.tmem_base = reinterpret_cast<uint32_t*>(take(16, 16));
  return s;
}

// Offset (in halves) of element (n, k) of a [W x 32] K-major canonical operand.
__device__ __forceinline__ int b0_off(int W, int n, int k) { return ((k >> 3) * (W >> 3) + (n >> 3)) * 64 + (n & 7) * 8 + (k & 7); }

// fp32 -> three fp16 parts (hi + mid + lo = x to ~2^-33 relative, subnormals aside).
__device__ __forceinline__ void split3(float x, __half& hi, __half& mid, __half& lo) {
  hi = __float2half_rn(x);
  const float r = x - __half2float(hi);
  mid = __float2half_rn(r);
  lo = __float2half_rn(r - __half2float(mid));
}

// Per-row inputs of a non-trace tile, software-pipelined two tiles ahead: the list slot of
// tile t+2 is loaded while tile t runs, its point while tile t+1 runs.
struct RowIn {
  int slot;
  float p[3];
};

__device__ __forceinline__ int load_slot(const TcArgs& a, int item, int n_items) {
  if (item >= n_items) return -1;
  if (a.op == kOpEval || a.op == kOpNormalMap) return item;
  const int slot = __ldg(a.in_list + item);
  return in_bounds(slot, a.st.cap, kChkSlot) ? slot : -1;
}

__device__ __forceinline__ RowIn load_row(const TcArgs& a, int slot) {
  RowIn r;
  r.slot = slot;
  r.p[0] = r.p[1] = r.p[2] = 0.0f;
  if (slot < 0) return r;
  if (a.op == kOpEval || a.op == kOpNormalMap) {
    for (int k = 0; k < 3; ++k) r.p[k] = __ldg(a.pts + size_t(k) * a.k + slot);
    return r;
  }
  r.p[0] = a.st.px[slot];
  r.p[1] = a.st.py[slot];
  r.p[2] = a.st.pz[slot];
  return r;
}

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// Named barrier with an OR vote over the participating threads.
__device__ __forceinline__ bool bar_vote_any(int id, int threads, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(uint32_t(pred)), "r"(id), "r"(threads)
      : "memory");
  return r != 0;
}
// Claim ticket (the cursor counts claims): atom.inc, which the compiler cannot turn into a
// warp-aggregated atomic.  An aggregated fetch-add broadcasts the old value with a shuffle
// right after the atomic, putting the contended atomic's round trip on the critical path;
// here the result is only waited for where it is used (claims run one reservation ahead).
__device__ __forceinline__ int fetch_ticket(int* p) {
  unsigned old;
  asm volatile("atom.global.inc.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(0x7fffffffu) : "memory");
  return int(old);
}
// Position of the n-th (0-based) set bit of m (n < popc(m)).
__device__ __forceinline__ int nth_set_bit(uint32_t m, int n) {
  int pos = 0;
#pragma unroll
  for (int w = 16; w > 0; w >>= 1) {
    const int c = __popc(m & ((1u << w) - 1u));
    if (n >= c) {
      n -= c;
      m >>= w;
      pos += w;
    }
  }
  return pos;
}

// CTA-local staging of compaction appends: warps append with shared atomics; the staged
// slots are flushed to the global list with one global atomic per flush (every few tiles)
// instead of one per warp per tile.
struct StageList {
  int* buf;
  int* count;
};

__device__ __forceinline__ void stage_append(bool pred, int value, StageList s) {
  const unsigned mask = __ballot_sync(0xffffffffu, pred);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(s.count, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  const int at = base + __popc(mask & ((1u << lane) - 1u));
  if (pred && in_bounds(at, kStageCap, kChkStage)) s.buf[at] = value;
}

// Flush body for callers that already synchronised the appends (the count is uniform).
// `cap`: capacity of the destination list.
__device__ __forceinline__ void stage_flush_now(StageList s, int* list, int* gcount, int* gbase, int ctid, int cap) {
  const int n = min(*s.count, kStageCap);
  if (ctid == 0) *gbase = atomicAdd(gcount, n);
  named_bar(2, 128);
  const int base = *gbase;
  for (int i = ctid; i < n; i += 128)
    if (in_bounds(base + i, cap, kChkListWrite)) list[base + i] = s.buf[i];
  named_bar(2, 128);
  if (ctid == 0) *s.count = 0;
}

// Called by the 128 consumer threads (named barrier 2) after a tile's appends.
__device__ __forceinline__ void stage_flush(StageList s, int* list, int* gcount, int* gbase, int ctid, bool force,
                                            int cap) {
  named_bar(2, 128);
  const int n = min(*s.count, kStageCap);
  if (n == 0 || (!force && n <= kStageCap - kRows)) return;  // uniform decision
  if (ctid == 0) *gbase = atomicAdd(gcount, n);
  named_bar(2, 128);
  const int base = *gbase;
  for (int i = ctid; i < n; i += 128)
    if (in_bounds(base + i, cap, kChkListWrite)) list[base + i] = s.buf[i];
  named_bar(2, 128);
  if (ctid == 0) *s.count = 0;
}

// Ray-slot pipeline of the persistent trace (kPersist): every epilogue row of group 0 owns
// one ray; when a ray leaves the level its row takes a prefetched ray from the warp's pool
// (one prefetch register set per lane).  A lane's prefetch runs NEED -> LISTED (claimed
// list item, slot load in flight) -> READY (ray state loads in flight), one stage per
// tile, so no load sits on the critical path of a tile.
enum PfStage : int { kPfNeed = 0, kPfListed = 1, kPfReady = 2 };

// The fused SIREN tile kernel.
//  kGroups   column groups of 4 epilogue warps; 16-column block b of every layer belongs
//            to group b % kGroups (TMEM lane quadrant = warp % 4)
//  kResident all hidden-layer weights stay in SMEM (64-wide nets); otherwise a producer
//            warp streams (N-block, K chunk) pieces through a tc_stages(W)-deep ring
//  kPersist  one launch traces a whole level: rows are refilled from the level's input
//            list until it drains (sphere_trace_level, trace.cpp:61-84)
// Residency: 64-wide 4 CTAs/SM, 128-wide 2, 256-wide 1 (TMEM), so the 256-wide kernels get
// the registers of a whole SM (the 1-term normal tiles use ~160: config 4 1.54 -> 1.51 ms).
// MMA layer m = 0 is layer 0 (K = 32, B0 resident), m = 1..L-2 the hidden layers; the
// last hidden layer's epilogue folds in the 1 x W output layer.
template <int W, bool kGrad, int kGroups, int kTerms, bool kResident, bool kPersist, int kHid, bool kF8On>
__global__ void __launch_bounds__(32 * (kResident ? 1 : 2) + 128 * kGroups,
                                  (W == 64 ? 4 : (W == 256 ? 1 : 2))) tc_mlp_kernel(TcArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  constexpr int kCtl = kResident ? 1 : 2;  // control warps: MMA issuer [+ weight producer]
  constexpr int kThreads = 32 * kCtl + 128 * kGroups;
  const TcNet& net = a.net;
  const int L = net.n_layers;
  const TcSmem sm = tc_carve(smem_raw, W, L, kTerms, kResident, kPersist);
  constexpr int kNW = kTerms == 3 ? 2 : 1;  // weight parts (hi [, lo])
  uint64_t* full = sm.bars;
  constexpr int kStages = tc_stages(W);
  uint64_t* empty = sm.bars + kMaxStages;
  uint64_t* kready = sm.bars + 2 * kMaxStages;  // [kSub]: A block row i written by every group
  uint64_t* a0ready = sm.bars + 2 * kMaxStages + kMaxSub;
  uint64_t* tstart = sm.bars + 2 * kMaxStages + kMaxSub + 1;
  uint64_t* dfull = sm.bars + 2 * kMaxStages + kMaxSub + 2;  // [kNH]: N-block nb of a layer complete
  float* part = sm.part;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // hidden (W x W) MMA layers: compile-time for the standard architectures (kHid > 0), so
  // the layer loops unroll and every per-layer constant folds
  const int n_hidden = kHid > 0 ? kHid : L - 2;
  constexpr int kRaysPerTile = kGrad ? kRows / 4 : kRows;
  // tc_split8 nets (mlp_tc.cuh): hidden weights scaled by 2^s; forward 3-term tiles of nets
  // whose upload chose it (kF8On: DevNet::tc_f8_mask) run the correction terms as one E4M3
  // MMA per K step (compile-time: a runtime per-layer choice cost the 256-wide level 30%)
  constexpr bool kScaled = tc_split8(W);
  constexpr bool kF8 = kF8On && kScaled && !kGrad && kTerms == 3;
  constexpr int kParts = tc_parts(W);
  // N-blocks: every MMA layer is issued as kNH column blocks of kNB outputs, each with its
  // own completion barrier (dfull[nb]), so the epilogue of block 0 (and with it the next
  // layer's first K rows) runs under the MMAs of block 1 and the tensor pipe goes straight
  // on into the next layer.  Weights stream as (N-block, K chunk) pieces of kNB x kKCh.
  constexpr int kNH = tc_halves(W);
  constexpr int kNB = W / kNH;
  constexpr int kKCh = kKC * kNH;           // K per streamed chunk (same bytes per stage)
  constexpr int kChunks = W / kKCh;         // chunks per N-block
  constexpr int kStepsPerChunk = kKCh / kBlk;
  constexpr uint32_t kChunkBytes = uint32_t(kNB) * kKCh * 2;
  constexpr size_t kStageHalves = size_t(kNB) * kKCh * kNW;
  // K streaming: block b of a layer's output belongs to group b % kGroups, so the groups
  // together produce the next layer's A operand in natural K order, block row i = blocks
  // [i*kGroups, (i+1)*kGroups), and the MMA of layer m+1 starts on block row 0 while the
  // epilogue still works on layer m.  Accumulators alternate between two TMEM regions
  // (layer m in columns (m & 1) * W).
  constexpr int kSub = W / kBlk / kGroups;
  constexpr int kSubNB = kSub / kNH;  // blocks per group per N-block
  static_assert(kSub <= kMaxSub, "kready barriers");
  static_assert(kSub % kNH == 0 && kChunkBytes * kNW == size_t(W) * kKC * 2 * kNW, "N-block split");
  constexpr uint32_t kTmemCols = 2 * W;
  // The hidden layers' A operand lives in TMEM, written IN PLACE over the accumulator
  // it is computed from: the epilogue reads D block b (16 fp32 columns of its lane), and
  // stores the block's activations back into the same 16 columns as 8 columns of packed
  // fp16 hi parts + 8 of lo parts, which is exactly K-block b of the next layer's A.  The
  // next layer accumulates into the other region, so K streaming is unchanged and no SMEM
  // holds A (no STS, no SMEM operand reads for A).

  const int n_items = (a.op == kOpEval || a.op == kOpNormalMap) ? a.k : *a.in_count;
  int my_tiles, claim = 1;
  if (kPersist) {
    // claim granularity: up to 32 list items per warp claim, fewer for short lists so the
    // items spread over the CTAs
    // A short list (a small tile share of a frame, the fine levels' hand-offs) runs on fewer
    // CTAs, each with at least min_items rays: the rows of a CTA stay full instead of
    // idling through the level's tail, and the SMs of the CTAs that exit at once take the
    // next frame's kernels (frames in flight).  The count is the level's real input size,
    // known here (stream order) though not at launch.
    const int active = max(1, min(int(gridDim.x), (n_items + a.min_items - 1) / max(a.min_items, 1)));
    const int div = active * a.claim_div;
    claim = max(1, min(32, (n_items + div - 1) / div));
    if (n_items == 0 || int(blockIdx.x) >= active || int(blockIdx.x) * 4 * claim >= n_items) return;
    my_tiles = 0x7fffffff;
  } else {
    const int n_tiles = (n_items + kRaysPerTile - 1) / kRaysPerTile;
    my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (my_tiles == 0) return;
  }

  // ---- setup: B0, biases, barriers, TMEM ----
  for (int i = threadIdx.x; i < W * kK0; i += kThreads) {
    const int n = i / kK0, k = i % kK0;
    const float* w = net.w0 + n * net.input_dim;
    __half v = __float2half_rn(0.0f);
    if (k < 9 || (k >= 10 && k < 16)) {
      const float x = net.omega * w[(k < 9 ? k : k - 10) % 3];  // radians
      const __half hi = __float2half_rn(x);
      v = k < 9 ? hi : __float2half_rn(x - __half2float(hi));
    } else if (k == 9 || k == 16 || k == 17) {
      // a 4-input net's time column joins the bias (the slice time, field.cpp:213-220)
      float b0 = net.b[n];
      if (net.input_dim == 4) b0 = fmaf(w[3], a.time, b0);
      __half hi, mid, lo;
      split3(net.omega * b0, hi, mid, lo);
      v = k == 9 ? hi : (k == 16 ? mid : lo);
    }
    sm.b0[b0_off(W, n, k)] = v;
  }
  // Hidden-layer biases on the tensor cores: one extra K = 16 MMA per layer, A = a constant
  // block with ones at k = 0..2 (value rows only: tangent chains carry no bias), B = the
  // three fp16 parts of omega*b.  With omega folded into the hidden weights (upload), every
  // accumulator is the sine argument in radians: the epilogue has no FFMA and no bias loads.
  for (int i = threadIdx.x; i < (L - 2) * W * kBlk; i += kThreads) {
    const int h = i / (W * kBlk), n = (i / kBlk) % W, k = i % kBlk;
    __half v = __float2half_rn(0.0f);
    if (k < 3) {
      __half hi, mid, lo;
      split3(net.b[(h + 1) * W + n] * net.omega * (kScaled ? net.scale : 1.0f), hi, mid, lo);
      v = k == 0 ? hi : (k == 1 ? mid : lo);
    }
    sm.bb[size_t(h) * W * kBlk + b0_off(W, n, k)] = v;
  }
  for (int i = threadIdx.x; i < kRows * kBlk; i += kThreads) {
    const int r = i / kBlk, k = i % kBlk;
    const bool one = k < 3 && (!kGrad || (r & 3) == 0);
    sm.ones[a_off(r, 0) + (k >> 3) * (kRows / 8) * 64 + (k & 7)] = __float2half_rn(one ? 1.0f : 0.0f);
  }
  for (int i = threadIdx.x; i < W; i += kThreads) sm.wout[i] = net.wout[i];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    // one arrival per epilogue warp (after a __syncwarp behind each thread's fence)
    for (int i = 0; i < kSub; ++i) mbar_init(&kready[i], 4 * kGroups);
    mbar_init(a0ready, 4 * kGroups);
    for (int nb = 0; nb < kNH; ++nb) mbar_init(&dfull[nb], 1);
    mbar_init(tstart, 1);
    *sm.stage_count = 0;
    *sm.done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(sm.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async();  // B0 (generic-proxy writes) -> tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sm.tmem_base;
  if (kTimeline && a.dbg && threadIdx.x == 0 && blockIdx.x < kDbgMaxCta) {
    a.dbg[kDbgCta + 5 * blockIdx.x] = global_ns();
    a.dbg[kDbgCta + 5 * blockIdx.x + 3] = clock64();
  }

  // Control warps' tile loop: a fixed tile count, or (persistent) one tstart phase per tile
  // published by the epilogue, with the done flag ending the loop.
  uint32_t ts_phase = 0;
  auto more_tiles = [&](int t) -> bool {
    if (!kPersist) return t < my_tiles;
    mbar_wait(tstart, ts_phase);
    ts_phase ^= 1;
    return *reinterpret_cast<volatile int*>(sm.done) == 0;
  };

  if (warp == 0) {
    // ================= MMA issuer (resident mode: also loads the weights once) =================
    // the whole warp runs this loop; MMAs and commits are issued by one elected lane
    {
      const uint32_t idesc = umma_idesc(kNB);
      const uint32_t b0_base = smem_addr(sm.b0);
      const uint64_t ones_desc = umma_desc(smem_addr(sm.ones), kRows * 16, 128);
      if (kResident) {
        const uint32_t bytes = uint32_t(n_hidden) * W * W * 2 * kParts;
        if (lane == 0) {
          mbar_expect_tx(&full[0], bytes);
          bulk_g2s(sm.wst, net.wq, bytes, &full[0]);
        }
        mbar_wait(&full[0], 0);
        __syncwarp();
      }
      uint32_t chunk_iter = 0, kr_phase = 0, a0_phase = 0;
      // debug timeline (NSDF_TC_TIMELINE): cycles the issuer waits for A0, A blocks, weights
      const bool mdbg = kTimeline && a.dbg && blockIdx.x == 0 && lane == 0;
      long long w_a0 = 0, w_k = 0, w_full = 0, t_loop = 0;
      auto timed_wait = [&](uint64_t* bar, uint32_t ph, long long& acc) {
        const long long c0 = mdbg ? clock64() : 0;
        mbar_wait(bar, ph);
        if (mdbg) acc += clock64() - c0;
      };
      for (int t = 0; more_tiles(t); ++t) {
        const long long tl0 = mdbg ? clock64() : 0;
        // ---- layer 0: D0 = A0 . B0^T, K = 32 (the split lives in K: one term) ----
        timed_wait(a0ready, a0_phase, w_a0);
        a0_phase ^= 1;
        tc_fence_after();
#pragma unroll
        for (int nb = 0; nb < kNH; ++nb) {
#pragma unroll
          for (int ks = 0; ks < kK0 / 16; ++ks) {
            const uint64_t bd = umma_desc(b0_base + uint32_t(ks * 2) * (W / 8) * 128 + uint32_t(nb * kNB * 16), W * 16, 128);
            tc_mma_ts(tmem + uint32_t(nb * kNB), tmem + uint32_t(W + ks * 8), bd, idesc, ks != 0);
          }
          tc_commit(&dfull[nb]);
        }
        // ---- hidden layers, K-streamed behind the epilogue, N-block by N-block ----
        for (int h = 0; h < n_hidden; ++h) {
          const uint32_t d_tmem = tmem + uint32_t((h + 1) & 1) * W;
          const uint32_t a_tmem = tmem + uint32_t(h & 1) * W;  // A in place of layer h's D
#pragma unroll
          for (int nb = 0; nb < kNH; ++nb) {
            const uint32_t dn = d_tmem + uint32_t(nb * kNB);
            // D = omega*b (value rows) first: it reads no A, and this region's last readers
            // (the previous layer's MMAs) precede it in the tensor pipe's issue order
            tc_mma(dn, ones_desc, umma_desc(smem_addr(sm.bb + size_t(h) * W * kBlk) + uint32_t(nb * kNB * 16), W * 16, 128),
                   idesc, false);
            uint32_t b_base = 0, lo_off = 0;
            int s = 0;
#pragma unroll
            for (int blk = 0; blk < W / kBlk; ++blk) {
              if (nb == 0 && blk % kGroups == 0) {  // block row of the A operand written by every group
                timed_wait(&kready[blk / kGroups], kr_phase, w_k);
                tc_fence_after();
              }
              const int c = blk / kStepsPerChunk, ks = blk % kStepsPerChunk;  // weight chunk, K=16 step in it
              if (ks == 0) {
                s = chunk_iter % kStages;
                if (kResident) {
                  // resident layout per layer: [hi W*W][lo W*W] (tc_wq_offset)
                  b_base = smem_addr(sm.wst + size_t(h) * kParts * W * W + size_t(nb) * kNB * W + size_t(c) * kNB * kKCh);
                  lo_off = uint32_t(kF8 ? 2 : 1) * W * W * 2;
                } else {
                  timed_wait(&full[s], (chunk_iter / kStages) & 1, w_full);
                  tc_fence_after();
                  b_base = smem_addr(sm.wst + size_t(s) * kStageHalves);
                  lo_off = kChunkBytes;
                }
              }
              const uint32_t boff = uint32_t(ks * 2) * (kNB / 8) * 128;
              const uint64_t bd = umma_desc(b_base + boff, kNB * 16, 128);
              const uint32_t at = a_tmem + uint32_t(blk * kBlk);  // hi parts; lo parts 8 columns on
              tc_mma_ts(dn, at, bd, idesc, true);
              if (kTerms == 3) {  // split precision: + A_lo.W_hi + A_hi.W_lo
                const uint64_t bdl = umma_desc(b_base + lo_off + boff, kNB * 16, 128);
                if (kF8) {
                  tc_mma_ts_f8(dn, at + 8, bdl, idesc);  // [fp8 A | fp8 A_lo 2^s] . [fp8 W_lo ; fp8 W_hi 2^-s]
                } else {
                  tc_mma_ts(dn, at + 8, bd, idesc, 1);
                  tc_mma_ts(dn, at, bdl, idesc, 1);
                }
              }
              if (ks == kStepsPerChunk - 1) {
                if (!kResident) tc_commit(&empty[s]);  // frees the weight stage once these MMAs retire
                ++chunk_iter;
              }
            }
            tc_commit(&dfull[nb]);  // N-block nb of the accumulator complete
          }
          kr_phase ^= 1;
        }
        if (mdbg && t >= a.dbg_skip && t - a.dbg_skip < 64) {
          t_loop = clock64() - tl0;
          a.dbg[65 * 16 + (t - a.dbg_skip) * 4 + 0] = w_a0;
          a.dbg[65 * 16 + (t - a.dbg_skip) * 4 + 1] = w_k;
          a.dbg[65 * 16 + (t - a.dbg_skip) * 4 + 2] = w_full;
          a.dbg[65 * 16 + (t - a.dbg_skip) * 4 + 3] = t_loop;
          w_a0 = w_k = w_full = 0;
        }
      }
    }
  } else if (!kResident && warp == 1) {
    // ================= weight producer =================
    if (lane == 0) {
      uint32_t chunk_iter = 0;
      for (int t = 0; more_tiles(t); ++t) {
        for (int h = 0; h < n_hidden; ++h) {
          const __half* lw = reinterpret_cast<const __half*>(net.wq) + size_t(h) * kParts * W * W;
          for (int nb = 0; nb < kNH; ++nb)
            for (int c = 0; c < kChunks; ++c, ++chunk_iter) {
              const int s = chunk_iter % kStages;
              const size_t piece = size_t(nb) * kNB * W + size_t(c) * kNB * kKCh;  // (N-block, chunk)
              mbar_wait(&empty[s], ((chunk_iter / kStages) & 1) ^ 1);
              mbar_expect_tx(&full[s], kChunkBytes * kNW);
              bulk_g2s(sm.wst + size_t(s) * kStageHalves, lw + piece, kChunkBytes, &full[s]);
              if (kTerms == 3)
                bulk_g2s(sm.wst + size_t(s) * kStageHalves + size_t(kNB) * kKCh, lw + size_t(kF8 ? 2 : 1) * W * W + piece, kChunkBytes,
                         &full[s]);
            }
        }
      }
    }
  } else {
    // ================= epilogue warps =================
    const int ew = warp - kCtl;                          // epilogue warp index
    const int eg = ew >> 2;                              // column group
    const int q = warp & 3;                              // TMEM lane quadrant of this warp
    const int row = q * 32 + lane;                       // TMEM lane = A row
    const int ctid = (ew & 3) * 32 + lane;               // consumer thread id within group 0
    const uint32_t taddr = tmem + (uint32_t(q * 32) << 16);
    const int ray = kGrad ? row >> 2 : row;             // ray within the tile
    const int chain = kGrad ? row & 3 : 0;               // 0 = value, 1..3 = d/dx, d/dy, d/dz
    const unsigned group_mask = 0xFu << (lane & ~3);
    uint32_t dfull_phase = 0;

    // One tile through the net from each row's point p (group 0 rows; `live` = the row
    // carries a point): A0 -> layer 0 and the hidden layers on the tensor cores, sine
    // epilogues here -> output dot.  Returns the output pre-bias in group 0 (the other
    // groups' partials are combined through SMEM).
    int dbg_t = 0;
    auto mark = [&](int k) {
      if (kTimeline && a.dbg && blockIdx.x == 0 && ew == 0 && lane == 0 && k == 0 && dbg_t < kDbgMaxTiles)
        a.dbg[kDbgTileT + dbg_t] = clock64();
      if (kTimeline && a.dbg && blockIdx.x == 0 && ew == 0 && lane == 0 && dbg_t >= a.dbg_skip &&
          dbg_t - a.dbg_skip < 64)
        a.dbg[(dbg_t - a.dbg_skip) * 16 + k] = clock64();
    };
    // gap0 / gap1: work for the warp's idle waits on the tensor core — gap0 runs after A0 is
    // handed to the MMA issuer (the layer-0 round trip), gap1 before the last layer's
    // accumulator wait (its MMA tail); the persistent trace runs its ray prefetch there.
    auto eval_tile = [&](const float* p, bool live, auto&& gap0, auto&& gap1) -> float {
      mark(0);
      if (eg == 0) {
        // ---- A0: the point in three fp16 parts (value rows) or a unit tangent ----
        // 32-bit words = K pairs (k, k+1); layout in the kK0 comment above
        auto pk2 = [](__half lo16, __half hi16) {
          return uint32_t(__half_as_ushort(lo16)) | (uint32_t(__half_as_ushort(hi16)) << 16);
        };
        const __half one = __float2half_rn(1.0f), zero = __float2half_rn(0.0f);
        uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0, w4 = 0, w8 = 0;
        if (live) {
          if (!kGrad || chain == 0) {
            __half h0, m0, l0, h1, m1, l1, h2, m2, l2;
            split3(p[0], h0, m0, l0);
            split3(p[1], h1, m1, l1);
            split3(p[2], h2, m2, l2);
            w0 = pk2(h0, h1);
            w1 = pk2(h2, m0);
            w2 = pk2(m1, m2);
            w3 = pk2(l0, l1);
            w4 = pk2(l2, one);
            w8 = pk2(one, one);
          } else {
            w0 = chain == 1 ? pk2(one, zero) : (chain == 2 ? pk2(zero, one) : 0u);
            w1 = chain == 3 ? pk2(one, zero) : 0u;
          }
        }
        // A0 in TMEM, columns 0-15 of region 1 (K pairs packed per column, 8 columns per
        // K = 16 step): region 1 is free here — it held the last layer's accumulator (read by
        // this thread's own earlier loads; the other groups never read block 0) or, for an
        // even hidden-layer count, an A operand whose MMAs have completed
        tmem_st8(taddr + uint32_t(W), w0, w1, w2, w3, w4, w0, w1, w2);
        tmem_st8(taddr + uint32_t(W) + 8u, w8, 0u, 0u, 0u, 0u, 0u, 0u, 0u);
        tmem_wait_st();
        mark(10);
      }
      // every epilogue thread: done with the previous tile's TMEM (region 0 is reused)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a0ready);
      mark(1);
      gap0();
      float2 acc2 = make_float2(0.0f, 0.0f);
      // one MMA layer's epilogue; the last one (compile-time) folds in the output dot
      auto layer = [&](int m, auto last_tag) {
        constexpr bool last = decltype(last_tag)::value;
        if constexpr (last) gap1();
        // D is the sine argument in radians (omega and the bias are inside the MMAs)
        const uint32_t treg = taddr + uint32_t(m & 1) * W;
        // sine epilogue of one 16-column block (value rows; tangent rows scale by omega cos)
        auto activate = [&](const uint32_t (&r)[16], int cc, float (&v)[16]) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
          if (kScaled && m > 0) {  // accumulators of scaled weights hold 2^s x the argument
            const float2 is = make_float2(net.inv_scale, net.inv_scale);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float2 t = __fmul2_rn(make_float2(v[2 * j], v[2 * j + 1]), is);
              v[2 * j] = t.x;
              v[2 * j + 1] = t.y;
            }
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (kGrad) {
              // the value row's pre-activation, broadcast to its 3 tangent rows; every lane
              // issues ONE sine: sin(z) on the value row, cos(z) = sin(z + pi/2) on tangents
              const float z = __shfl_sync(group_mask, v[j], lane & ~3, 32);
              const float r1 = fast_sin(chain == 0 ? z : z + kHalfPi);
              // tangent rows: G = (W.G_prev) * omega cos(z); D = omega (W.G_prev)
              v[j] = chain == 0 ? r1 : v[j] * r1;
            } else {
              v[j] = fast_sin(v[j]);
            }
          }
        };
        // TMEM loads software-pipelined one block ahead of the math, within an N-block
        uint32_t raw[2][16];
#pragma unroll
        for (int i = 0; i < kSub; ++i) {
          const int buf = i & 1;
          const int cc = (i * kGroups + eg) * kBlk;
          if (i % kSubNB == 0) {  // first block of N-block i / kSubNB: wait for its MMAs
            mbar_wait(&dfull[i / kSubNB], dfull_phase);
            if (i == 0) mark(2 + 2 * min(m, 3));
            tc_fence_after();
            tmem_issue16(treg + uint32_t(cc), raw[buf]);
          }
          tmem_wait16(raw[buf]);
          if (i + 1 < kSub && (i + 1) % kSubNB != 0) tmem_issue16(treg + uint32_t(cc + kGroups * kBlk), raw[buf ^ 1]);
          float v[16];
          activate(raw[buf], cc, v);
          if constexpr (!last) {
            // in place: A block i of the next layer over the D columns just read; the MMA may
            // start on block row i while this thread continues with block i + 1 (waiting
            // for the stores one block later, to overlap their latency, was measured slower:
            // the MMA start matters more)
            uint32_t hw[8], lw[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) hw[j] = pack_half2(v[2 * j], v[2 * j + 1]);
            if (kF8) {
              // columns 8-11: fp8(A), 12-15: fp8((A - fp16(A)) * 2^s) (one f8f6f4 K = 32 step)
              float lo[16];
              const float2 sc = make_float2(net.scale, net.scale);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const __half2 h = *reinterpret_cast<const __half2*>(&hw[j]);
                const float2 d = __ffma2_rn(__half22float2(h), make_float2(-1.0f, -1.0f), make_float2(v[2 * j], v[2 * j + 1]));
                const float2 ds = __fmul2_rn(d, sc);  // exact (power of 2)
                lo[2 * j] = ds.x;
                lo[2 * j + 1] = ds.y;
              }
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                lw[q] = pack_e4m3x4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                lw[4 + q] = pack_e4m3x4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
              }
            } else if (kTerms == 3) {
#pragma unroll
              for (int j = 0; j < 8; ++j) lw[j] = pack_half2_lo(v[2 * j], v[2 * j + 1], hw[j]);
            }
            tmem_st8(treg + uint32_t(cc), hw[0], hw[1], hw[2], hw[3], hw[4], hw[5], hw[6], hw[7]);
            if (kTerms == 3)
              tmem_st8(treg + uint32_t(cc + 8), lw[0], lw[1], lw[2], lw[3], lw[4], lw[5], lw[6], lw[7]);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&kready[i]);
          } else {
            // the 1 x W output layer as packed FFMA2s (two partial sums per thread)
            const float2* wo = reinterpret_cast<const float2*>(sm.wout + cc);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc2 = __ffma2_rn(wo[j], make_float2(v[2 * j], v[2 * j + 1]), acc2);
          }
        }
        dfull_phase ^= 1;
        mark(3 + 2 * min(m, 3));
      };
#pragma unroll
      for (int m = 0; m < n_hidden; ++m) layer(m, std::false_type{});
      layer(n_hidden, std::true_type{});
      float acc_out = acc2.x + acc2.y;
      ++dbg_t;
      // ---- combine the column groups' partial output dots ----
      if (kGroups > 1) {
        if (eg > 0) part[(eg - 1) * kRows + row] = acc_out;
        named_bar(1, 128 * kGroups);
        if (eg == 0)
          for (int g = 1; g < kGroups; ++g) acc_out += part[(g - 1) * kRows + row];
      }
      return acc_out;
    };

    if constexpr (kPersist) {
      // ============ persistent level trace (sphere_trace_level, trace.cpp:61-84) ============
      const bool g0 = eg == 0;
      const RayState& st = a.st;
      const StageList st_adv{sm.stage_buf, sm.stage_count};
      const uint32_t lt = (1u << lane) - 1u;
      int slot = -1, it = 0, evals = 0, n_tiles = 0;
      float px = 0.f, py = 0.f, pz = 0.f, t = 0.f, dx = 0.f, dy = 0.f, dz = 0.f;
      int pf_slot = -1, pf_stage = kPfNeed, fit = 0;  // fit: prefetched iteration count (resume)
      float fpx = 0.f, fpy = 0.f, fpz = 0.f, fpt = 0.f, fdx = 0.f, fdy = 0.f, fdz = 0.f;
      int res_base = 0, res_end = 0, nres = 0;  // claimed list range; next claim ticket (lane 0)
      bool exhausted = false;
      if (g0 && lane == 0) nres = fetch_ticket(a.cursor);
      // the ray pipeline (group 0 only): assign = READY prefetches -> empty rows, right after
      // the trace update; the other two stages advance in the tile's tensor-core waits
      auto assign = [&]() {
        // READY prefetches -> empty rows (the k-th empty row takes the k-th ready lane)
        const uint32_t emp = __ballot_sync(0xffffffffu, slot < 0);
        const uint32_t rdy = __ballot_sync(0xffffffffu, pf_stage == kPfReady);
        if (emp && (emp & ~rdy) == 0) {
          // common case: every empty row's own prefetch is ready (no shuffles)
          if (slot < 0) {
            slot = pf_slot;
            it = fit;
            px = fpx, py = fpy, pz = fpz, t = fpt, dx = fdx, dy = fdy, dz = fdz;
            st.level_reached[slot] = a.lv.level;
            pf_stage = kPfNeed;
          }
        } else if (emp && rdy) {
          const int k = min(__popc(emp), __popc(rdy));
          const int r = __popc(emp & lt);
          const bool take = slot < 0 && r < k;
          const int src = take ? nth_set_bit(rdy, r) : lane;
          const int s_slot = __shfl_sync(0xffffffffu, pf_slot, src);
          const int s_it = __shfl_sync(0xffffffffu, fit, src);
          const float s_px = __shfl_sync(0xffffffffu, fpx, src), s_py = __shfl_sync(0xffffffffu, fpy, src),
                      s_pz = __shfl_sync(0xffffffffu, fpz, src), s_t = __shfl_sync(0xffffffffu, fpt, src),
                      s_dx = __shfl_sync(0xffffffffu, fdx, src), s_dy = __shfl_sync(0xffffffffu, fdy, src),
                      s_dz = __shfl_sync(0xffffffffu, fdz, src);
          if (take) {
            slot = s_slot;
            it = s_it;
            px = s_px, py = s_py, pz = s_pz, t = s_t, dx = s_dx, dy = s_dy, dz = s_dz;
            st.level_reached[slot] = a.lv.level;
          }
          if (pf_stage == kPfReady && __popc(rdy & lt) < k) pf_stage = kPfNeed;
        }
        if (W == 64) mark(8);  // (64-wide: layer marks 6-9 are free) refill sub-steps
      };
      // LISTED -> READY: the slot arrived last tile; issue the ray-state loads
      auto to_ready = [&]() {
        if (pf_stage == kPfListed) {
          fpx = __ldg(st.px + pf_slot);
          fpy = __ldg(st.py + pf_slot);
          fpz = __ldg(st.pz + pf_slot);
          fpt = __ldg(st.t + pf_slot);
          fdx = __ldg(st.dx + pf_slot);
          fdy = __ldg(st.dy + pf_slot);
          fdz = __ldg(st.dz + pf_slot);
          fit = a.resume ? int(st.iters[size_t(pf_slot) * kMaxLevels + a.lv.level]) : 0;
          pf_stage = kPfReady;
        }
        if (W == 64) mark(9);
      };
      // NEED -> LISTED: claim list items (warp claims of `claim` items, one claim ahead)
      auto claim_items = [&]() {
        uint32_t need = __ballot_sync(0xffffffffu, pf_stage == kPfNeed);
        while (need && !exhausted) {
          if (res_base == res_end) {
            res_base = __shfl_sync(0xffffffffu, nres, 0) * claim;
            if (res_base >= n_items) {
              exhausted = true;
              break;
            }
            res_end = min(res_base + claim, n_items);
            if (lane == 0) nres = fetch_ticket(a.cursor);
          }
          const int k = min(__popc(need), res_end - res_base);
          const int r = __popc(need & lt);
          if (((need >> lane) & 1u) && r < k && in_bounds(res_base + r, n_items, kChkListRead)) {
            pf_slot = __ldg(a.in_list + res_base + r);
            if (in_bounds(pf_slot, st.cap, kChkSlot)) pf_stage = kPfListed;
          }
          res_base += k;
          need = __ballot_sync(0xffffffffu, pf_stage == kPfNeed);
        }
      };
      bool pend_conv = false;
      int pend_slot = -1;
      auto append_pending = [&]() {
        stage_append(pend_conv, pend_slot, st_adv);
        pend_conv = false;
      };
      auto advance = [&]() {
        to_ready();
        claim_items();
      };
      if (g0)
        for (int i = 0; i < 3; ++i) {  // prime: rows filled, prefetches claimed
          assign();
          advance();
        }
      for (bool first = true;; first = false) {
        if (g0 && !first) assign();
        mark(14);
        // one barrier per tile: the live-row vote also orders every warp's staged appends of
        // the previous tile before the flush decision below
        const bool live = bar_vote_any(3, 128 * kGroups, g0 && slot >= 0);
        if (g0 && *sm.stage_count > kStageCap - kRows) stage_flush_now(st_adv, a.adv_list, a.adv_count, sm.stage_base, ctid, st.cap);
        if (!live) {
          // no live row: either prefetches are still in flight (refill again) or done
          if (g0) append_pending();
          if (bar_vote_any(3, 128 * kGroups, g0 && pf_stage != kPfNeed)) {
            if (g0) advance();
            continue;
          }
          break;
        }
        mark(15);
        if (ew == 0 && lane == 0) {
          mbar_arrive(tstart);  // control warps: one more tile
          ++n_tiles;
        }
        const float p[3] = {px, py, pz};
        const float acc = eval_tile(
            p, slot >= 0,
            [&] {
              if (g0) {
                append_pending();
                to_ready();
              }
            },
            [&] { if (g0) claim_items(); });
        mark(11);
        if (g0) {
          const int s0 = slot;
          bool conv = false, parked = false;
          if (slot >= 0) {
            // trace update (trace.cpp:61-84; same arithmetic as trace_update, device_ops.cuh)
            ++evals;
            const float f = acc + net.bout;
            const float fd = __fsub_rn(f, a.lv.delta);
            const float afd = fabsf(fd);
            conv = a.lv.final_level ? afd <= a.eps : fd <= a.eps;
            bool cont = false;
            bool park = false;
            if constexpr (kF8) park = a.refine_list && fabsf(afd - a.eps) <= kRefineBand;
            parked = park;
            if (park) {
              // defer the decision: the state as it was before this evaluation, for the resume
              st.px[slot] = px;
              st.py[slot] = py;
              st.pz[slot] = pz;
              st.t[slot] = t;
              st.iters[size_t(slot) * kMaxLevels + a.lv.level] = uint16_t(it);
              --evals;
              conv = false;
            } else if (!conv) {
              float step = fd;
              if (a.lv.final_level && step < 0.0f) step = 0.0f;  // trace.cpp:73
              px = __fadd_rn(px, __fmul_rn(step, dx));
              py = __fadd_rn(py, __fmul_rn(step, dy));
              pz = __fadd_rn(pz, __fmul_rn(step, dz));
              t = __fadd_rn(t, step);
              cont = !(t > a.t_max);  // trace.cpp:78
            }
            if (!park) ++it;
            if (park) {
              slot = -1;
            } else if (!cont || it == a.lv.budget) {  // the ray leaves the level: write its state once
              st.px[slot] = px;
              st.py[slot] = py;
              st.pz[slot] = pz;
              st.t[slot] = t;
              st.iters[size_t(slot) * kMaxLevels + a.lv.level] = uint16_t(it);
              st.final_dist[slot] = afd;
              slot = -1;
            }
          }
          if constexpr (kF8) {
            // parked rays -> refine list (rare: one aggregated atomic per warp that has any)
            if (a.refine_list) {
              const unsigned pm = __ballot_sync(0xffffffffu, parked);
              if (pm) {
                const int leader = __ffs(pm) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(a.refine_count, __popc(pm));
                base = __shfl_sync(0xffffffffu, base, leader);
                const int at = base + __popc(pm & lt);
                if (parked && in_bounds(at, st.cap, kChkListWrite)) a.refine_list[at] = s0;
              }
            }
          }
          mark(12);
          // the compaction append runs in the next tile's first tensor-core wait (off the
          // update -> next point chain); the vote before every flush decision orders it
          pend_conv = conv;
          pend_slot = s0;
          mark(13);
        }
      }
      if (ew == 0 && lane == 0) {
        *reinterpret_cast<volatile int*>(sm.done) = 1;
        mbar_arrive(tstart);
        if (kTimeline && a.dbg) {
          atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg + kDbgTiles), (unsigned long long)n_tiles);
          if (blockIdx.x < kDbgMaxCta) a.dbg[kDbgCta + 5 * blockIdx.x + 2] = n_tiles;
        }
      }
      if (g0) {
        stage_flush(st_adv, a.adv_list, a.adv_count, sm.stage_base, ctid, true, st.cap);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
        if (lane == 0 && evals) atomicAdd(a.evals, evals);
      }
    } else {
      // ============ fixed tiles: normals / batch eval / normal map ============
      auto item_of = [&](int t) { return (blockIdx.x + t * gridDim.x) * kRaysPerTile + ray; };
      RowIn now = eg == 0 ? load_row(a, load_slot(a, item_of(0), n_items)) : RowIn{-1};
      int slot_next = my_tiles > 1 && eg == 0 ? load_slot(a, item_of(1), n_items) : -1;
      for (int t = 0; t < my_tiles; ++t) {
        const int item = item_of(t);
        const bool valid = item < n_items;
        // prefetch: point of tile t+1 (slot known), list slot of tile t+2
        const RowIn next = t + 1 < my_tiles && eg == 0 ? load_row(a, slot_next) : RowIn{-1};
        slot_next = t + 2 < my_tiles && eg == 0 ? load_slot(a, item_of(t + 2), n_items) : -1;
        const float acc_out = eval_tile(now.p, valid, [] {}, [] {});
        if (eg == 0) {
          // ---- consumer (group 0) ----
          const float fval = (!kGrad || chain == 0) ? acc_out + net.bout : acc_out;
          if (kGrad) {
            const int base = lane & ~3;
            const float gx = __shfl_sync(0xffffffffu, fval, base + 1);
            const float gy = __shfl_sync(0xffffffffu, fval, base + 2);
            const float gz = __shfl_sync(0xffffffffu, fval, base + 3);
            const float f = __shfl_sync(0xffffffffu, fval, base);
            bool defer = false;
            const bool lead = chain == 0 && valid;
            if (a.op == kOpNormals) {
              if (lead) {
                float nrm[3];
                if (!normalize_normal(gx, gy, gz, nrm)) {
                  nrm[0] = 0.0f;
                  nrm[1] = 1.0f;
                  nrm[2] = 0.0f;
                  defer = a.defer_fallback != 0;
                }
                if (!defer) shade_and_write(a.sp, a.st, now.slot, nrm, a.rgb, a.depth, a.mask);
              }
              warp_append(defer, now.slot, a.fb_list, a.fb_count, a.st.cap);
            } else if (a.op == kOpNormalMap) {
              bool outside = false, fell_back = false;
              if (lead) {
                outside = fabs(double(f)) > a.delta;
                float nrm[3];
                if (!normalize_normal(gx, gy, gz, nrm)) {
                  fell_back = true;
                  for (int c = 0; c < 3; ++c)
                    nrm[c] = a.fallback ? a.fallback[size_t(c) * a.k + item] : (c == 1 ? 1.0f : 0.0f);
                }
                for (int c = 0; c < 3; ++c) a.grad[size_t(c) * a.k + item] = nrm[c];
              }
              const unsigned mo = __ballot_sync(0xffffffffu, outside), mf = __ballot_sync(0xffffffffu, fell_back);
              if (lane == 0 && (mo | mf)) {
                atomicAdd(a.counts + 0, (unsigned long long)__popc(mo));
                atomicAdd(a.counts + 1, (unsigned long long)__popc(mf));
              }
            } else if (lead) {
              if (a.out) a.out[item] = f;
              if (a.grad) {
                a.grad[item] = gx;
                a.grad[size_t(a.k) + item] = gy;
                a.grad[size_t(2) * a.k + item] = gz;
              }
            }
          } else if (valid) {
            a.out[item] = fval;
          }
        }
        now = next;
      }
    }
  }
  // ---- teardown ----
  if (kTimeline && a.dbg && threadIdx.x == 0 && blockIdx.x < kDbgMaxCta) {
    a.dbg[kDbgCta + 5 * blockIdx.x + 1] = global_ns();
    a.dbg[kDbgCta + 5 * blockIdx.x + 4] = clock64();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

thread_local cudaError_t g_tc_error = cudaSuccess;

TcLaunch tc_failed(cudaError_t e) {
  g_tc_error = e == cudaSuccess ? cudaErrorLaunchFailure : e;
  return TcLaunch::kFailed;
}

template <int W, bool kGrad, int kTerms, bool kResident, bool kPersist, int kHid, bool kF8On>
TcLaunch launch_w(TcArgs& a, int n_max_items, cudaStream_t s) {
  // column groups: 256-wide 4 (16 epilogue warps; the 1-term normal tiles too: 24.2k -> 21.6k
  // cycles per tile, their epilogue being the tile's critical path), 128-wide 2, 64-wide 1
  constexpr int kGroups = W == 64 ? 1 : (W == 256 ? 4 : 2);
  constexpr int kThreads = 32 * (kResident ? 1 : 2) + 128 * kGroups;
  auto kernel = tc_mlp_kernel<W, kGrad, kGroups, kTerms, kResident, kPersist, kHid, kF8On>;
  const size_t smem = tc_smem_bytes(W, a.net.n_layers, kTerms, kResident, kPersist);
  // per-device attributes (kernel_cfg): every device a context lives on gets the opt-in
  const KernelCfg kc = kernel_cfg(reinterpret_cast<const void*>(kernel), kThreads, smem, /*max_carveout=*/true);
  if (kc.err != cudaSuccess) return tc_failed(kc.err);
  // Residency from first principles (228 KB SMEM incl. 1 KB per CTA, 64K registers, TMEM
  // columns); the occupancy API is reported for reference only.
  const int by_smem = int((228 * 1024) / (smem + 1024));
  const int by_regs = 65536 / (std::max(kc.regs, 1) * kThreads);
  const int per_sm = std::max(1, std::min(by_smem, by_regs));
  if (getenv("NSDF_DEBUG_TC"))
    fprintf(stderr, "tc_mlp_kernel<%d,%d,%d,%d,%d,%d,%d>: smem %zu B, regs %d, %d CTAs/SM (occupancy API %d)\n", W,
            int(kGrad), kGroups, kTerms, int(kResident), int(kPersist), kHid, smem, kc.regs, per_sm, kc.occupancy);
  const int tmem_limit = 512 / (2 * W);  // two accumulator regions per CTA
  const int per = std::max(1, std::min(per_sm, tmem_limit));
  constexpr int kRaysPerTile = kGrad ? kRows / 4 : kRows;
  const int tiles = (n_max_items + kRaysPerTile - 1) / kRaysPerTile;
  const int grid = std::max(1, std::min(tiles, kc.sms * per));
  kernel<<<grid, kThreads, smem, s>>>(a);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TcLaunch::kRan : tc_failed(e);
}

// The hidden-layer count is compiled in for the standard architectures (64x1, 128x2, 256x3:
// the nets of every BASELINE config); other depths take the runtime-count kernels.
template <int W, bool kGrad, int kTerms, bool kResident, bool kPersist, bool kF8On>
TcLaunch launch_f(TcArgs& a, int n_max_items, cudaStream_t s) {
  constexpr int kStd = W == 64 ? 1 : (W == 128 ? 2 : 3);
  return a.net.n_layers - 2 == kStd ? launch_w<W, kGrad, kTerms, kResident, kPersist, kStd, kF8On>(a, n_max_items, s)
                                    : launch_w<W, kGrad, kTerms, kResident, kPersist, 0, kF8On>(a, n_max_items, s);
}
template <int W, bool kGrad, int kTerms, bool kResident, bool kPersist>
TcLaunch launch_h(TcArgs& a, int n_max_items, cudaStream_t s) {
  if constexpr (tc_split8(W) && !kGrad && kTerms == 3)
    if (a.net.f8_mask && !a.resume) return launch_f<W, kGrad, kTerms, kResident, kPersist, true>(a, n_max_items, s);
  return launch_f<W, kGrad, kTerms, kResident, kPersist, false>(a, n_max_items, s);
}

template <bool kGrad, int kTerms, bool kPersist>
TcLaunch launch_terms(TcArgs& a, int n_max_items, cudaStream_t s) {
  // 64-wide nets keep every hidden layer resident in SMEM when it fits (<= 4 layers).
  const bool resident = a.net.width == 64 && a.net.n_layers - 2 <= 4;
  switch (a.net.width) {
    case 64:
      return resident ? launch_h<64, kGrad, kTerms, true, kPersist>(a, n_max_items, s)
                      : launch_h<64, kGrad, kTerms, false, kPersist>(a, n_max_items, s);
    case 128: return launch_h<128, kGrad, kTerms, false, kPersist>(a, n_max_items, s);
    case 256: return launch_h<256, kGrad, kTerms, false, kPersist>(a, n_max_items, s);
    default: return TcLaunch::kDeclined;
  }
}

long long* timeline_buffer() {
  static long long* buf = nullptr;
  if (!getenv("NSDF_TC_TIMELINE")) return nullptr;
  if (!kTimeline) {
    static bool warned = false;
    if (!warned) fprintf(stderr, "NSDF_TC_TIMELINE: rebuild with NSDF_TC_TIMELINE_BUILD=1 (instrumentation not compiled in)\n");
    warned = true;
    return nullptr;
  }
  if (!buf) {
    cudaMallocManaged(&buf, kDbgSize * sizeof(long long));
    cudaMemset(buf, 0, kDbgSize * sizeof(long long));
  }
  return buf;
}
void timeline_dump(long long* buf, const char* what) {
  if (!buf) return;
  cudaDeviceSynchronize();
  fprintf(stderr,
          "timeline %s (SM cycles from the tile's start)\n  tile: a0fence  a0arr | dfull, epilogue end per MMA layer | "
          "ret  upd  flush || refill vote next\n",
          what);
  for (int t = 0; t < 12; ++t) {
    const long long* r = buf + t * 16;
    const long long* nx = buf + (t + 1) * 16;  // marks taken after the tile counter advanced
    auto d = [&](const long long* q, int k) { return q[k] ? q[k] - r[0] : -1; };
    fprintf(stderr, "  %2d: %6lld %6lld |", t, d(r, 10), d(r, 1));
    for (int k = 2; k < 10; ++k) fprintf(stderr, " %6lld", d(r, k));
    fprintf(stderr, " | %6lld %6lld %6lld || %6lld %6lld %6lld [refill steps %lld %lld]\n", d(nx, 11), d(nx, 12),
            d(nx, 13), d(nx, 14), d(nx, 15), nx[0] ? nx[0] - r[0] : -1, nx[8] ? nx[8] - r[0] : -1,
            nx[9] ? nx[9] - r[0] : -1);
  }
  for (int t = 0; t < 12; ++t) {
    const long long* q = buf + 65 * 16 + t * 4;
    fprintf(stderr, "  MMA issuer tile %2d: waits A0 %6lld, A blocks %6lld, weights %6lld of %6lld cycles\n", t, q[0],
            q[1], q[2], q[3]);
  }
  fprintf(stderr, "  tiles (all CTAs): %lld\n", buf[kDbgTiles]);
  // per-CTA spans (globaltimer): how long the level's tail keeps part of the GPU busy
  long long t0 = 0, t1 = 0;
  int n = 0;
  std::vector<long long> ends;
  std::vector<long long> tiles;
  double cyc = 0, nsec = 0;
  for (int c = 0; c < kDbgMaxCta; ++c) {
    const long long* q = buf + kDbgCta + 5 * c;
    if (!q[0]) continue;
    if (!n || q[0] < t0) t0 = q[0];
    t1 = std::max(t1, q[1]);
    ends.push_back(q[1]);
    tiles.push_back(q[2]);
    cyc += double(q[4] - q[3]);
    nsec += double(q[1] - q[0]);
    ++n;
  }
  if (n) {
    std::sort(ends.begin(), ends.end());
    std::sort(tiles.begin(), tiles.end());
    auto pe = [&](double f) { return (ends[std::min(n - 1, int(f * n))] - t0) / 1000.0; };
    fprintf(stderr, "  CTAs %d: span %.1f us; CTA end p10 %.1f p50 %.1f p90 %.1f max %.1f us; tiles/CTA min %lld "
            "p50 %lld max %lld; SM clock over the CTAs' lifetimes %.0f MHz\n", n, (t1 - t0) / 1000.0, pe(0.1), pe(0.5),
            pe(0.9), pe(1.0), tiles[0], tiles[n / 2], tiles[n - 1], nsec > 0 ? cyc / nsec * 1000.0 : 0.0);
  }
  {  // CTA 0's tile durations over the whole launch, in eighths of its tile sequence
    int nt = 0;
    while (nt < kDbgMaxTiles && buf[kDbgTileT + nt]) ++nt;
    if (nt > 16) {
      fprintf(stderr, "  CTA 0: %d tiles, mean cycles per tile by eighth of the launch:", nt);
      for (int e = 0; e < 8; ++e) {
        const int a0 = e * (nt - 1) / 8, a1 = (e + 1) * (nt - 1) / 8;
        fprintf(stderr, " %lld", a1 > a0 ? (buf[kDbgTileT + a1] - buf[kDbgTileT + a0]) / (a1 - a0) : 0ll);
      }
      fprintf(stderr, "\n");
    }
  }
  cudaMemset(buf, 0, kDbgSize * sizeof(long long));
}

template <bool kGrad, bool kPersist = false>
TcLaunch launch_any(TcArgs& a, int n_max_items, cudaStream_t s) {
  static const int claim_div = [] {
    const char* e = getenv("NSDF_TC_CLAIM_DIV");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  a.claim_div = claim_div;
  // rays per active CTA of a persistent level (NSDF_TC_MIN_ITEMS_<W> overrides): one tile's
  // rows for the short-tile 64/128-wide nets; several tiles' worth for the 256-wide level,
  // whose 29k-cycle tiles make a half-empty CTA the costliest idle (tools/shardsim.py)
  static const int min_items[3] = {
      [] { const char* e = getenv("NSDF_TC_MIN_ITEMS_64"); return e ? std::max(1, atoi(e)) : kRows; }(),
      [] { const char* e = getenv("NSDF_TC_MIN_ITEMS_128"); return e ? std::max(1, atoi(e)) : kRows; }(),
      [] { const char* e = getenv("NSDF_TC_MIN_ITEMS_256"); return e ? std::max(1, atoi(e)) : kRows; }()};
  a.min_items = min_items[a.net.width == 64 ? 0 : a.net.width == 128 ? 1 : 2];
  a.dbg = timeline_buffer();
  a.dbg_skip = getenv("NSDF_TC_TIMELINE_SKIP") ? std::max(0, atoi(getenv("NSDF_TC_TIMELINE_SKIP"))) : 0;
  if (a.dbg) {
    const TcLaunch ok = a.terms == 3 ? launch_terms<kGrad, 3, kPersist>(a, n_max_items, s)
                                     : launch_terms<kGrad, 1, kPersist>(a, n_max_items, s);
    char what[64];
    snprintf(what, sizeof what, "W=%d grad=%d persist=%d", a.net.width, int(kGrad), int(kPersist));
    timeline_dump(a.dbg, what);
    return ok;
  }
  return a.terms == 3 ? launch_terms<kGrad, 3, kPersist>(a, n_max_items, s)
                      : launch_terms<kGrad, 1, kPersist>(a, n_max_items, s);
}

TcNet tc_net(const DevNet& n) {
  TcNet t;
  t.n_layers = n.n_layers;
  t.width = n.rows[0];
  t.input_dim = n.input_dim;
  t.omega = n.omega;
  t.wq = reinterpret_cast<const __half*>(n.wq);
  t.w0 = n.w[0];
  t.b = n.bias_cat;
  t.wout = n.w[n.n_layers - 1];
  t.bout = n.bout;
  t.scale = std::ldexp(1.0f, n.tc_shift);
  t.inv_scale = std::ldexp(1.0f, -n.tc_shift);
  t.f8_mask = n.tc_f8_mask;
  return t;
}

}  // namespace

bool tc_supported(const DevNet& n) { return n.tc_ok != 0; }
bool tc_uses_e4m3(const DevNet& n) { return n.tc_ok != 0 && n.tc_f8_mask != 0 && tc_split8(n.rows[0]); }

cudaError_t tc_last_error() { return g_tc_error; }

TcLaunch tc_trace_level(int terms, const LevelDesc& lv, float eps, float t_max, const int* in_list, const int* in_count,
                    int* cursor, int* evals, int* adv_list, int* adv_count, const RayState& st, int n_max,
                    cudaStream_t s, int* refine_list, int* refine_count, bool resume) {
  TcArgs a{};
  a.refine_list = refine_list;
  a.refine_count = refine_count;
  a.resume = resume ? 1 : 0;
  a.terms = terms;
  a.net = tc_net(lv.field.net);
  a.op = kOpTrace;
  a.lv = lv;
  a.eps = eps;
  a.t_max = t_max;
  a.in_list = in_list;
  a.in_count = in_count;
  a.cursor = cursor;
  a.evals = evals;
  a.adv_list = adv_list;
  a.adv_count = adv_count;
  a.st = st;
  a.time = lv.time;
  return launch_any<false, true>(a, n_max, s);
}

TcLaunch tc_normals_shade(int terms, const DevField& nf, float time, const int* list, const int* count, int n_max,
                      const RayState& st, const ShadeParams& sp, bool defer_fallback, int* fb_list, int* fb_count,
                      float* rgb, float* depth, uint8_t* mask, cudaStream_t s) {
  TcArgs a{};
  a.terms = terms;
  a.net = tc_net(nf.net);
  a.op = kOpNormals;
  a.in_list = list;
  a.in_count = count;
  a.st = st;
  a.time = time;
  a.sp = sp;
  a.defer_fallback = defer_fallback ? 1 : 0;
  a.fb_list = fb_list;
  a.fb_count = fb_count;
  a.rgb = rgb;
  a.depth = depth;
  a.mask = mask;
  return launch_any<true>(a, n_max, s);
}

TcLaunch tc_eval(int terms, const DevField& f, const float* pts, int rows, int k, float time, float* out, float* grad,
             cudaStream_t s) {
  TcArgs a{};
  a.terms = terms;
  a.net = tc_net(f.net);
  a.op = kOpEval;
  a.pts = pts;
  a.rows = rows;
  a.k = k;
  a.time = time;
  a.out = out;
  a.grad = grad;
  // a 4-row batch carries a per-column time; the tiles fold a single slice time into the
  // layer-0 bias, so such batches take the FFMA tiles
  if (rows == 4) return TcLaunch::kDeclined;
  if (grad) return launch_any<true>(a, k, s);
  return launch_any<false>(a, k, s);
}

TcLaunch tc_normal_map(int terms, const DevField& f, const float* pts, int k, float time, double delta,
                   const float* fallback, float* normals, unsigned long long* counts, cudaStream_t s) {
  TcArgs a{};
  a.terms = terms;
  a.net = tc_net(f.net);
  a.op = kOpNormalMap;
  a.pts = pts;
  a.rows = 3;
  a.k = k;
  a.time = time;
  a.grad = normals;
  a.delta = delta;
  a.fallback = fallback;
  a.counts = counts;
  return launch_any<true>(a, k, s);
}

// The fast mode's activation, exactly as the tile epilogues evaluate it: sin(x) for value
// rows and sin(x + pi/2) = cos(x) for the tangent rows' derivative factor.
__global__ void fast_sine_probe_kernel(const float* x, int n, float* s, float* c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    s[i] = fast_sin(x[i]);
    c[i] = fast_sin(x[i] + kHalfPi);
  }
}

cudaError_t launch_fast_sine_probe(const float* x, int n, float* s, float* c, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  fast_sine_probe_kernel<<<std::min((n + 255) / 256, 148 * 8), 256, 0, st>>>(x, n, s, c);
  return cudaGetLastError();
}

cudaError_t check_report_tc(CheckRecord* out, bool reset) {
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
