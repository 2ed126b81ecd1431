// Shared device-side definitions of the nsdf B200 engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "nsdf_cuda.h"

namespace nsdf_b200 {

constexpr int kMaxLayers = 16;     // hidden blocks <= 14
constexpr int kMaxLevels = NSDF_MAX_LEVELS;
constexpr int kMaxWidth = 256;     // widest layer the device engine tiles
constexpr int kThreads = 256;      // CTA size of the narrow FFMA (oracle-mode) tiles (engine.cu: wide_tile)
constexpr int kTileCols = 64;      // activation columns per FFMA tile (rays, or rays x 4 chains)

enum FieldKind : int { kFieldMlp = 0, kFieldSphere = 1, kFieldTorus = 2, kFieldBox = 3 };

// Device view of an uploaded network (MlpParams<float>, the f32 cast of field.cpp:150).
//   w[l]   row-major out x in (layer 0 and the output layer read it directly)
//   wt[l]  transposed in x rows_pad (rows padded to a multiple of 4 with zeros) so a
//          thread's 4 consecutive output rows are one aligned float4 per k step.
struct DevNet {
  int n_layers;
  int input_dim;
  int activation;  // NSDF_ACT_SINE / NSDF_ACT_IDENTITY
  float omega;     // float(ActivationSpec::omega0), as sine_f32 receives it (ops.cpp:299)
  int max_width;
  int rows[kMaxLayers];
  int cols[kMaxLayers];
  int rows_pad[kMaxLayers];
  const float* w[kMaxLayers];
  const float* wt[kMaxLayers];
  const float* b[kMaxLayers];
  // Fast-mode (tcgen05) copy, built at upload when tc-eligible (mlp_tc.cu):
  int tc_ok;
  const uint16_t* wq;      // hidden layers [h][hi | lo][W*W] fp16, canonical layout in N-blocks (tc_wq_offset)
  const float* bias_cat;   // biases of layers 0 .. L-2, [L-1][width]
  float bout;              // output bias
  int tc_shift;            // hidden weights / biases uploaded x 2^tc_shift (tc_split8 nets, mlp_tc.cuh)
  int tc_f8_mask;          // bit h: hidden layer h runs its correction terms as one E4M3 MMA
  // FP64 master copy (the certification path, mlp_f64.cu): same layouts as w / wt / b.
  double omega_d;
  const double* w64[kMaxLayers];
  const double* wt64[kMaxLayers];
  const double* b64[kMaxLayers];
};

struct DevField {
  int kind;
  DevNet net;
  double analytic[4];
};

// Ray state, structure of arrays indexed by ray slot (SoA as BatchState, trace.cpp:26-31).
struct RayState {
  float* px;
  float* py;
  float* pz;
  float* t;
  float* dx;
  float* dy;
  float* dz;
  uint16_t* iters;      // [slot * kMaxLevels + level]
  int* level_reached;
  float* final_dist;
  uint8_t* hit;
  int* pixel;           // image pixel of the slot (render/trace_image); null = identity
  int cap;              // slot capacity (the length of every per-slot array and list)
  int n_pix;            // framebuffer pixels (W*H) the slots' pixels index
};

// ---------------------------------------------------------------------------------
// Oracle-mode sin/cos: the Cephes restatement of sincos_poly.hpp:90-133 (the scalar twin
// of the AVX2 lanes, kernels_avx2.cpp:203-257), every multiply and add separately
// rounded so nvcc cannot contract them.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void sincos_ref(float x, float& s, float& c) {
  const float kFourOverPi = 1.27323954473516f;
  const float kDp1 = -0.78515625f;
  const float kDp2 = -2.4187564849853515625e-4f;
  const float kDp3 = -3.77489497744594108e-8f;
  const float kSin0 = -1.9515295891e-4f;
  const float kSin1 = 8.3321608736e-3f;
  const float kSin2 = -1.6666654611e-1f;
  const float kCos0 = 2.443315711809948e-5f;
  const float kCos1 = -1.388731625493765e-3f;
  const float kCos2 = 4.166664568298827e-2f;
  uint32_t bits = __float_as_uint(x);
  uint32_t sign_sin = bits & 0x80000000u;
  float ax = __uint_as_float(bits & 0x7fffffffu);
  float y = __fmul_rn(ax, kFourOverPi);
  int q = __float2int_rz(y);
  q = (q + 1) & ~1;
  y = __int2float_rn(q);
  uint32_t swap_sign = uint32_t(q & 4) << 29;
  bool poly_sin = (q & 2) == 0;
  float r = ax;
  r = __fadd_rn(r, __fmul_rn(y, kDp1));
  r = __fadd_rn(r, __fmul_rn(y, kDp2));
  r = __fadd_rn(r, __fmul_rn(y, kDp3));
  float z = __fmul_rn(r, r);
  float pc = kCos0;
  pc = __fadd_rn(__fmul_rn(pc, z), kCos1);
  pc = __fadd_rn(__fmul_rn(pc, z), kCos2);
  pc = __fmul_rn(__fmul_rn(pc, z), z);
  pc = __fsub_rn(pc, __fmul_rn(z, 0.5f));
  pc = __fadd_rn(pc, 1.0f);
  float ps = kSin0;
  ps = __fadd_rn(__fmul_rn(ps, z), kSin1);
  ps = __fadd_rn(__fmul_rn(ps, z), kSin2);
  ps = __fmul_rn(__fmul_rn(ps, z), r);
  ps = __fadd_rn(ps, r);
  float ysin = poly_sin ? ps : pc;
  s = __uint_as_float(__float_as_uint(ysin) ^ sign_sin ^ swap_sign);
  int qc = q - 2;
  uint32_t cos_sign = uint32_t(~qc & 4) << 29;
  bool cos_poly_sin = (qc & 2) == 0;
  float ycos = cos_poly_sin ? ps : pc;
  c = __uint_as_float(__float_as_uint(ycos) ^ cos_sign);
}

// std::hypot as the reference's host computes it (glibc >= 2.35, x86-64 build without FMA:
// Borges' corrected kernel, with the EPS early-out and power-of-two rescaling at the
// extremes).  CUDA's hypot differs from it in the last bit (~0.6% of arguments), which the
// float cast of a torus distance can expose; this restatement matched glibc 2.39 on 5e6
// random argument pairs, and tests/test_gpu_parity.py checks it against the compiled
// reference's analytic torus bit for bit.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    const double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    const double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

__device__ __forceinline__ double hypot_ref(double x, double y) {
  double ax = fabs(x), ay = fabs(y);
  if (isinf(ax) || isinf(ay)) return __longlong_as_double(0x7ff0000000000000ll);
  if (isnan(ax) || isnan(ay)) return __dadd_rn(ax, ay);
  if (ax < ay) {
    const double t = ax;
    ax = ay;
    ay = t;
  }
  constexpr double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
    return __ddiv_rn(hypot_kernel(__dmul_rn(ax, kScale), __dmul_rn(ay, kScale)), kScale);
  }
  if (ay < kTiny) {
    if (ax >= __ddiv_rn(ay, kEps)) return __dadd_rn(ax, ay);
    return __dmul_rn(hypot_kernel(__ddiv_rn(ax, kScale), __ddiv_rn(ay, kScale)), kScale);
  }
  if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
  return hypot_kernel(ax, ay);
}

// Analytic fields in double, cast to float like Field::eval_batch's default
// (field.cpp:11-29); shapes from field.cpp:57-124.  Test scenes, not the perf path.
__device__ __forceinline__ double analytic_eval(const DevField& f, double x, double y, double z) {
  const double* a = f.analytic;
  if (f.kind == kFieldSphere) {
    double dx = __dadd_rn(x, -a[0]), dy = __dadd_rn(y, -a[1]), dz = __dadd_rn(z, -a[2]);
    double n2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    return __dadd_rn(__dsqrt_rn(n2), -a[3]);
  }
  if (f.kind == kFieldTorus) {
    double s = hypot_ref(x, z);
    return __dsub_rn(hypot_ref(__dsub_rn(s, a[0]), y), a[1]);
  }
  double qx = fabs(x) - a[0], qy = fabs(y) - a[1], qz = fabs(z) - a[2];
  double px = fmax(qx, 0.0), py = fmax(qy, 0.0), pz = fmax(qz, 0.0);
  double outside = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), __dmul_rn(pz, pz)));
  double inside = fmin(fmax(qx, fmax(qy, qz)), 0.0);
  return outside + inside;
}

__device__ __forceinline__ void analytic_grad(const DevField& f, double x, double y, double z, double g[3]) {
  const double* a = f.analytic;
  g[0] = g[1] = g[2] = 0.0;
  if (f.kind == kFieldSphere) {
    double dx = __dadd_rn(x, -a[0]), dy = __dadd_rn(y, -a[1]), dz = __dadd_rn(z, -a[2]);
    double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    if (n == 0) return;
    g[0] = __ddiv_rn(dx, n);
    g[1] = __ddiv_rn(dy, n);
    g[2] = __ddiv_rn(dz, n);
    return;
  }
  if (f.kind == kFieldTorus) {
    double s = hypot_ref(x, z);
    double q = __dsub_rn(s, a[0]);
    double d = hypot_ref(q, y);
    if (d == 0) return;
    if (s == 0) {
      g[1] = __ddiv_rn(y, d);
      return;
    }
    double ff = __ddiv_rn(q, __dmul_rn(d, s));
    g[0] = __dmul_rn(x, ff);
    g[1] = __ddiv_rn(y, d);
    g[2] = __dmul_rn(z, ff);
    return;
  }
  auto sgn = [](double v) { return v < 0 ? -1.0 : 1.0; };
  double qx = fabs(x) - a[0], qy = fabs(y) - a[1], qz = fabs(z) - a[2];
  if (qx > 0 || qy > 0 || qz > 0) {
    double px = fmax(qx, 0.0), py = fmax(qy, 0.0), pz = fmax(qz, 0.0);
    double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), __dmul_rn(pz, pz)));
    if (n == 0) return;
    g[0] = sgn(x) * px / n;
    g[1] = sgn(y) * py / n;
    g[2] = sgn(z) * pz / n;
    return;
  }
  if (qx >= qy && qx >= qz) g[0] = sgn(x);
  else if (qy >= qz) g[1] = sgn(y);
  else g[2] = sgn(z);
}

// ---------------------------------------------------------------------------------
// Checked build (NSDF_CHECKED=1: build.py build_cuda(checked=True) ->
// paper_2201_09147_b200/_checked/libnsdf_cuda.so).  Every list index, ray slot, staged
// append and framebuffer pixel the kernels compute is bounds-checked on the device: a
// violation is counted (the first one's site, value and bound recorded, per translation
// unit) and the access skipped, so tests can assert a clean run
// (nsdf_cuda_check_report; tests/test_gpu_checked.py).  Compiled out otherwise.
// ---------------------------------------------------------------------------------
#ifndef NSDF_CHECKED
#define NSDF_CHECKED 0
#endif
enum CheckSite : int {
  kChkListRead = 1,   // list item index < list length
  kChkSlot = 2,       // ray slot < slot capacity
  kChkStage = 3,      // CTA staging index < staging capacity
  kChkListWrite = 4,  // compaction / flush write index < list capacity
  kChkPixel = 5,      // framebuffer pixel < W*H
};
struct CheckRecord {
  unsigned long long count;
  int site, value, bound, pad;
};
#if NSDF_CHECKED
static __device__ CheckRecord g_check;
#endif
__device__ __forceinline__ bool in_bounds(long long v, long long bound, int site) {
#if NSDF_CHECKED
  if (v >= 0 && v < bound) return true;
  if (atomicAdd(&g_check.count, 1ull) == 0ull) {
    g_check.site = site;
    g_check.value = int(v);
    g_check.bound = int(bound);
  }
  return false;
#else
  (void)v, (void)bound, (void)site;
  return true;
#endif
}

// Warp-aggregated append of `pred` lanes to a global list of `cap` entries (one atomic per warp).
__device__ __forceinline__ void warp_append(bool pred, int value, int* list, int* count, int cap = 0x7fffffff) {
  const unsigned mask = __ballot_sync(0xffffffffu, pred);
  if (mask == 0) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(count, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
  const int at = base + __popc(mask & ((1u << lane) - 1u));
  if (pred && in_bounds(at, cap, kChkListWrite)) list[at] = value;
}

}  // namespace nsdf_b200
