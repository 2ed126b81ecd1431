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

}  // namespace nsdf_b200
