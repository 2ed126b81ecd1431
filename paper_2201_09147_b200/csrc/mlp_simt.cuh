// FP32 "oracle mode" MLP tile: the accuracy path of the SIREN evaluator.
//
// One CTA (256 threads) evaluates a tile of kTileCols = 64 activation columns through the
// whole network, activations resident in shared memory (two ping-pong buffers of
// max_width x 64 floats).  Columns are either 64 points (value chain only) or 16 points x
// 4 chains (value + the 3 input-tangent chains of Alg. 2): the "width x 4 tile" of the
// analytic normal kernel.
//
// Arithmetic restates the reference AVX2 backend exactly (kernels_avx2.cpp:30-87,
// 152-176, 259-275; mlp.cpp:104-167):
//   - every output is acc = bias (or 0 on gradient chains), then acc = fma(W[i,kk], x[kk],
//     acc) for kk ascending — each thread owns whole outputs, so the chain is never split;
//   - sin / omega*cos via sincos_ref with separately rounded operations;
//   - G0_c = W0[i,c] * dphi, G_i = gemm(W_i, G) * dphi, output = Wn . G_c from 0.
// Hence results are bit-identical to the CPU path for any batch split.
//
// Thread mapping per hidden layer pass (kT threads: 256, or 1024 for 256-wide nets): rb =
// tid/16 owns 4 output rows, cb = tid%16 owns 4 columns; per k step one float4 of W^T (L1/L2, broadcast within the warp) and one float4
// of activations (conflict-free shared load) feed 16 FFMA.
#pragma once

#include "common.cuh"

namespace nsdf_b200 {

// Shared memory of one tile: two activation buffers [max_width][64] + staging.
__host__ __device__ constexpr size_t simt_tile_smem_bytes(int max_width) {
  return size_t(2) * size_t(max_width < 4 ? 4 : max_width) * kTileCols * sizeof(float);
}

template <bool kGrad, int kT>
__device__ __forceinline__ void simt_input_layer(const DevNet& n, const float* __restrict__ pts,
                                                 float* __restrict__ out) {
  // pts: [input_dim][kRays] staged points (row 3 = time for 4-input nets).
  constexpr int kRays = kGrad ? kTileCols / 4 : kTileCols;
  const int M = n.rows[0], K = n.cols[0];
  const float* __restrict__ w = n.w[0];
  const float* __restrict__ b = n.b[0];
  const bool sine = n.activation == NSDF_ACT_SINE;
  for (int idx = threadIdx.x; idx < M * kRays; idx += kT) {
    const int r = idx / kRays, ray = idx - r * kRays;
    float z = __ldg(b + r);
    for (int kk = 0; kk < K; ++kk) z = fmaf(__ldg(w + r * K + kk), pts[kk * kRays + ray], z);
    float s = z, c = 1.0f;
    if (sine) {
      sincos_ref(__fmul_rn(n.omega, z), s, c);
      c = __fmul_rn(n.omega, c);
    }
    if (kGrad) {
      float* o = out + r * kTileCols + ray * 4;
      o[0] = s;
      o[1] = __fmul_rn(__ldg(w + r * K + 0), c);  // scale_rows: W0[i,c] * dphi
      o[2] = __fmul_rn(__ldg(w + r * K + 1), c);
      o[3] = __fmul_rn(__ldg(w + r * K + 2), c);
    } else {
      out[r * kTileCols + ray] = s;
    }
  }
}

template <bool kGrad, int kT>
__device__ __forceinline__ void simt_hidden_layer(const DevNet& n, int l, const float* __restrict__ in,
                                                  float* __restrict__ out) {
  const int M = n.rows[l], K = n.cols[l], Mp = n.rows_pad[l];
  const float* __restrict__ wt = n.wt[l];
  const float* __restrict__ b = n.b[l];
  const bool sine = n.activation == NSDF_ACT_SINE;
  const int cb = threadIdx.x & 15, rb = threadIdx.x >> 4;
  const int c0 = cb * 4;
  for (int r0 = rb * 4; r0 < M; r0 += 4 * (kT / 16)) {
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float bi = r0 + i < M ? __ldg(b + r0 + i) : 0.0f;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = (!kGrad || j == 0) ? bi : 0.0f;
    }
    const float* __restrict__ wp = wt + r0;
    const float* __restrict__ xp = in + c0;
#pragma unroll 4
    for (int kk = 0; kk < K; ++kk) {
      const float4 w4 = __ldg(reinterpret_cast<const float4*>(wp + size_t(kk) * Mp));
      const float4 x4 = *reinterpret_cast<const float4*>(xp + kk * kTileCols);
      const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
      const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(wv[i], xv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (r0 + i >= M) break;
      float* o = out + (r0 + i) * kTileCols + c0;
      if (kGrad) {
        float s = acc[i][0], c = 1.0f;
        if (sine) {
          sincos_ref(__fmul_rn(n.omega, acc[i][0]), s, c);
          c = __fmul_rn(n.omega, c);
        }
        o[0] = s;
        o[1] = __fmul_rn(acc[i][1], c);  // hadamard(gemm, dphi), kernels_avx2.cpp:152-157
        o[2] = __fmul_rn(acc[i][2], c);
        o[3] = __fmul_rn(acc[i][3], c);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float s = acc[i][j], c;
          if (sine) sincos_ref(__fmul_rn(n.omega, acc[i][j]), s, c);
          o[j] = s;
        }
      }
    }
  }
}

// Whole network on one tile.  pts: [input_dim][rays]; results: vals[64] where column j is
// the network output of column j (for kGrad: column 4r = value, 4r+1..3 = gradient).
// bufA/bufB: [max_width][64].  Ends with a __syncthreads().
template <bool kGrad, int kT>
__device__ void simt_mlp_tile(const DevNet& n, const float* pts, float* bufA, float* bufB, float* vals) {
  constexpr int kRays = kGrad ? kTileCols / 4 : kTileCols;
  const int L = n.n_layers;
  if (L == 1) {  // affine network: mlp.cpp:115-126
    const int K = n.cols[0];
    for (int col = threadIdx.x; col < kTileCols; col += kT) {
      const int ray = kGrad ? col / 4 : col, chain = kGrad ? col % 4 : 0;
      float v;
      if (chain == 0) {
        v = __ldg(n.b[0]);
        for (int kk = 0; kk < K; ++kk) v = fmaf(__ldg(n.w[0] + kk), pts[kk * kRays + ray], v);
      } else {
        v = __ldg(n.w[0] + chain - 1);
      }
      vals[col] = v;
    }
    __syncthreads();
    return;
  }
  simt_input_layer<kGrad, kT>(n, pts, bufA);
  __syncthreads();
  float* in = bufA;
  float* out = bufB;
  for (int l = 1; l + 1 < L; ++l) {
    simt_hidden_layer<kGrad, kT>(n, l, in, out);
    __syncthreads();
    float* t = in;
    in = out;
    out = t;
  }
  // Output layer (1 x K): one fma chain per column, value from the bias, tangents from 0.
  const int K = n.cols[L - 1];
  const float* __restrict__ w = n.w[L - 1];
  for (int col = threadIdx.x; col < kTileCols; col += kT) {
    float acc = (!kGrad || (col & 3) == 0) ? __ldg(n.b[L - 1]) : 0.0f;
    for (int kk = 0; kk < K; ++kk) acc = fmaf(__ldg(w + kk), in[kk * kTileCols + col], acc);
    vals[col] = acc;
  }
  __syncthreads();
}

}  // namespace nsdf_b200
