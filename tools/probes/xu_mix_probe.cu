// Does the epilogue's fp16 packing compete with MUFU.SIN for the XU pipe?  Sines per SM per
// clock (clock64 over the kernel, so the power-capped clock does not matter) for:
//   0: sin.approx only            1: + F2FP pack of each pair (hi parts)
//   2: + the full split (hi pack, unpack, FFMA2 residual, lo pack) as the 64-wide epilogue does
//   3: F2FP packs only (no sine)
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

template <int kOp>
__global__ void probe(float* out, unsigned long long* cyc, int iters, float seed) {
  float x[16];
  for (int i = 0; i < 16; ++i) x[i] = seed + threadIdx.x * 1e-3f + i;
  uint32_t acc = 0;
  const long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float a = x[i], b = x[i + 1];
      if (kOp != 3) {
        a = __sinf(a);
        b = __sinf(b);
      }
      if (kOp >= 1) {
        __half2 h = __floats2half2_rn(a, b);
        uint32_t hw = *reinterpret_cast<uint32_t*>(&h);
        acc ^= hw;
        if (kOp == 2) {
          const float2 d = __ffma2_rn(__half22float2(h), make_float2(-1.0f, -1.0f), make_float2(a, b));
          __half2 l = __floats2half2_rn(d.x, d.y);
          acc += *reinterpret_cast<uint32_t*>(&l);
        }
        if (kOp == 3) { a += 1e-7f; b += 1e-7f; }
      }
      x[i] = a + 0.5f;
      x[i + 1] = b + 0.5f;
    }
  }
  const long long c1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) atomicAdd(cyc, (unsigned long long)(c1 - c0));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  unsigned long long* cyc; cudaMalloc(&cyc, 8);
  const int iters = 2048, blocks_per_sm = 4, threads = 512;
  const char* names[4] = {"sin only", "sin + F2FP hi pack", "sin + hi/lo split (64-wide epilogue)", "F2FP packs only"};
  for (int op = 0; op < 4; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cyc, 0, 8);
      if (op == 0) probe<0><<<sms * blocks_per_sm, threads>>>(out, cyc, iters, 0.5f);
      if (op == 1) probe<1><<<sms * blocks_per_sm, threads>>>(out, cyc, iters, 0.5f);
      if (op == 2) probe<2><<<sms * blocks_per_sm, threads>>>(out, cyc, iters, 0.5f);
      if (op == 3) probe<3><<<sms * blocks_per_sm, threads>>>(out, cyc, iters, 0.5f);
      cudaDeviceSynchronize();
      unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // per CTA: threads * iters * 16 values over its cycles; CTAs per SM run concurrently
      const double cyc_per_cta = double(c) / (sms * blocks_per_sm);
      const double vals_per_sm_clk = double(threads) * iters * 16 * blocks_per_sm / cyc_per_cta;
      if (rep) printf("%-40s %6.2f values per SM per clock\n", names[op], vals_per_sm_clk);
    }
  }
  return 0;
}
