// Throughput probe: sin.approx (MUFU.SIN), F2FP pack, FFMA — per SM per clock on this GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

template <int kOp>
__global__ void probe(float* out, int iters, float seed) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = seed + threadIdx.x * 1e-3f + i;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (kOp == 0) x[i] = __sinf(x[i]) + 1.0f;            // MUFU.SIN (+FMUL.RZ, FADD)
      if (kOp == 1) {                                     // F2FP pack + unpack
        __half2 h = __floats2half2_rn(x[i], x[(i + 1) & 7]);
        acc += *reinterpret_cast<uint32_t*>(&h);
        x[i] = x[i] * 1.0001f + 1e-7f;
      }
      if (kOp == 2) x[i] = fmaf(x[i], 1.0001f, 1e-7f);     // FFMA
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  const int iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[3] = {"sin.approx (FMUL.RZ+MUFU.SIN+FADD)", "F2FP pack (+FFMA)", "FFMA"};
  for (int op = 0; op < 3; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (op == 0) probe<0><<<sms * 8, 256>>>(out, iters, 0.5f);
      if (op == 1) probe<1><<<sms * 8, 256>>>(out, iters, 0.5f);
      if (op == 2) probe<2><<<sms * 8, 256>>>(out, iters, 0.5f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = double(sms) * 8 * 256 * iters * 8;
      if (rep) printf("%-40s %8.1f Gop/s = %6.2f per SM per clk (at %d MHz nominal)\n", names[op], ops / ms / 1e6,
                      ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
