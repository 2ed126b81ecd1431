// Throughput probe: TMEM reads (tcgen05.ld.32x32b) and writes (tcgen05.st) per SM per clock
// on this GPU, and the mix the SIREN epilogue runs (one 16-column fp32 load, 16 sines, one
// 8-column store per block).  One CTA per SM owns all 512 TMEM columns; W warps (a multiple
// of 4: warp w reads lanes 32*(w%4)..+31) each loop over their column slice.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/tmem_probe tools/probes/tmem_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// kOp 0: loads only (x16 per instruction, wait per instruction)
//     1: loads, two in flight per wait (x16 + x16)
//     2: stores only (x8)
//     3: epilogue mix: load x16 -> 16 MUFU sines -> store x8 (hi parts)
template <int kOp>
__global__ void probe(unsigned long long* cycles, uint32_t* sink, int iters) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t q = warp & 3, slice = warp >> 2, nslices = nw >> 2;
  const uint32_t cols = 512 / nslices;  // this warp's column slice
  const uint32_t taddr = tbase + (q * 32 << 16) + slice * cols;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (uint32_t c = 0; c + 32 <= cols; c += 32) {
      uint32_t r[32];
      if (kOp == 0 || kOp == 3) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr + c));
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
              "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr + c + 16));
      } else if (kOp == 1) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
              "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr + c), "r"(taddr + c + 16));
      }
      if (kOp == 3) {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__sinf(__uint_as_float(r[j]) + float(it)));
      }
      if (kOp == 2 || kOp == 3) {
        const uint32_t v = kOp == 2 ? acc + c : r[0];
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n\t"
            "tcgen05.st.sync.aligned.32x32b.x8.b32 [%9], {%10,%11,%12,%13,%14,%15,%16,%17};\n\t"
            "tcgen05.wait::st.sync.aligned;" ::"r"(taddr + c),
            "r"(v), "r"(kOp == 3 ? r[1] : v), "r"(kOp == 3 ? r[2] : v), "r"(kOp == 3 ? r[3] : v),
            "r"(kOp == 3 ? r[4] : v), "r"(kOp == 3 ? r[5] : v), "r"(kOp == 3 ? r[6] : v), "r"(kOp == 3 ? r[7] : v),
            "r"(taddr + c + 16), "r"(kOp == 3 ? r[16] : v), "r"(kOp == 3 ? r[17] : v), "r"(kOp == 3 ? r[18] : v),
            "r"(kOp == 3 ? r[19] : v), "r"(kOp == 3 ? r[20] : v), "r"(kOp == 3 ? r[21] : v),
            "r"(kOp == 3 ? r[22] : v), "r"(kOp == 3 ? r[23] : v)
            : "memory");
      }
      if (kOp != 2)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc ^= r[j];
    }
  }
  const long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) atomicMax(cycles + blockIdx.x, (unsigned long long)(t1 - t0));
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  cudaMalloc(&sink, sizeof(uint32_t) * sms * 1024);
  const int iters = 2000;
  const char* names[4] = {"ld x16 (wait each)", "ld 2 x x16 in flight", "st x8", "ld x16 + 16 sin + st x8 (epilogue mix)"};
  for (int op = 0; op < 4; ++op)
    for (int warps : {4, 8, 16}) {
      unsigned long long best = ~0ull;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(cyc, 0, sizeof(unsigned long long) * sms);
        if (op == 0) probe<0><<<sms, warps * 32>>>(cyc, sink, iters);
        if (op == 1) probe<1><<<sms, warps * 32>>>(cyc, sink, iters);
        if (op == 2) probe<2><<<sms, warps * 32>>>(cyc, sink, iters);
        if (op == 3) probe<3><<<sms, warps * 32>>>(cyc, sink, iters);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        unsigned long long h[1024];
        cudaMemcpy(h, cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
        unsigned long long m = 0;
        for (int i = 0; i < sms; ++i) m = h[i] > m ? h[i] : m;
        best = m < best ? m : best;
      }
      // per SM and iteration the warps cover 128 lanes x 512 columns; loads move 4 B per
      // column, stores (x8 of every 16 columns) half of that
      const double elems = double(iters) * 128 * 512;
      const double bytes = op == 2 ? elems * 2 : elems * 4;
      printf("%-40s warps %2d: %8.1f B/clk/SM (%s), %.2f activations/clk/SM\n", names[op], warps,
             bytes / double(best), op == 2 ? "stored" : "loaded", elems / double(best));
    }
  return 0;
}
