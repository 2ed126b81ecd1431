// Dense tensor kernels of the reference's kernel table (tensor/kernels.hpp:26-39) on the
// device: the drop-in's tensor::gemm / hadamard / scale_rows / activate (ops.cpp:24-95) run
// here, reproducing the reference's AVX2 backend bit for bit (compiled with -fmad=false, every
// product and sum explicitly rounded):
//   gemm        every output element one k-sequential fma chain from the bias (or 0):
//               acc = fma(a[i,kk], b[kk,j], acc), kk ascending (kernels_avx2.cpp:30-54, the
//               column tail :78-86 and the f64 twin use the same chain)
//   hadamard    a[i] * b[i];  scale_rows  col[i] * m[i,j]
//   sine        sin(omega*x) / omega*cos(omega*x), the argument rounded as omega*x first, the
//               Cephes polynomials of sincos_poly_avx2(_d) (kernels_avx2.cpp:203-333)
// One thread per output element, threads along the column index (coalesced B / C rows).
#include "engine.cuh"
#include "common_f64.cuh"

namespace nsdf_b200 {
namespace {

template <class T>
__device__ __forceinline__ T fma_rn(T a, T b, T c);
template <>
__device__ __forceinline__ float fma_rn<float>(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <>
__device__ __forceinline__ double fma_rn<double>(double a, double b, double c) { return __fma_rn(a, b, c); }

template <class T>
__global__ void gemm_kernel(const T* __restrict__ a, const T* __restrict__ b, const T* __restrict__ bias,
                            T* __restrict__ c, int m, int n, int k) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int i = blockIdx.y; i < m; i += gridDim.y) {
    const T* ar = a + size_t(i) * k;
    T acc = bias ? bias[i] : T(0);
    for (int kk = 0; kk < k; ++kk) acc = fma_rn<T>(ar[kk], b[size_t(kk) * n + j], acc);
    c[size_t(i) * n + j] = acc;
  }
}

template <class T>
__global__ void hadamard_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out, size_t n) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = a[i] * b[i];
}

template <class T>
__global__ void scale_rows_kernel(const T* __restrict__ col, const T* __restrict__ m, T* __restrict__ out, int rows,
                                  int cols) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  for (int i = blockIdx.y; i < rows; i += gridDim.y) out[size_t(i) * cols + j] = col[i] * m[size_t(i) * cols + j];
}

__global__ void sine_f32_kernel(const float* __restrict__ x, float* __restrict__ out, size_t n, float omega,
                                int derivative) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    float s, c;
    sincos_ref(__fmul_rn(omega, x[i]), s, c);
    out[i] = derivative ? __fmul_rn(omega, c) : s;
  }
}

__global__ void sine_f64_kernel(const double* __restrict__ x, double* __restrict__ out, size_t n, double omega,
                                int derivative) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    double s, c;
    sincos_ref_d(__dmul_rn(omega, x[i]), s, c);
    out[i] = derivative ? __dmul_rn(omega, c) : s;
  }
}

int grid_1d(size_t n) { return int(std::min<size_t>((n + 255) / 256, size_t(148) * 16)); }

}  // namespace

void launch_tensor_gemm(bool f64, const void* a, const void* b, const void* bias, void* c, int m, int n, int k,
                        cudaStream_t s) {
  if (m <= 0 || n <= 0) return;
  const dim3 grid((n + 127) / 128, std::min(m, 65535));
  if (f64)
    gemm_kernel<double><<<grid, 128, 0, s>>>(static_cast<const double*>(a), static_cast<const double*>(b),
                                             static_cast<const double*>(bias), static_cast<double*>(c), m, n, k);
  else
    gemm_kernel<float><<<grid, 128, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(b),
                                            static_cast<const float*>(bias), static_cast<float*>(c), m, n, k);
}

void launch_tensor_hadamard(bool f64, const void* a, const void* b, void* out, size_t n, cudaStream_t s) {
  if (n == 0) return;
  if (f64)
    hadamard_kernel<double><<<grid_1d(n), 256, 0, s>>>(static_cast<const double*>(a), static_cast<const double*>(b),
                                                       static_cast<double*>(out), n);
  else
    hadamard_kernel<float><<<grid_1d(n), 256, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(b),
                                                      static_cast<float*>(out), n);
}

void launch_tensor_scale_rows(bool f64, const void* col, const void* m, void* out, int rows, int cols,
                              cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  const dim3 grid((cols + 127) / 128, std::min(rows, 65535));
  if (f64)
    scale_rows_kernel<double><<<grid, 128, 0, s>>>(static_cast<const double*>(col), static_cast<const double*>(m),
                                                   static_cast<double*>(out), rows, cols);
  else
    scale_rows_kernel<float><<<grid, 128, 0, s>>>(static_cast<const float*>(col), static_cast<const float*>(m),
                                                  static_cast<float*>(out), rows, cols);
}

void launch_tensor_sine(bool f64, const void* x, void* out, size_t n, double omega, bool derivative,
                        cudaStream_t s) {
  if (n == 0) return;
  if (f64)
    sine_f64_kernel<<<grid_1d(n), 256, 0, s>>>(static_cast<const double*>(x), static_cast<double*>(out), n, omega,
                                               derivative ? 1 : 0);
  else
    sine_f32_kernel<<<grid_1d(n), 256, 0, s>>>(static_cast<const float*>(x), static_cast<float*>(out), n,
                                               float(omega), derivative ? 1 : 0);
}

}  // namespace nsdf_b200
