// SIREN training on the B200 in FP64: the reference trainer's
// arithmetic restated on the device, bit for bit.
//
//   backprop_chunk   (backprop.cpp:17-62)  forward with the layer inputs and pre-activations
//                    kept, delta = scale*(f - y), per layer dW = delta . X^T, db = delta . 1,
//                    back = W^T . delta, delta = back (.) omega*cos(omega*pre)
//   batch_gradients  (backprop.cpp:93-124)  4096-point chunks, partials summed in chunk order
//   full_batch_loss  (backprop.cpp:126-152) forward per 4096-point chunk, sequential sums
//   momentum_step    (fit.cpp:31-49), fit_mlp (fit.cpp:87-196): shuffles, warmup, checkpoint,
//                    runaway rollback, plateau halving — the loop runs on the host, every
//                    tensor lives on the device.
//
// Every matrix product is the reference's gemm: each output is one fma chain over the inner
// index ascending from the bias (or 0) — gemm_f64_avx2 (kernels_avx2.cpp:89-150).  Here a CTA
// owns a 64 x 64 output tile, a thread 4 x 4 outputs, and the inner index is streamed through
// shared memory in order, so every chain is kept whole.  Compiled with -fmad=false: the
// explicit __fma_rn are the only fused operations; sin/cos via the separately rounded double
// Cephes scheme (common_f64.cuh).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common_f64.cuh"
#include "engine.cuh"

namespace nsdf_b200 {

namespace {

constexpr int kChunk = 4096;  // backprop.cpp:79 kTrainChunk
constexpr int kGT = 64;       // output tile edge
constexpr int kGK = 32;       // inner-index slab

// C[M x N] = init + op(A)[M x K] . op(B)[K x N];  A(i, kk) = kTA ? A[kk*lda + i] : A[i*lda + kk],
// B(kk, j) = kTB ? B[j*ldb + kk] : B[kk*ldb + j];  init = bias[i] (bias != null) or 0.
// kPer: outputs per thread edge (4: 64 x 64 CTA tile for wide products; 1: 16 x 16 tiles for
// the weight gradients, whose few outputs each carry a chain over all the chunk's points).
// The inner index runs in slabs of kGK through shared memory; the next slab is loaded into
// registers while the current one is consumed.
template <bool kTA, bool kTB, int kPer>
__global__ void __launch_bounds__(256) gemm_f64_kernel(const double* __restrict__ A, int lda,
                                                       const double* __restrict__ B, int ldb,
                                                       const double* __restrict__ bias, double* __restrict__ C,
                                                       int ldc, int M, int N, int K) {
  constexpr int kT = 16 * kPer;
  constexpr int kE = kGK * kT / 256;  // slab elements of A (and of B) per thread
  __shared__ double sa[kGK][kT + 1];
  __shared__ double sb[kGK][kT + 1];
  const int i0 = blockIdx.y * kT, j0 = blockIdx.x * kT;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  double acc[kPer][kPer];
#pragma unroll
  for (int a = 0; a < kPer; ++a) {
    const int i = i0 + ty * kPer + a;
    const double init = (bias && i < M) ? bias[i] : 0.0;
#pragma unroll
    for (int b = 0; b < kPer; ++b) acc[a][b] = init;
  }
  double ra[kE], rb[kE];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      const int e = threadIdx.x + q * 256;
      // element e of the slab: for A, (row r, k) with k fastest when A is K-contiguous
      const int kk = kTA ? e / kT : e % kGK, r = kTA ? e % kT : e / kGK;
      const int i = i0 + r, k = k0 + kk;
      ra[q] = (i < M && k < K) ? (kTA ? A[size_t(k) * lda + i] : A[size_t(i) * lda + k]) : 0.0;
      const int kb = kTB ? e % kGK : e / kT, cb = kTB ? e / kGK : e % kT;
      const int j = j0 + cb, k2 = k0 + kb;
      rb[q] = (j < N && k2 < K) ? (kTB ? B[size_t(j) * ldb + k2] : B[size_t(k2) * ldb + j]) : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      const int e = threadIdx.x + q * 256;
      const int kk = kTA ? e / kT : e % kGK, r = kTA ? e % kT : e / kGK;
      sa[kk][r] = ra[q];
      const int kb = kTB ? e % kGK : e / kT, cb = kTB ? e / kGK : e % kT;
      sb[kb][cb] = rb[q];
    }
  };
  load(0);
  for (int k0 = 0; k0 < K; k0 += kGK) {
    store();
    __syncthreads();
    if (k0 + kGK < K) load(k0 + kGK);  // next slab in flight while this one is consumed
    const int kn = min(kGK, K - k0);
    for (int kk = 0; kk < kn; ++kk) {
      double av[kPer], bv[kPer];
#pragma unroll
      for (int a = 0; a < kPer; ++a) av[a] = sa[kk][ty * kPer + a];
#pragma unroll
      for (int b = 0; b < kPer; ++b) bv[b] = sb[kk][tx * kPer + b];
#pragma unroll
      for (int a = 0; a < kPer; ++a)
#pragma unroll
        for (int b = 0; b < kPer; ++b) acc[a][b] = __fma_rn(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < kPer; ++a) {
    const int i = i0 + ty * kPer + a;
    if (i >= M) continue;
#pragma unroll
    for (int b = 0; b < kPer; ++b) {
      const int j = j0 + tx * kPer + b;
      if (j < N) C[size_t(i) * ldc + j] = acc[a][b];
    }
  }
}

// db = delta . 1 (backprop.cpp:53): per row one chain acc = fma(delta[i][j], 1.0, acc) over j
// ascending, i.e. a sequential sum; one thread per row.
__global__ void rowsum_kernel(const double* __restrict__ d, int ld, int M, int K, double* __restrict__ out, int ldo) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const double* r = d + size_t(i) * ld;
  double acc = 0.0;
  int j = 0;
  for (; j + 4 <= K; j += 4) {
    const double a0 = r[j], a1 = r[j + 1], a2 = r[j + 2], a3 = r[j + 3];
    acc = __fma_rn(a0, 1.0, acc);
    acc = __fma_rn(a1, 1.0, acc);
    acc = __fma_rn(a2, 1.0, acc);
    acc = __fma_rn(a3, 1.0, acc);
  }
  for (; j < K; ++j) acc = __fma_rn(r[j], 1.0, acc);
  out[size_t(i) * ldo] = acc;
}

template <bool kTA, bool kTB>
void gemm(const double* A, int lda, const double* B, int ldb, const double* bias, double* C, int ldc, int M, int N,
          int K, cudaStream_t s) {
  if (M <= 0 || N <= 0) return;
  const long wide_tiles = long((N + kGT - 1) / kGT) * ((M + kGT - 1) / kGT);
  if (wide_tiles >= 296 || K < 1024) {
    dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT);
    gemm_f64_kernel<kTA, kTB, 4><<<grid, 256, 0, s>>>(A, lda, B, ldb, bias, C, ldc, M, N, K);
  } else {  // few outputs, long chains: spread the outputs over more SMs
    dim3 grid((N + 15) / 16, (M + 15) / 16);
    gemm_f64_kernel<kTA, kTB, 1><<<grid, 256, 0, s>>>(A, lda, B, ldb, bias, C, ldc, M, N, K);
  }
}

// sine_f64 (kernels_avx2.cpp:336-352): value sin(w*x), derivative w*cos(w*x)
__global__ void activate_kernel(const double* x, double* out, size_t n, double omega, int sine, int derivative) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    if (!sine) {
      out[i] = derivative ? 1.0 : x[i];
      continue;
    }
    double s, c;
    sincos_ref_d(__dmul_rn(omega, x[i]), s, c);
    out[i] = derivative ? __dmul_rn(omega, c) : s;
  }
}

__global__ void hadamard_kernel(const double* a, const double* b, double* out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = __dmul_rn(a[i], b[i]);
}

// delta = scale * (out - y) (backprop.cpp:36-42); the sum of squares runs in point order
// in a single thread (sse = sse + r*r, separately rounded) when requested
__global__ void delta_kernel(const double* out, const double* y, int k, double scale, double* delta) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x)
    delta[j] = __dmul_rn(scale, __dsub_rn(out[j], y[j]));
}
__global__ void sse_chunks_kernel(const double* out, const double* y, int n, int chunk, double* sse) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int lo = c * chunk;
  if (lo >= n) return;
  const int hi = min(n, lo + chunk);
  double s = 0.0;
  for (int j = lo; j < hi; ++j) {
    const double r = __dsub_rn(out[j], y[j]);
    s = __dadd_rn(s, __dmul_rn(r, r));
  }
  sse[c] = s;
}

__global__ void add_kernel(double* into, const double* from, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    into[i] = __dadd_rn(into[i], from[i]);
}

// v = momentum*v - lr*g; w += v (fit.cpp:31-49)
__global__ void momentum_kernel(double* w, double* v, const double* g, size_t n, double momentum, double lr) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    v[i] = __dsub_rn(__dmul_rn(momentum, v[i]), __dmul_rn(lr, g[i]));
    w[i] = __dadd_rn(w[i], v[i]);
  }
}

// minibatch columns in shuffled order: dst[r][j] = src[r][order[start + j]]
__global__ void gather_kernel(const double* src, int n, int rows, const int* order, int start, int count, double* dst,
                              const double* ysrc, double* ydst) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x) {
    const int c = order[start + j];
    for (int r = 0; r < rows; ++r) dst[size_t(r) * count + j] = src[size_t(r) * n + c];
    ydst[j] = ysrc[c];
  }
}

__global__ void fill_kernel(double* p, size_t n, double v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = v;
}

// wt (K x Rp) element (k, i) = W[i][k]; the pad rows stay zero
__global__ void transpose_kernel(const double* w, int R, int K, int Rp, double* wt) {
  const size_t n = size_t(K) * Rp;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
    const int k = int(e / Rp), i = int(e % Rp);
    wt[e] = i < R ? w[size_t(i) * K + k] : 0.0;
  }
}

int grid1(size_t n) { return int(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 148 * 16))); }

}  // namespace

// Device state of one training run; packed parameter layout = the C ABI's (per layer W then b).
struct TrainNet {
  int L = 0, input_dim = 3, sine = 1;
  double omega = 30.0;
  std::vector<int> rows, cols;
  std::vector<size_t> woff, boff;
  size_t total = 0;
  int max_width = 0;
  void layout(int n_layers, const int32_t* r, const int32_t* c) {
    L = n_layers;
    rows.assign(r, r + n_layers);
    cols.assign(c, c + n_layers);
    woff.resize(L);
    boff.resize(L);
    size_t o = 0;
    max_width = input_dim;
    for (int l = 0; l < L; ++l) {
      woff[l] = o;
      o += size_t(rows[l]) * cols[l];
      boff[l] = o;
      o += rows[l];
      max_width = std::max(max_width, std::max(rows[l], cols[l]));
    }
    total = o;
  }
};

namespace {

struct DBuf {
  double* p = nullptr;
  size_t n = 0;
  cudaError_t reserve(size_t need) {
    if (need <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, need * sizeof(double));
    if (e == cudaSuccess) n = need;
    return e;
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

struct TrainScratch {
  DBuf acts;   // inputs[l] and pre[l] of one chunk
  DBuf tmp;    // delta / back / dphi
  DBuf ones;   // all 1.0 (the bias gradient's gemm(delta, ones))
  DBuf part;   // one chunk's parameter gradients
  DBuf xc;     // one chunk's points
};

// One chunk: backprop_chunk (backprop.cpp:17-62).  params/grads packed; X: input_dim x k; y: k.
// grads are written (not accumulated).  When sse != null, the chunk's sum of squares lands there.
static cudaError_t backprop_chunk_dev(const TrainNet& net, const double* params, const double* X, const double* y,
                                      int k, double scale, double* grads, double* sse, TrainScratch& sc,
                                      cudaStream_t s) {
  const int L = net.L;
  // activation storage: inputs[l] (cols[l] x k) for l = 0..L-1 (inputs[0] = X), pre[l] (rows[l] x k)
  std::vector<size_t> in_off(L), pre_off(L);
  size_t o = 0;
  for (int l = 0; l < L; ++l) {
    in_off[l] = o;
    if (l > 0) o += size_t(net.cols[l]) * k;
    pre_off[l] = o;
    o += size_t(net.rows[l]) * k;
  }
  if (cudaError_t e = sc.acts.reserve(o + 1)) return e;
  const size_t tmpn = size_t(net.max_width) * k;
  if (cudaError_t e = sc.tmp.reserve(3 * tmpn + 1)) return e;
  if (sc.ones.n < size_t(k)) {
    if (cudaError_t e = sc.ones.reserve(size_t(k))) return e;
    fill_kernel<<<grid1(sc.ones.n), 256, 0, s>>>(sc.ones.p, sc.ones.n, 1.0);
  }
  auto inp = [&](int l) -> const double* { return l == 0 ? X : sc.acts.p + in_off[l]; };
  // ---- forward: pre_l = W_l . in_l + b_l; in_{l+1} = sin(omega pre_l) ----
  for (int l = 0; l < L; ++l) {
    double* pre = sc.acts.p + pre_off[l];
    gemm<false, false>(params + net.woff[l], net.cols[l], inp(l), k, params + net.boff[l], pre, k, net.rows[l], k,
                       net.cols[l], s);
    if (l + 1 < L) {
      const size_t n = size_t(net.rows[l]) * k;
      activate_kernel<<<grid1(n), 256, 0, s>>>(pre, sc.acts.p + in_off[l + 1], n, net.omega, net.sine, 0);
    }
  }
  // ---- output delta (1 x k) ----
  double* delta = sc.tmp.p;
  double* back = sc.tmp.p + tmpn;
  double* dphi = sc.tmp.p + 2 * tmpn;
  const double* out = sc.acts.p + pre_off[L - 1];
  delta_kernel<<<grid1(k), 256, 0, s>>>(out, y, k, scale, delta);
  if (sse) sse_chunks_kernel<<<1, 32, 0, s>>>(out, y, k, k, sse);
  // ---- backward ----
  for (int l = L - 1; l >= 0; --l) {
    const int R = net.rows[l], K = net.cols[l];
    // dW = delta (R x k) . in_l^T (k x K);  db = delta . 1
    gemm<false, true>(delta, k, inp(l), k, nullptr, grads + net.woff[l], K, R, K, k, s);
    rowsum_kernel<<<(R + 127) / 128, 128, 0, s>>>(delta, k, R, k, grads + net.boff[l], 1);
    if (l > 0) {
      // back = W^T (K x R) . delta (R x k); delta = back (.) omega cos(omega pre_{l-1})
      gemm<true, false>(params + net.woff[l], K, delta, k, nullptr, back, k, K, k, R, s);
      const size_t n = size_t(K) * k;
      activate_kernel<<<grid1(n), 256, 0, s>>>(sc.acts.p + pre_off[l - 1], dphi, n, net.omega, net.sine, 1);
      hadamard_kernel<<<grid1(n), 256, 0, s>>>(back, dphi, delta, n);
    }
  }
  return cudaGetLastError();
}

// batch_gradients (backprop.cpp:93-124): 4096-point chunks, scale 2/n of the whole batch,
// partials summed in chunk order.
static cudaError_t batch_gradients_dev(const TrainNet& net, const double* params, const double* X, const double* y,
                                       int n, double* grads, TrainScratch& sc, cudaStream_t s) {
  const int rows = net.input_dim;
  if (cudaError_t e = sc.part.reserve(net.total)) return e;
  // chunk columns are contiguous slices only when rows == 1; copy each chunk's points
  DBuf& xc = sc.xc;
  if (cudaError_t e = xc.reserve(size_t(rows) * kChunk)) return e;
  const double scale = 2.0 / n;
  for (int ci = 0, lo = 0; lo < n; ++ci, lo += kChunk) {
    const int k = std::min(kChunk, n - lo);
    for (int r = 0; r < rows; ++r)
      cudaMemcpyAsync(xc.p + size_t(r) * k, X + size_t(r) * n + lo, size_t(k) * 8, cudaMemcpyDeviceToDevice, s);
    double* dst = ci == 0 ? grads : sc.part.p;
    if (cudaError_t e = backprop_chunk_dev(net, params, xc.p, y + lo, k, scale, dst, nullptr, sc, s)) return e;
    if (ci > 0) add_kernel<<<grid1(net.total), 256, 0, s>>>(grads, sc.part.p, net.total);
  }
  return cudaGetLastError();
}

// Packed parameters -> the FP64 evaluator's DevNet view (row-major W, transposed copy, biases).
static cudaError_t bind_devnet(const TrainNet& net, const double* params, DBuf& wt, DevNet& dn, cudaStream_t s) {
  std::memset(&dn, 0, sizeof(dn));
  dn.n_layers = net.L;
  dn.input_dim = net.input_dim;
  dn.activation = net.sine ? NSDF_ACT_SINE : NSDF_ACT_IDENTITY;
  dn.omega_d = net.omega;
  dn.omega = float(net.omega);
  dn.max_width = net.max_width;
  size_t need = 0;
  for (int l = 0; l < net.L; ++l) need += size_t(net.cols[l]) * ((net.rows[l] + 3) / 4 * 4);
  if (cudaError_t e = wt.reserve(need + 1)) return e;
  size_t o = 0;
  for (int l = 0; l < net.L; ++l) {
    const int R = net.rows[l], K = net.cols[l], Rp = (R + 3) / 4 * 4;
    dn.rows[l] = R;
    dn.cols[l] = K;
    dn.rows_pad[l] = Rp;
    dn.w64[l] = params + net.woff[l];
    dn.b64[l] = params + net.boff[l];
    transpose_kernel<<<grid1(size_t(K) * Rp), 256, 0, s>>>(params + net.woff[l], R, K, Rp, wt.p + o);
    dn.wt64[l] = wt.p + o;
    o += size_t(K) * Rp;
  }
  return cudaGetLastError();
}

// full_batch_loss (backprop.cpp:126-152): forward of every point, chunk sums in point order,
// chunks summed in order (host), / n.
static double full_batch_loss_dev(const TrainNet& net, const double* params, const double* X, const double* y, int n,
                                  DBuf& wt, DBuf& outb, cudaStream_t s, cudaError_t* err) {
  DevNet dn;
  *err = bind_devnet(net, params, wt, dn, s);
  if (*err) return 0.0;
  const int chunks = (n + kChunk - 1) / kChunk;
  if ((*err = outb.reserve(size_t(n) + chunks + 1))) return 0.0;
  if ((*err = launch_eval_f64(dn, X, net.input_dim, n, 0.0, outb.p, nullptr, s))) return 0.0;
  sse_chunks_kernel<<<(chunks + 63) / 64, 64, 0, s>>>(outb.p, y, n, kChunk, outb.p + n);
  std::vector<double> sse(chunks);
  cudaMemcpyAsync(sse.data(), outb.p + n, size_t(chunks) * 8, cudaMemcpyDeviceToHost, s);
  if ((*err = cudaStreamSynchronize(s))) return 0.0;
  double total = 0;
  for (double v : sse) total += v;
  return total / n;
}

// ---- public entry points (capi.cu) ------------------------------------------------------
cudaError_t train_backprop(int n_layers, const int32_t* rows, const int32_t* cols, const double* params_h,
                           int activation, double omega0, int input_dim, const double* points_h,
                           const double* targets_h, int k, double* grads_h, double* loss, cudaStream_t s) {
  TrainNet net;
  net.input_dim = input_dim;
  net.sine = activation == NSDF_ACT_SINE;
  net.omega = omega0;
  net.layout(n_layers, rows, cols);
  DBuf p, x, y, g, sse;
  cudaError_t e;
  if ((e = p.reserve(net.total)) || (e = x.reserve(size_t(input_dim) * k + 1)) || (e = y.reserve(size_t(k) + 1)) ||
      (e = g.reserve(net.total)) || (e = sse.reserve(1)))
    return e;
  cudaMemcpyAsync(p.p, params_h, net.total * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(x.p, points_h, size_t(input_dim) * k * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(y.p, targets_h, size_t(k) * 8, cudaMemcpyHostToDevice, s);
  TrainScratch sc;
  // backprop_sine_mlp (backprop.cpp:66-78): the whole batch as ONE chunk, scale 2/n
  if ((e = backprop_chunk_dev(net, p.p, x.p, y.p, k, 2.0 / k, g.p, sse.p, sc, s))) return e;
  double sse_h = 0;
  cudaMemcpyAsync(grads_h, g.p, net.total * 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&sse_h, sse.p, 8, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s))) return e;
  if (loss) *loss = sse_h / k;
  return cudaSuccess;
}

cudaError_t train_fit(int n_layers, const int32_t* rows, const int32_t* cols, double* params_h, int activation,
                      double omega0, int input_dim, uint64_t* rng, const double* points_h, const double* targets_h,
                      int n, const double* val_points_h, const double* val_targets_h, int n_val,
                      const nsdf_train_config* cfg, double* epoch_loss, nsdf_train_report* rep, cudaStream_t s) {
  TrainNet net;
  net.input_dim = input_dim;
  net.sine = activation == NSDF_ACT_SINE;
  net.omega = omega0;
  net.layout(n_layers, rows, cols);
  const size_t P = net.total;
  DBuf params, vel, ckpt, grads, X, Y, bx, by, wt, outb, vX, vY;
  DBuf order_d;  // int order, stored in a double buffer
  cudaError_t e;
  const int batch = cfg->batch_size > 0 ? std::min(cfg->batch_size, n) : n;
  if ((e = params.reserve(P)) || (e = vel.reserve(P)) || (e = ckpt.reserve(P)) || (e = grads.reserve(P)) ||
      (e = X.reserve(size_t(input_dim) * n + 1)) || (e = Y.reserve(size_t(n) + 1)) ||
      (e = bx.reserve(size_t(input_dim) * batch + 1)) || (e = by.reserve(size_t(batch) + 1)) ||
      (e = order_d.reserve(size_t(n) / 2 + 1)))
    return e;
  cudaMemcpyAsync(params.p, params_h, P * 8, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(vel.p, 0, P * 8, s);
  cudaMemcpyAsync(X.p, points_h, size_t(input_dim) * n * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(Y.p, targets_h, size_t(n) * 8, cudaMemcpyHostToDevice, s);
  // Rng (core.hpp xoshiro256++) continued from the caller's state after random_init
  auto next_u64 = [&]() {
    auto rotl = [](uint64_t v, int k) { return (v << k) | (v >> (64 - k)); };
    const uint64_t result = rotl(rng[0] + rng[3], 23) + rng[0];
    const uint64_t t = rng[1] << 17;
    rng[2] ^= rng[0];
    rng[3] ^= rng[1];
    rng[1] ^= rng[2];
    rng[0] ^= rng[3];
    rng[2] ^= t;
    rng[3] = rotl(rng[3], 45);
    return result;
  };
  std::memset(rep, 0, sizeof(*rep));
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  int* order_dev = reinterpret_cast<int*>(order_d.p);
  TrainScratch sc;
  double lr = cfg->learning_rate;
  cudaMemcpyAsync(ckpt.p, params.p, P * 8, cudaMemcpyDeviceToDevice, s);
  double checkpoint_loss = full_batch_loss_dev(net, params.p, X.p, Y.p, n, wt, outb, s, &e);
  if (e) return e;
  std::vector<double> loss_history;
  int window_start = 0, recorded = 0;
  for (int epoch = 0; epoch < cfg->epochs; ++epoch) {
    const double warm =
        cfg->warmup_epochs > 0 ? std::min(1.0, double(epoch + 1) / cfg->warmup_epochs) : 1.0;
    for (int i = n - 1; i > 0; --i) std::swap(order[i], order[next_u64() % uint64_t(i + 1)]);
    cudaMemcpyAsync(order_dev, order.data(), size_t(n) * 4, cudaMemcpyHostToDevice, s);
    for (int start = 0; start < n; start += batch) {
      const int count = std::min(batch, n - start);
      gather_kernel<<<grid1(count), 256, 0, s>>>(X.p, n, input_dim, order_dev, start, count, bx.p, Y.p, by.p);
      if ((e = batch_gradients_dev(net, params.p, bx.p, by.p, count, grads.p, sc, s))) return e;
      momentum_kernel<<<grid1(P), 256, 0, s>>>(params.p, vel.p, grads.p, P, cfg->momentum, lr * warm);
    }
    const double loss = full_batch_loss_dev(net, params.p, X.p, Y.p, n, wt, outb, s, &e);
    if (e) return e;
    if (!std::isfinite(loss)) {
      rep->diverged = 1;
      epoch_loss[recorded++] = checkpoint_loss;
      break;
    }
    if (loss > 100.0 * checkpoint_loss + 1e-12) {  // runaway pass: back to the checkpoint at half the rate
      cudaMemcpyAsync(params.p, ckpt.p, P * 8, cudaMemcpyDeviceToDevice, s);
      cudaMemsetAsync(vel.p, 0, P * 8, s);
      lr *= 0.5;
      ++rep->halvings;
      epoch_loss[recorded++] = checkpoint_loss;
      if (lr < cfg->min_learning_rate) break;
      continue;
    }
    if (loss < checkpoint_loss) {
      cudaMemcpyAsync(ckpt.p, params.p, P * 8, cudaMemcpyDeviceToDevice, s);
      checkpoint_loss = loss;
    }
    epoch_loss[recorded++] = checkpoint_loss;
    loss_history.push_back(checkpoint_loss);
    const int window = int(loss_history.size()) - window_start;
    if (window >= cfg->plateau_patience) {
      const double before = loss_history[window_start];
      if (checkpoint_loss > before * (1.0 - cfg->plateau_threshold)) {
        cudaMemcpyAsync(params.p, ckpt.p, P * 8, cudaMemcpyDeviceToDevice, s);
        cudaMemsetAsync(vel.p, 0, P * 8, s);
        lr *= 0.5;
        ++rep->halvings;
        if (lr < cfg->min_learning_rate) break;
      }
      window_start = int(loss_history.size());
    }
  }
  cudaMemcpyAsync(params_h, ckpt.p, P * 8, cudaMemcpyDeviceToHost, s);
  rep->final_loss = checkpoint_loss;
  rep->final_learning_rate = lr;
  rep->epochs_recorded = recorded;
  // validation_stats (fit.cpp:51-62): forward, sequential mse and max |error|
  if (n_val > 0) {
    if ((e = vX.reserve(size_t(input_dim) * n_val)) || (e = vY.reserve(size_t(n_val)))) return e;
    cudaMemcpyAsync(vX.p, val_points_h, size_t(input_dim) * n_val * 8, cudaMemcpyHostToDevice, s);
    DevNet dn;
    if ((e = bind_devnet(net, ckpt.p, wt, dn, s))) return e;
    if ((e = launch_eval_f64(dn, vX.p, input_dim, n_val, 0.0, vY.p, nullptr, s))) return e;
    std::vector<double> out(n_val);
    cudaMemcpyAsync(out.data(), vY.p, size_t(n_val) * 8, cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s))) return e;
    double mse = 0, mx = 0;
    for (int j = 0; j < n_val; ++j) {
      const double err = out[j] - val_targets_h[j];
      mse += err * err;
      mx = std::max(mx, std::abs(err));
    }
    rep->validation_mse = mse / n_val;
    rep->validation_max_error = mx;
  }
  return cudaStreamSynchronize(s);
}

}  // namespace nsdf_b200
