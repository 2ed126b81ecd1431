// Tensor-core (tcgen05) fast path of the SIREN evaluator — launchers implemented in
// mlp_tc.cu.  Each returns kDeclined when the request is outside what the tiles handle
// (the caller then runs the FFMA tile on the device and reports NSDF_PATH_SIMT; there is
// no CPU path) and kFailed when a launch it should have made did not happen (attribute
// opt-in or launch error; tc_last_error() holds the CUDA error) — a hard error for the
// caller, never a silent fallback.
#pragma once

#include "engine.cuh"

namespace nsdf_b200 {

enum class TcLaunch { kRan, kDeclined, kFailed };

// Hidden-layer weights of a W-wide net are issued as tc_halves(W) N-blocks of W / halves
// output columns each (256-wide: two), so the epilogue of a layer's first half runs under the
// MMAs of its second half.  (128-wide: one — two 64-column blocks measured slower, 1.66 vs
// 1.60 ms for the level; two CTAs per SM already overlap each other's layer boundaries.)  Upload layout of one part (hi or lo, W x W fp16):
// [N-block][K/8][NB/8][8 rows][8 k], NB = W / halves — every (N-block, K chunk) piece is one
// contiguous bulk copy in the UMMA canonical K-major layout (SBO 128 B, LBO NB*16 B).
#ifndef NSDF_TC_NH128
#define NSDF_TC_NH128 1
#endif
__host__ __device__ constexpr int tc_halves(int W) { return W == 256 ? 2 : (W == 128 ? NSDF_TC_NH128 : 1); }
__host__ __device__ constexpr size_t tc_wq_offset(int W, int n, int k) {
  return size_t(n / (W / tc_halves(W))) * size_t(W / tc_halves(W)) * W +
         size_t(((k / 8) * (W / tc_halves(W) / 8) + (n % (W / tc_halves(W))) / 8) * 64 + (n % 8) * 8 + k % 8);
}
// FP8 correction terms (128- and 256-wide nets, forward tiles): the split-precision product
//   A.W = A_hi.W_hi + A_lo.W_hi + A_hi.W_lo
// keeps A_hi.W_hi as one kind::f16 MMA and runs both correction terms as ONE kind::f8f6f4
// MMA of K = 32 (E4M3): A'' = [fp8(A) | fp8(A_lo * 2^s)] (16 + 16 K values, the 8 spare
// TMEM columns of each in-place A block), B'' = [fp8(W_lo) ; fp8(W_hi * 2^-s)] — at twice
// the f16 rate, so 2 MMA slots per K step instead of 3.  The hidden weights of such nets are
// uploaded scaled by 2^s (s = tc_shift, <= 11: fp8's range needs A_lo * 2^s), so their
// accumulators hold 2^s x the sine argument and the epilogue scales by 2^-s.  Per hidden
// layer: [hi | lo (fp16, for the normal tiles) | lo8 (the B'' pieces, 2 W^2 bytes)].
#ifndef NSDF_TC_F8
#define NSDF_TC_F8 1
#endif
#ifndef NSDF_TC_F8_128
#define NSDF_TC_F8_128 1  // 128-wide nets too (frame 6.83 -> 6.69 ms, tools/ab.py)
#endif
#ifndef NSDF_TC_F8_64
#define NSDF_TC_F8_64 0
#endif
__host__ __device__ constexpr bool tc_split8(int W) {
  return NSDF_TC_F8 && (W == 256 || (NSDF_TC_F8_128 && W == 128) || (NSDF_TC_F8_64 && W == 64));
}
constexpr double kF8MaxOmega = 15.0;  // nets at larger omega0 keep fp16 correction terms (capi.cu)
__host__ __device__ constexpr int tc_parts(int W) { return tc_split8(W) ? 3 : 2; }  // fp16-sized parts per layer
// Byte offset of B''(n, k2) of 16-K block b (k2 < 16: fp8(W_lo[n][16b + k2]); k2 >= 16:
// fp8(W_hi[n][16b + k2 - 16] * 2^-s)): per N-block, blocks in K order, each [NB][32] in the
// K-major canonical layout of 8-bit operands (core matrices of 8 rows x 16 bytes, LBO NB*16 B,
// SBO 128 B) — so a streamed (N-block, K chunk) piece has the byte offset and size of the
// fp16 lo piece it replaces.
__host__ __device__ constexpr size_t tc_w8_offset(int W, int n, int b, int k2) {
  return size_t(n / (W / tc_halves(W))) * size_t(W / tc_halves(W)) * W * 2 + size_t(b) * (W / tc_halves(W)) * 32 +
         size_t(((k2 / 16) * (W / tc_halves(W) / 8) + (n % (W / tc_halves(W))) / 8) * 128 + (n % 8) * 16 + k2 % 16);
}
cudaError_t tc_last_error();  // CUDA error of this thread's last kFailed launch

// Persistent level trace: one launch runs every iteration of a level; rows are refilled
// from in_list (claimed through *cursor) until it drains.  Converged slots -> adv_list,
// evaluations -> *evals.  cursor / evals / adv_count must be zeroed.
// E4M3 levels (tc_uses_e4m3): with refine_list (final levels), rays whose stop decision falls
// within a small band of eps are parked there (count in *refine_count); a second call with
// resume = true over that list (fp16 correction terms, iteration counts from st.iters)
// finishes them, so every decision is the fp16-term one.
TcLaunch tc_trace_level(int terms, const LevelDesc& lv, float eps, float t_max, const int* in_list, const int* in_count,
                    int* cursor, int* evals, int* adv_list, int* adv_count, const RayState& st, int n_max,
                    cudaStream_t s, int* refine_list = nullptr, int* refine_count = nullptr, bool resume = false);
bool tc_uses_e4m3(const DevNet& n);
TcLaunch tc_normals_shade(int terms, const DevField& nf, float time, const int* list, const int* count, int n_max,
                      const RayState& st, const ShadeParams& sp, bool defer_fallback, int* fb_list, int* fb_count,
                      float* rgb, float* depth, uint8_t* mask, cudaStream_t s);
TcLaunch tc_eval(int terms, const DevField& f, const float* pts, int rows, int k, float time, float* out, float* grad,
             cudaStream_t s);

TcLaunch tc_normal_map(int terms, const DevField& f, const float* pts, int k, float time, double delta,
                   const float* fallback, float* normals, unsigned long long* counts, cudaStream_t s);

// The fast-mode sine exactly as the epilogues use it (sin and sin(x + pi/2)), for the
// accuracy test at large omega0 * z arguments.
cudaError_t launch_fast_sine_probe(const float* x, int n, float* s, float* c, cudaStream_t st);

}  // namespace nsdf_b200
