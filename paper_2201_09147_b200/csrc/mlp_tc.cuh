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
cudaError_t tc_last_error();  // CUDA error of this thread's last kFailed launch

// Persistent level trace: one launch runs every iteration of a level; rows are refilled
// from in_list (claimed through *cursor) until it drains.  Converged slots -> adv_list,
// evaluations -> *evals.  cursor / evals / adv_count must be zeroed.
TcLaunch tc_trace_level(int terms, const LevelDesc& lv, float eps, float t_max, const int* in_list, const int* in_count,
                    int* cursor, int* evals, int* adv_list, int* adv_count, const RayState& st, int n_max,
                    cudaStream_t s);
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
