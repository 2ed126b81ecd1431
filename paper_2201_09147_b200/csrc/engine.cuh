// Host-side launch interface of the engine kernels (engine.cu).  Used by the C ABI
// (capi.cu); everything here is device-pointer based and asynchronous on `stream`.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace nsdf_b200 {

// Camera basis computed on the host in double exactly as generate_rays does
// (camera.cpp:21-26); per-pixel arithmetic runs on the device.
struct CamBasis {
  double fwd[3], right[3], up[3];
  double half_h, half_w;
  float origin[3];
  int width, height;
};

// Lights normalized on the host exactly as shade() does (shade.cpp:59-65).
struct ShadeParams {
  float albedo[3];
  float ambient, diffuse, specular, shininess;
  int n_lights;
  float light[NSDF_MAX_LIGHTS][4];  // x, y, z, intensity
  float background[3];
  float cam[3];                     // Vec3f::from(camera.position), shade.cpp:53
};

// One traced level as the kernels see it.
struct LevelDesc {
  DevField field;
  float time;
  float delta;    // float(seq.deltas[j]) or 0 at the final level (trace.cpp:111)
  int budget;
  int final_level;
  int level;      // index j into iterations_used
};

// Resizable device workspace owned by a context.
struct Workspace {
  void* base = nullptr;
  size_t bytes = 0;
  void* host_pinned = nullptr;
  size_t host_bytes = 0;
  ~Workspace();
  cudaError_t reserve(size_t need);
  cudaError_t reserve_host(size_t need);
};

// Carves the ray-state arrays and lists out of a workspace.
struct FrameBuffers {
  RayState st;
  int* list[3];
  int* counters;   // per-iteration list sizes + adv counts + misc
  int n_counters;
  int* fallback_list;
};
size_t frame_workspace_bytes(int n_rays, int n_counters);
FrameBuffers carve_frame(void* base, int n_rays, int n_counters);

// CUDA-event timing per kernel family (nsdf_cuda_set_profiling).  Events are recorded on
// the launching stream around each family and folded into `acc` by collect().
struct Profiler {
  enum Kind { kLevel0 = 0, kNormals = NSDF_MAX_LEVELS, kFrame = NSDF_MAX_LEVELS + 1 };
  bool on = false;
  nsdf_profile acc{};
  std::vector<cudaEvent_t> pool;
  struct Span {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Span> pending;
  cudaEvent_t begin(cudaStream_t s);
  void end(int kind, cudaEvent_t a, cudaStream_t s);
  void collect();
  void reset();
  ~Profiler();
};

// Which kernel family runs the MLP tiles.
enum class Mode : int { Fp32Oracle = 0, Fp16Fast = 1, Fp16Low = 2 };
inline int mode_terms(Mode m) { return m == Mode::Fp16Low ? 1 : 3; }
// The render's normal + shading tiles only need a DIRECTION within the 0.5 deg tolerance:
// one fp16 term per K step (angle error at identical points <= 0.07 deg on the omega0 = 10
// sequence, 0.16 deg at omega0 = 30; tests/test_gpu_fast.py) instead of the trace's three,
// whose depth tolerance (1e-3, the eps_stop jitter) needs |df| ~ 1e-5.  NSDF_NORMAL_TERMS=3
// restores the split.  The normal-map API (a13: its delta-gate counts compare |f| with delta)
// keeps the trace's arithmetic.
int normal_tile_terms(Mode m);
inline bool mode_tc(Mode m) { return m != Mode::Fp32Oracle; }

struct TraceResult {
  int* hit_list;        // device: slots that converged at the final level
  int* hit_count;       // device counter
  std::vector<int> counter_layout_base;  // offsets of per-level iteration counters
  std::vector<char> persistent;          // level traced by one persistent launch
  int launches = 0;
  cudaError_t error = cudaSuccess;       // a tcgen05 launch failed (the frame is invalid)
  int failed_level = -1;
};

// Ray generation for all pixels (world == 1, slot == pixel) or the owned image tiles.
// Returns the number of slots on the device counter `n_slots` (host value written when
// world == 1).
// `owners` (device, one entry per tile, may be null): explicit tile -> rank map instead of
// tile % tile_world (nsdf_cuda_set_tile_owners).
void launch_generate_rays(const CamBasis& cb, int tile_size, int tile_rank, int tile_world, const int* owners,
                          RayState st, int* n_slots_dev, cudaStream_t s);
void launch_rays_to_host_layout(const RayState& st, int n, float* rays6, cudaStream_t s);
void launch_init_state_from_rays(const float* rays6, int n, RayState st, cudaStream_t s);
void launch_reset_state(RayState st, int n, cudaStream_t s);

// Multiscale sphere tracing of `n_slots` rays (trace.cpp:86-132): level by level — one
// persistent launch per level (tensor-core modes) or one compacting launch per iteration
// (FFMA oracle tiles).  counters must be zeroed.  Returns the hit list.
TraceResult run_trace(Mode mode, const std::vector<LevelDesc>& levels, float eps, float t_max,
                      FrameBuffers& fb, int n_slots_host_max, const int* n_slots_dev,
                      cudaStream_t s, Profiler* prof = nullptr);

void launch_write_records(const RayState& st, int n, nsdf_hit_record* out, cudaStream_t s);
void launch_mark_hits(const int* list, const int* count, int n_max, RayState st, cudaStream_t s);

// Framebuffer background for the slots' pixels (render.cpp:28-33).
// Pack the framebuffer pixels of the frame's slots (the owned tiles of a sharded frame) into
// slot order: rgb 3 x n, depth, mask and the pixel index of every slot.
void launch_pack_owned(const RayState& st, const int* n_slots_dev, int n_max, const float* rgb, const float* depth,
                       const uint8_t* mask, float* p_rgb, float* p_depth, uint8_t* p_mask, int* p_pixel,
                       cudaStream_t s);

void launch_scatter_packed(const int* count_dev, int n_max, const float* p_rgb, const float* p_depth,
                           const uint8_t* p_mask, const int* p_pixel, float* rgb, float* depth, uint8_t* mask,
                           cudaStream_t s);

void launch_fb_background(const RayState& st, const int* n_slots_dev, int n_max,
                          const ShadeParams& sp, float* rgb, float* depth, uint8_t* mask,
                          cudaStream_t s);
// Normals (fused fwd + 3 tangent chains) + normalize/fallback + shade + framebuffer write
// for the hit list (render.cpp:48-80).  With `defer_fallback`, zero-gradient hits are
// appended to fb_list instead of getting (0,1,0).  Returns the kernel path that ran
// (NSDF_PATH_TCGEN05 / NSDF_PATH_SIMT) or -1 when a tcgen05 launch failed.
int launch_normals_shade(Mode mode, const DevField& nf, float time, const int* list,
                         const int* count, int n_max, const RayState& st, const ShadeParams& sp,
                         bool defer_fallback, int* fb_list, int* fb_count, float* rgb,
                         float* depth, uint8_t* mask, cudaStream_t s);

// Batch evaluation of a field (API path).
cudaError_t launch_eval(Mode mode, const DevField& f, const float* pts, int rows, int k, float time,
                        float* out, float* grad, cudaStream_t s);
cudaError_t launch_normal_map(Mode mode, const DevField& f, const float* pts, int k, float time,
                       double delta, const float* fallback, float* normals,
                       unsigned long long* counts, cudaStream_t s);
// shading::map_normals_to_mesh on the device: vertices k x 3 double (Vec3 array), normals
// k x 3 double (pre-filled with the kept normals), counts {mapped, violators, fallbacks};
// pts / vals / grads are 3k / k / 3k float scratch.
cudaError_t launch_map_mesh_normals(Mode mode, const DevField& f, float time, const double* vertices, int k,
                                    double delta, float* pts, float* vals, float* grads, double* normals,
                                    unsigned long long* counts, cudaStream_t s);
void launch_shade(const float* pts, const float* normals, int k, const ShadeParams& sp, float* rgb,
                  cudaStream_t s);

// Mesh G-buffer: nearest ray-triangle hit per pixel (Moller-Trumbore, fp32).
void launch_raycast_mesh(const CamBasis& cb, const float* tri_verts /* n_tri x 9 */, int n_tri, float* positions,
                         uint8_t* mask, cudaStream_t s);

// FP64 batch evaluation (mlp_f64.cu): forward_batch<double> / gradient_batch<double>
// bit-exact with the reference's AVX2 double path.  pts rows x k (device), out k, grad 3 x k.
cudaError_t launch_eval_f64(const DevNet& n, const double* pts, int rows, int k, double time, double* out, double* grad,
                     cudaStream_t s);

// FP64 evaluation of any device field (neural: launch_eval_f64; sphere / torus / box in
// double as field.cpp:57-124), device buffers.
cudaError_t launch_eval_field_f64(const DevField& f, const double* pts, int rows, int k, double time, double* out,
                                  double* grad, cudaStream_t s);
// sample_near_surface's projection (nesting.cpp:98-127) on resident points: `steps` Newton
// steps from the k candidates (Vec3 array), keep |f| <= keep_tol; the kept points and the
// field gradient at them (Vec3 arrays, input order) and their count (device int).
size_t projection_workspace_doubles(int k);
cudaError_t launch_project_to_surface(const DevField& f, double time, const double* cand, int k, double keep_tol,
                                      int steps, double* ws, double* kept, double* kept_g, int* d_count,
                                      cudaStream_t s);

// FP64 SIREN training (train_f64.cu), host buffers in/out.
cudaError_t train_backprop(int n_layers, const int32_t* rows, const int32_t* cols, const double* params_h,
                           int activation, double omega0, int input_dim, const double* points_h,
                           const double* targets_h, int k, double* grads_h, double* loss, cudaStream_t s);
cudaError_t train_fit(int n_layers, const int32_t* rows, const int32_t* cols, double* params_h, int activation,
                      double omega0, int input_dim, uint64_t* rng, const double* points_h, const double* targets_h,
                      int n, const double* val_points_h, const double* val_targets_h, int n_val,
                      const nsdf_train_config* cfg, double* epoch_loss, nsdf_train_report* rep, cudaStream_t s);

// The reference's dense kernel table on the device (tensor_ops.cu, tensor/kernels.hpp:26-39),
// bit-exact with its AVX2 backend; f64 selects double buffers.  Device pointers, async.
void launch_tensor_gemm(bool f64, const void* a, const void* b, const void* bias, void* c, int m, int n, int k,
                        cudaStream_t s);
void launch_tensor_hadamard(bool f64, const void* a, const void* b, void* out, size_t n, cudaStream_t s);
void launch_tensor_scale_rows(bool f64, const void* col, const void* m, void* out, int rows, int cols,
                              cudaStream_t s);
void launch_tensor_sine(bool f64, const void* x, void* out, size_t n, double omega, bool derivative, cudaStream_t s);

// Tensor-core availability of a net for the fast mode (mlp_tc.cu).
bool tc_supported(const DevNet& n);

// Launch configuration of a kernel on the CURRENT device.  CUDA function attributes (the
// dynamic-SMEM opt-in above 48 KB, the carveout) are per device, so they are kept per
// (device, kernel) under a process-wide lock — the opt-in raised to the largest size any
// launch needed — and the occupancy per (threads, smem) is cached: contexts on several
// devices, and host threads racing on first use, each see a configured kernel.  err !=
// cudaSuccess when the opt-in failed (the caller reports it; nothing is cached then).
struct KernelCfg {
  cudaError_t err = cudaSuccess;
  int sms = 0;        // multiprocessors of the device
  int occupancy = 0;  // cudaOccupancyMaxActiveBlocksPerMultiprocessor
  int regs = 0;       // registers per thread
};
KernelCfg kernel_cfg(const void* kernel, int threads, size_t smem, bool max_carveout = false);
void reset_kernel_cfg();  // forget every cached configuration (the next launches redo the opt-in)
int device_sms();  // multiprocessors of the current device

// Checked-build violation records of the engine / tensor-core translation units (zero in the
// normal build); `reset` clears them.
cudaError_t check_report_engine(CheckRecord* out, bool reset);
cudaError_t check_report_tc(CheckRecord* out, bool reset);
cudaError_t launch_check_selftest(cudaStream_t s);  // one deliberate violation (positive control)

}  // namespace nsdf_b200
