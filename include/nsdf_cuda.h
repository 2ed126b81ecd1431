/*
 * nsdf_cuda.h — the C ABI of libnsdf_cuda.so, the B200 (sm_100a) engine behind the
 * reference renderer's C++ API.
 *
 * This is the drop-in boundary: every entry point here replaces one C++ entry point
 * of the reference library (paths relative to /root/reference/proj):
 *
 *   nsdf_cuda_upload_mlp      NeuralField ctor, f64 master -> f32 copy   src/fields/field.cpp:149-154
 *                             NeuralTimeField ctor                      src/fields/field.cpp:256-261
 *   nsdf_cuda_upload_analytic SphereField / TorusField / BoxField       include/nsdf/fields/field.hpp:42-80
 *   nsdf_cuda_eval            mlp::forward_batch<float>                 src/mlp/mlp.cpp:171-177 (mlp.cpp:267-273)
 *                             Field::eval_batch(Matrix<float>)          src/fields/field.cpp:167-169, 303-305
 *   nsdf_cuda_grad            mlp::gradient_batch<float> /              src/mlp/mlp.cpp:275-295
 *                             spatial_gradient_batch<float>
 *                             Field::grad_batch(Matrix<float>)          src/fields/field.cpp:173-175, 309-311
 *   nsdf_cuda_eval_grad       mlp::forward_and_gradient_batch<float>    src/mlp/mlp.cpp:297-306
 *   nsdf_cuda_eval_f64        mlp::forward_batch / forward_and_gradient_batch / (spatial_)
 *                             gradient_batch<double>                    src/mlp/mlp.cpp:104-210
 *                             NeuralField / NeuralTimeField f64 batches src/fields/field.cpp:167-178, 301-311
 *                             (the certification path: nesting.cpp:131-361)
 *   nsdf_cuda_project_to_surface fields::sample_near_surface projection nesting.cpp:98-127
 *   nsdf_cuda_backprop_f64    trainer::backprop_sine_mlp                src/trainer/backprop.cpp:66-78
 *   nsdf_cuda_fit_mlp         trainer::fit_mlp (device-resident loop)   src/trainer/fit.cpp:87-196
 *   nsdf_cuda_generate_rays   tracer::generate_rays                     src/tracer/camera.cpp:20-43
 *   nsdf_cuda_trace_rays      tracer::multiscale_sphere_trace (batched) src/tracer/trace.cpp:86-132, 162-169
 *   nsdf_cuda_sphere_trace    tracer::sphere_trace                      src/tracer/trace.cpp:136-160
 *   nsdf_cuda_trace_image     tracer::trace_image                       src/tracer/trace.cpp:171-186
 *   nsdf_cuda_normal_map      shading::neural_normal_map                src/shading/shade.cpp:8-42
 *   nsdf_cuda_map_normals_to_mesh shading::map_normals_to_mesh          src/shading/mesh.cpp:122-156
 *   nsdf_cuda_shade           shading::shade                            src/shading/shade.cpp:44-93
 *   nsdf_cuda_render          shading::render                           src/shading/render.cpp:12-82
 *   nsdf_cuda_render_device   shading::render, device-resident framebuffer + tile sharding
 *                             (the multi-GPU frame/tile scheduler's per-rank call)
 *   nsdf_cuda_tensor_gemm     tensor::kernels::Table::gemm_f32 / gemm_f64, tensor::gemm
 *                             include/nsdf/tensor/kernels.hpp:26-29, src/tensor/ops.cpp:24-41
 *   nsdf_cuda_tensor_hadamard Table::hadamard_f32 / _f64, tensor::hadamard   kernels.hpp:31-32, ops.cpp:43-55
 *   nsdf_cuda_tensor_scale_rows Table::scale_rows_f32 / _f64, tensor::scale_rows kernels.hpp:34-36, ops.cpp:81-95
 *   nsdf_cuda_tensor_sine     Table::sine_f32 / _f64, tensor::activate (sine) kernels.hpp:38-39, ops.cpp:57-79
 *   nsdf_cuda_render_multi    shading::render over N contexts (N GPUs) from one process:
 *                             interleaved tiles per context, stored by each GPU straight into
 *                             the root GPU's framebuffer over NVLink (SURVEY.md §8b
 *                             "nsdf_cuda_render_multi(ctxs[], n, ...)")
 *   nsdf_cuda_replicate_field the once-per-sequence weight broadcast of the multi-GPU path
 *                             (device-to-device; NeuralField ctor on the other GPUs)
 *
 * Conventions
 *   - Plain C types only; no exceptions cross this boundary.  Every function returns an
 *     nsdf_status; on failure nsdf_cuda_last_error() (thread-local) holds the message and
 *     the host shim rethrows nsdf::Error with the matching ErrorKind (core.hpp:12-18).
 *   - Point batches keep the reference layout: `rows x k` row-major float, one point per
 *     column (matrix.hpp:32-33).  rows is the network input dim (3 or 4); a 3-row batch
 *     fed to a 4-input net gets the constant `time` row appended (field.cpp:213-220).
 *   - Functions without the _device suffix take HOST pointers and are synchronous.
 *     _device variants take device pointers and run asynchronously on the context stream.
 *   - A context is bound to one device and one stream; calls on one context are
 *     serialised by an internal mutex, so concurrent callers are safe.
 *   - No CPU fallback: if the device or the kernels are unavailable, calls fail loudly
 *     with NSDF_ERR_DEVICE.
 */
#ifndef NSDF_CUDA_H_
#define NSDF_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSDF_CUDA_ABI_VERSION 2
#define NSDF_MAX_LEVELS 8 /* tracer::kMaxLevels, trace.hpp:32 */
#define NSDF_MAX_LIGHTS 8

typedef enum {
  NSDF_OK = 0,
  NSDF_ERR_CONTRACT = 1,   /* ErrorKind::contract   — shape / precondition violation   */
  NSDF_ERR_CONFIG = 2,     /* ErrorKind::config     — bad configuration value          */
  NSDF_ERR_VALIDATION = 3, /* ErrorKind::validation — inconsistent data                */
  NSDF_ERR_PARSE = 4,      /* ErrorKind::parse                                         */
  NSDF_ERR_DIVERGENCE = 5, /* ErrorKind::divergence                                    */
  NSDF_ERR_DEVICE = 6      /* CUDA failure / no device; the host shim maps to validation */
} nsdf_status;

/* Arithmetic mode of the MLP evaluator.
 *   FP32_ORACLE: FFMA kernels that restate the reference AVX2 arithmetic operation for
 *                operation (k-sequential fma chains from the bias, Cephes sincos with
 *                separately rounded mul/add) — bit-exact with the reference CPU path.
 *   FP16_FAST:   tcgen05 tensor-core tiles with split-fp16 operands (A_hi.W_hi +
 *                A_lo.W_hi + A_hi.W_lo, fp32 TMEM accumulators; for 128/256-wide nets at
 *                omega0 <= 15 the two correction terms run as one E4M3 MMA, and stop
 *                decisions near eps_stop are re-decided with fp16 terms — env
 *                NSDF_TC_E4M3=0/1 at upload overrides), fp32 first/output layers,
 *                range-reduced MUFU sine; |df| ~1e-5, parity within the BASELINE
 *                tolerances (mask >= 99.9%, |dt| <= 1e-3, normals <= 0.5 deg).
 *   FP16_LOW:    the same tiles with plain fp16 operands (one MMA per K step); fastest,
 *                |df| up to ~1e-3 at omega0 = 30 (depth p99.9 ~1.5e-3: outside tolerance). */
typedef enum { NSDF_MODE_FP32_ORACLE = 0, NSDF_MODE_FP16_FAST = 1, NSDF_MODE_FP16_LOW = 2 } nsdf_mode;

typedef enum { NSDF_ACT_SINE = 0, NSDF_ACT_IDENTITY = 1 } nsdf_activation; /* ops.hpp Activation */
typedef enum { NSDF_FIELD_SPHERE = 1, NSDF_FIELD_TORUS = 2, NSDF_FIELD_BOX = 3 } nsdf_analytic_kind;
typedef enum { NSDF_NORMALS_OWN = 0, NSDF_NORMALS_MAPPED = 1 } nsdf_normal_source; /* shading.hpp:113 */

typedef struct nsdf_ctx nsdf_ctx;
typedef int32_t nsdf_field; /* handle > 0 */

/* tracer::Camera (trace.hpp:13-22) */
typedef struct {
  double position[3];
  double look_at[3];
  double up[3];
  double vertical_fov_deg;
  int32_t width;
  int32_t height;
} nsdf_camera;

/* tracer::TraceConfig (trace.hpp:49-55); n_levels must equal the sequence size */
typedef struct {
  int32_t n_levels;
  int32_t budgets[NSDF_MAX_LEVELS];
  float eps_stop;
  float t_max;
} nsdf_trace_config;

/* tracer::HitRecord (trace.hpp:34-47) */
typedef struct {
  int32_t hit;
  float point[3];
  float t;
  int32_t level_reached;
  uint16_t iterations_used[NSDF_MAX_LEVELS];
  float final_distance;
} nsdf_hit_record;

/* shading::ShadeConfig / Material / DirectionalLight (shading.hpp:90-107) */
typedef struct {
  float albedo[3];
  float ambient;
  float diffuse;
  float specular;
  float shininess;
  int32_t n_lights;
  float light_direction[NSDF_MAX_LIGHTS][3];
  float light_intensity[NSDF_MAX_LIGHTS];
  float background[3];
} nsdf_shade_config;

/* One member of a nested sequence, coarse to fine (nesting.hpp:53-61).  `time` is the
 * slice time for 4-input nets (AnimatedSequence::slice, nesting.cpp:71-78), ignored
 * otherwise.  `delta` is the nesting threshold deltas[j]. */
typedef struct {
  nsdf_field field;
  float time;
  double delta;
} nsdf_level;

/* Per-frame accounting, filled by render/trace when non-NULL (the FLOP source of
 * iterations_used summed per level, hits, normal evaluations). */
typedef struct {
  uint64_t evals[NSDF_MAX_LEVELS]; /* MLP forward evaluations per level           */
  uint64_t hits;                   /* rays that converged at the final level       */
  uint64_t normal_evals;           /* fwd+gradient evaluations for normals         */
  uint64_t fallback_evals;         /* own-field normals computed for the fallback  */
  uint64_t kernel_launches;        /* engine kernels launched for the frame        */
  /* Which kernel family ran each part of the frame (nsdf_kernel_path).  A fast-mode frame
   * whose MLP levels do not all report NSDF_PATH_TCGEN05 did not run on the tensor cores;
   * a failed tcgen05 launch is an error (NSDF_ERR_DEVICE), never a silent FFMA fallback. */
  uint8_t level_path[NSDF_MAX_LEVELS]; /* per traced level; NSDF_PATH_NONE if skipped    */
  uint8_t normals_path;                /* the normal + shade tiles of the hit list      */
  uint8_t fallback_path;               /* own-field fallback normals (mapped mode)      */
  uint8_t reserved_[6];
} nsdf_frame_stats;

/* Kernel families reported in nsdf_frame_stats. */
typedef enum {
  NSDF_PATH_NONE = 0,    /* not run                                                       */
  NSDF_PATH_SIMT = 1,    /* FFMA tiles (FP32 oracle mode, analytic fields, other widths)  */
  NSDF_PATH_TCGEN05 = 2  /* tcgen05 tensor-core tiles (persistent level / normal tiles)   */
} nsdf_kernel_path;

/* Per-kernel-family device time (CUDA events on the context stream), accumulated over
 * frames while profiling is enabled — the "CUDA events per level and per frame" of
 * SURVEY.md §5.  Reading it synchronizes the stream. */
typedef struct {
  double level_ms[NSDF_MAX_LEVELS]; /* trace kernels (MLP tiles) per level             */
  double normals_ms;                /* fused normal + shade kernels                     */
  double frame_ms;                  /* whole frames (rays .. framebuffer)              */
  uint64_t frames;
  uint64_t trace_launches;
  uint64_t normal_launches;
} nsdf_profile;

/* SIREN training (trainer::TrainConfig minus the architecture / omega0 / seed, which the
 * caller applies through random_init, trainer.hpp:50-70) and its report (TrainReport). */
typedef struct {
  int epochs;
  int batch_size;           /* 0 = full batch */
  double learning_rate;     /* peak rate after warmup */
  double momentum;
  int warmup_epochs;
  int plateau_patience;
  double plateau_threshold;
  double min_learning_rate;
} nsdf_train_config;

typedef struct {
  double final_loss;
  double validation_mse;
  double validation_max_error;
  double final_learning_rate;
  int diverged;
  int halvings;
  int epochs_recorded;      /* entries written to epoch_loss */
} nsdf_train_report;

/* ---- context ---------------------------------------------------------------------- */
int nsdf_cuda_abi_version(void);
const char* nsdf_cuda_last_error(void);
/* Diagnostics: the fast mode's activation exactly as its tile epilogues evaluate it —
 * sin(x) and sin(x + pi/2) on the MUFU pipe (sin.approx: FMUL.RZ by 1/2pi reduces the
 * argument to revolutions, MUFU.SIN evaluates the fraction) — for x[0..n) (host buffers).
 * tests/test_gpu_fast.py bounds its error at the largest omega0 * z the fixtures produce. */
int nsdf_cuda_probe_fast_sine(nsdf_ctx* ctx, const float* x, int n, float* sin_out, float* cos_out);
/* Checked build (libnsdf_cuda.so built with NSDF_CHECKED=1, paper_2201_09147_b200/_checked/):
 * the number of out-of-bounds list indices, ray slots, staged appends and framebuffer pixels
 * the device kernels detected (and skipped) since the last reset, with the first one's site
 * (1 list read, 2 slot, 3 CTA staging, 4 list write, 5 pixel), value and bound;
 * *checked_build = 0 and *count = 0 in the normal build.  Synchronizes the context stream. */
int nsdf_cuda_check_report(nsdf_ctx* ctx, int reset, uint64_t* count, int32_t* site, int32_t* value,
                           int32_t* bound, int32_t* checked_build);
/* Positive control for the checked build: one deliberate out-of-bounds check on the device
 * (count + 1 in the checked build, no effect otherwise). */
int nsdf_cuda_check_selftest(nsdf_ctx* ctx);
/* Diagnostics: forget the per-(device, kernel) launch configuration (the dynamic-SMEM opt-in
 * and occupancy), so the next launch on every device takes the configuration path again —
 * how a test exercises the per-device setup on a one-GPU box. */
int nsdf_cuda_reset_kernel_config(void);
/* Number of visible CUDA devices (NSDF_ERR_DEVICE when there is none). */
int nsdf_cuda_device_count(int* n);
int nsdf_cuda_create(int device, nsdf_ctx** out);
int nsdf_cuda_destroy(nsdf_ctx* ctx);
int nsdf_cuda_set_mode(nsdf_ctx* ctx, int mode);
int nsdf_cuda_get_mode(nsdf_ctx* ctx, int* mode);
/* Bind the context to an existing cudaStream_t (NULL restores the context's own). */
int nsdf_cuda_set_stream(nsdf_ctx* ctx, void* stream);
int nsdf_cuda_synchronize(nsdf_ctx* ctx);
/* Device memory shared between the processes of one node (the multi-GPU scheduler's peer
 * framebuffer: every rank's shading kernels store their tile pixels straight into rank 0's
 * framebuffer over NVLink).  alloc/free: cudaMalloc on the context's device; ipc_export:
 * a 64-byte cudaIpcMemHandle of an nsdf_cuda_alloc pointer; ipc_open: map it in this process
 * (peer access enabled lazily); memcpy: any direction (cudaMemcpyDefault), synchronous on
 * the context stream. */
int nsdf_cuda_alloc(nsdf_ctx* ctx, size_t bytes, void** out);
int nsdf_cuda_free(nsdf_ctx* ctx, void* ptr);
int nsdf_cuda_ipc_export(nsdf_ctx* ctx, void* ptr, uint8_t* handle64);
int nsdf_cuda_ipc_open(nsdf_ctx* ctx, const uint8_t* handle64, void** out);
int nsdf_cuda_ipc_close(nsdf_ctx* ctx, void* ptr);
int nsdf_cuda_memcpy(nsdf_ctx* ctx, void* dst, const void* src, size_t bytes);
/* Enable / disable per-kernel-family CUDA-event timing (resets the accumulators). */
int nsdf_cuda_set_profiling(nsdf_ctx* ctx, int enable);
int nsdf_cuda_get_profile(nsdf_ctx* ctx, nsdf_profile* out);

/* ---- fields -------------------------------------------------------------------------
 * Packed weights: for each layer l, rows[l]*cols[l] row-major weights (out x in) then
 * rows[l] biases, as doubles (the f64 master of NeuralField).  The engine keeps the f32
 * cast (field.cpp:150) for the oracle mode and fp16 tiles for the fast mode.
 * Validation follows MlpParams::validate (mlp.cpp:13-39). */
int nsdf_cuda_upload_mlp(nsdf_ctx* ctx, int n_layers, const int32_t* rows, const int32_t* cols,
                         const double* packed, int activation, double omega0, int input_dim,
                         nsdf_field* out);
/* sphere: {cx, cy, cz, r}; torus: {R, r}; box: {hx, hy, hz} (field.hpp:42-80) */
int nsdf_cuda_upload_analytic(nsdf_ctx* ctx, int kind, const double* params, int n_params,
                              nsdf_field* out);
int nsdf_cuda_release(nsdf_ctx* ctx, nsdf_field field);
/* Weight broadcast for multi-GPU rendering: copies field `field` of `src` (its packed device
 * image: f32/f64 weights and the fp16 tensor-core copy, one allocation) to `dst`'s device
 * with one device-to-device peer copy (NVLink), no host round trip; *out is the handle in
 * dst.  The replica evaluates bit-identically to the source. */
int nsdf_cuda_replicate_field(nsdf_ctx* src, nsdf_field field, nsdf_ctx* dst, nsdf_field* out);
int nsdf_cuda_field_info(nsdf_ctx* ctx, nsdf_field field, int* input_dim, int* n_layers,
                         int* width);

/* Certification: the projection step of fields::sample_near_surface (nesting.cpp:98-127)
 * with the points resident on the device — `steps` Newton steps p -= f/|g|^2 g (skipped
 * where |g|^2 < 1e-16) from n candidates (Vec3 array, n <= 2^20), then the points with
 * |f| <= keep_tol, in input order, with the field's gradient there (Vec3 arrays); FP64,
 * bit-identical to the reference's double path.  Replaces 4 x (eval + grad) host round trips
 * per round with one H2D and one D2H. */
int nsdf_cuda_project_to_surface(nsdf_ctx* ctx, nsdf_field field, double time, const double* candidates,
                                 int n, double keep_tol, int steps, double* kept, double* kept_grads,
                                 int* n_kept);

/* ---- batch evaluation (Field::eval_batch / grad_batch, mlp::*_batch) ------------------
 * points: rows x k; out: 1 x k; grad: 3 x k.  Either output may be NULL in eval_grad. */
int nsdf_cuda_eval(nsdf_ctx* ctx, nsdf_field field, const float* points, int rows, int k,
                   float time, float* out);
int nsdf_cuda_grad(nsdf_ctx* ctx, nsdf_field field, const float* points, int rows, int k,
                   float time, float* grad);
int nsdf_cuda_eval_grad(nsdf_ctx* ctx, nsdf_field field, const float* points, int rows, int k,
                        float time, float* out, float* grad);
int nsdf_cuda_eval_grad_device(nsdf_ctx* ctx, nsdf_field field, const float* d_points, int rows,
                               int k, float time, float* d_out, float* d_grad);
/* FP64 evaluation of a neural field, bit-exact with the reference's double AVX2 path
 * (certification: estimate_sup_diff / verify_nesting / sample_near_surface).  points:
 * rows x k doubles (HOST); out: k or NULL; grad: 3 x k or NULL (not both NULL).  A 3-row
 * batch for a 4-input net gets the constant `time` row (double, field.cpp:213-220).
 * Sphere / torus / box fields evaluate in double exactly as field.cpp:57-124 (glibc hypot
 * restated for the torus). */
int nsdf_cuda_eval_f64(nsdf_ctx* ctx, nsdf_field field, const double* points, int rows, int k,
                       double time, double* out, double* grad);

/* ---- the reference's dense kernel table on the device ---------------------------------
 * HOST buffers, row-major; dtype NSDF_DTYPE_F32 (float) or NSDF_DTYPE_F64 (double).
 * Bit-exact with the reference's AVX2 backend (kernels_avx2.cpp): gemm c[m x n] = a[m x k] .
 * b[k x n] (+ bias[m], may be NULL), each output one k-sequential fma chain from the bias (or
 * 0); hadamard out = a * b (n elements); scale_rows out[i,j] = col[i] * m[i,j]; sine out =
 * sin(omega*x), or omega*cos(omega*x) when derivative != 0 (f32: omega rounded to float).
 * Shape checks are the caller's (tensor::gemm etc. in the drop-in library throw the
 * reference's contract errors). */
#define NSDF_DTYPE_F32 0
#define NSDF_DTYPE_F64 1
int nsdf_cuda_tensor_gemm(nsdf_ctx* ctx, int dtype, const void* a, const void* b, const void* bias, void* c,
                          int m, int n, int k);
int nsdf_cuda_tensor_hadamard(nsdf_ctx* ctx, int dtype, const void* a, const void* b, void* out, size_t n);
int nsdf_cuda_tensor_scale_rows(nsdf_ctx* ctx, int dtype, const void* col, const void* m, void* out, int rows,
                                int cols);
int nsdf_cuda_tensor_sine(nsdf_ctx* ctx, int dtype, const void* x, void* out, size_t n, double omega,
                          int derivative);

/* ---- training (FP64, bit-exact with the reference trainer) ----------------------------
 * Packed parameters as in nsdf_cuda_upload_mlp.  backprop: trainer::backprop_sine_mlp
 * (backprop.cpp:66-78) — grads packed like the parameters, loss = mean squared error.
 * fit: trainer::fit_mlp (fit.cpp:87-196) from caller-initialised parameters (random_init)
 * and the caller's Rng state after it (xoshiro256++ s[4], core.hpp:75-118; advanced by the
 * epoch shuffles); params returns the checkpoint; epoch_loss holds cfg->epochs entries. */
int nsdf_cuda_backprop_f64(nsdf_ctx* ctx, int n_layers, const int32_t* rows, const int32_t* cols,
                           const double* packed, int activation, double omega0, int input_dim,
                           const double* points, const double* targets, int k, double* grads,
                           double* loss);
int nsdf_cuda_fit_mlp(nsdf_ctx* ctx, int n_layers, const int32_t* rows, const int32_t* cols,
                      double* packed, int activation, double omega0, int input_dim,
                      uint64_t* rng_state, const double* points, const double* targets, int n,
                      const double* val_points, const double* val_targets, int n_val,
                      const nsdf_train_config* config, double* epoch_loss,
                      nsdf_train_report* report);

/* ---- tracing --------------------------------------------------------------------------
 * rays: n x 6 floats {ox, oy, oz, dx, dy, dz} (tracer::Ray, trace.hpp:24-27). */
int nsdf_cuda_generate_rays(nsdf_ctx* ctx, const nsdf_camera* camera, float* rays);
int nsdf_cuda_trace_rays(nsdf_ctx* ctx, const nsdf_level* levels, int m,
                         const nsdf_trace_config* config, const float* rays, int n,
                         nsdf_hit_record* out);
/* Classic sphere tracing of one field's delta-offset level set (tracer::sphere_trace,
 * trace.cpp:136-160): a single final level with fd = f - delta, two-sided convergence. */
int nsdf_cuda_sphere_trace(nsdf_ctx* ctx, nsdf_field field, float time, float delta, float eps_stop,
                           int max_iters, float t_max, const float* rays, int n, nsdf_hit_record* out);
int nsdf_cuda_trace_image(nsdf_ctx* ctx, const nsdf_level* levels, int m,
                          const nsdf_camera* camera, const nsdf_trace_config* config,
                          nsdf_hit_record* out, nsdf_frame_stats* stats);

/* ---- normals and shading -------------------------------------------------------------- */
int nsdf_cuda_normal_map(nsdf_ctx* ctx, nsdf_field fine, float time, const float* points, int k,
                         double delta, const float* fallback_normals, float* normals,
                         uint64_t* outside_count, uint64_t* fallback_count);
/* shading::map_normals_to_mesh (mesh.cpp:122-156) on the device: vertices k x 3 doubles (the
 * Mesh::vertices Vec3 array), normals k x 3 doubles — in: the normals kept for violators and
 * zero-gradient vertices (the mesh's own, or zeros), out: g/|g| (double) for mapped
 * vertices; counts = {mapped, violators, fallbacks}.  The caller replaces the mesh normals
 * only if mapped > 0, as the reference does.  Synchronous. */
int nsdf_cuda_map_normals_to_mesh(nsdf_ctx* ctx, nsdf_field fine, float time, const double* vertices,
                                  int k, double delta, double* normals, uint64_t* counts);
/* Device-pointer variant (async): points/normals/fallback 3 x k, counts = 2 x u64
 * {outside, fallback} accumulated (zero them first).  Used for mesh G-buffers. */
int nsdf_cuda_normal_map_device(nsdf_ctx* ctx, nsdf_field fine, float time, const float* d_points,
                                int k, double delta, const float* d_fallback_normals,
                                float* d_normals, uint64_t* d_counts);
/* G-buffer of a triangle mesh (BASELINE config 4; the reference has no rasterizer): the
 * nearest hit of every camera ray (generate_rays pixel centres) against the triangles,
 * written as positions 3 x (W*H) (device) and a 0/1 mask (device).  Deterministic. */
int nsdf_cuda_raycast_mesh(nsdf_ctx* ctx, const nsdf_camera* camera, const float* vertices,
                           int n_vertices, const int32_t* triangles, int n_triangles,
                           float* d_positions, uint8_t* d_mask);
int nsdf_cuda_shade(nsdf_ctx* ctx, const float* points, const float* normals, int k,
                    const nsdf_shade_config* config, const nsdf_camera* camera, float* rgb);

/* ---- whole frame ------------------------------------------------------------------------
 * rgb: 3*W*H, depth: W*H, mask: W*H (ImageBuffer, shading.hpp:22-34).  fine_index < 0
 * selects the finest member (RenderConfig::mapped_fine_index). */
int nsdf_cuda_render(nsdf_ctx* ctx, const nsdf_level* levels, int m, const nsdf_camera* camera,
                     const nsdf_trace_config* trace, const nsdf_shade_config* shade,
                     int normal_source, int fine_index, float* rgb, float* depth, uint8_t* mask,
                     nsdf_frame_stats* stats);
/* The same frame in two calls: begin validates and enqueues the whole frame into the
 * context's device framebuffer and returns at once; end (synchronous) copies it into the
 * caller's HOST buffers — so a caller can allocate and zero its framebuffer (the reference's
 * ImageBuffer is value-initialised std::vector storage) while the GPU renders.  One frame in
 * flight per context; end reports the frame's errors (e.g. the deferred light check). */
int nsdf_cuda_render_begin(nsdf_ctx* ctx, const nsdf_level* levels, int m, const nsdf_camera* camera,
                           const nsdf_trace_config* trace, const nsdf_shade_config* shade,
                           int normal_source, int fine_index);
int nsdf_cuda_render_end(nsdf_ctx* ctx, float* rgb, float* depth, uint8_t* mask, nsdf_frame_stats* stats);
/* Device framebuffer variant used by the frame/tile scheduler: renders the pixels of the
 * image tiles t with t % tile_world == tile_rank (tile_size x tile_size tiles, row-major
 * tile order; tile_world = 1 renders everything) into full-frame device buffers.  Pixels
 * of other tiles are left untouched.  Asynchronous on the context stream; `stats` (host,
 * may be NULL) forces a synchronize. */
/* Explicit tile ownership for the tile-sharded renders (nsdf_cuda_render_device with
 * tile_world > 1): owners[t] is the tile_rank that renders tile t (row-major tiles of
 * tile_size) instead of t % tile_world — e.g. a cost-balanced assignment from a previous
 * frame's per-tile work (scheduler.balanced_tile_owners).  The map must cover exactly the
 * frame's tiles (else NSDF_ERR_CONFIG at render); n_tiles = 0 restores t % tile_world.
 * Synchronizes the context stream. */
int nsdf_cuda_set_tile_owners(nsdf_ctx* ctx, const int32_t* owners, int n_tiles);
/* Single-process multi-GPU render: context i (its own device and stream) renders the image
 * tiles t % n == i (tile_size x tile_size, row-major tile order) with its own field handles
 * levels[i][0..m) (nsdf_cuda_replicate_field copies ctxs[0]'s weights device to device).
 * The framebuffer lives on ctxs[0]'s device: every context's background and shading
 * kernels store their pixels straight into it over NVLink (peer access, enabled on first
 * use); device pairs that cannot be peers pack their pixels, peer-copy them and scatter on
 * ctxs[0]'s device.  No host scatter: one D2H of the assembled frame into the caller's HOST
 * framebuffer (synchronous).  The contexts render concurrently (cross-device events, no
 * host synchronisation between them); the image equals nsdf_cuda_render's for any n
 * (per-ray work does not depend on the partition).  stats (optional) sums the contexts'
 * counters; a level's path is NSDF_PATH_TCGEN05 only if every context ran it there. */
int nsdf_cuda_render_multi(nsdf_ctx* const* ctxs, int n, const nsdf_level* const* levels, int m,
                           const nsdf_camera* camera, const nsdf_trace_config* trace,
                           const nsdf_shade_config* shade, int normal_source, int fine_index,
                           int tile_size, float* rgb, float* depth, uint8_t* mask,
                           nsdf_frame_stats* stats);
int nsdf_cuda_render_device(nsdf_ctx* ctx, const nsdf_level* levels, int m,
                            const nsdf_camera* camera, const nsdf_trace_config* trace,
                            const nsdf_shade_config* shade, int normal_source, int fine_index,
                            int tile_size, int tile_rank, int tile_world, float* d_rgb,
                            float* d_depth, uint8_t* d_mask, nsdf_frame_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* NSDF_CUDA_H_ */
