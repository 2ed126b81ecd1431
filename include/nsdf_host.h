/*
 * nsdf_host.h — extern "C" entry points of libnsdf_b200.so, the drop-in C++ library that
 * re-implements the reference API (include/nsdf/*.hpp) over libnsdf_cuda.so.  These let a
 * C / ctypes caller drive the reference-shaped chain end to end:
 *   fields::load_manifest -> shading::render | tracer::trace_image | mlp::*_batch.
 * Return nsdf_status; nsdf_host_last_error() has the message.
 */
#ifndef NSDF_HOST_H_
#define NSDF_HOST_H_

#include "nsdf_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* nsdf_host_last_error(void);
int nsdf_host_render_manifest(const char* manifest, double time, const nsdf_camera* camera,
                              const nsdf_trace_config* trace, const nsdf_shade_config* shade,
                              int normal_source, int fine_index, float* rgb, float* depth,
                              uint8_t* mask);
/* The reference-shaped caller timed: shading::render(seq, cam, cfg) into a fresh ImageBuffer
 * (pageable, value-initialised), `warmup` untimed frames then the mean seconds per frame of
 * `repeats` frames — the `nsdf bench` row timing with a warm-up. */
int nsdf_host_bench_render(const char* manifest, double time, const nsdf_camera* camera,
                           const nsdf_trace_config* trace, const nsdf_shade_config* shade, int normal_source,
                           int fine_index, int warmup, int repeats, double* seconds_per_frame);
int nsdf_host_trace_image_manifest(const char* manifest, double time, const nsdf_camera* camera,
                                   const nsdf_trace_config* trace, nsdf_hit_record* out);
int nsdf_host_forward_and_gradient(const char* sdfnet, const float* points, int k, float* dist,
                                   float* grad);

/* The reference CLI flows (proj/tools/nsdf_main.cpp) over this library: argv[1] is
 * train | render | bench, followed by the reference's --flag value pairs.  Returns the
 * reference's exit code (0 ok, 1 usage/config, 2 validation, 3 divergence); tools/nsdf_b200
 * is a main() around it. */
int nsdf_host_cli(int argc, const char* const* argv);

/* Framebuffer output (shading::write_ppm / write_png / read_ppm, image.cpp:32-120): the
 * format follows the path's extension (.png, else binary PPM); rgb is 3 x W x H floats. */
int nsdf_host_write_image(const char* path, int width, int height, const float* rgb);
int nsdf_host_read_ppm(const char* path, int* width, int* height, float* rgb, size_t capacity);

/* Certification (fields::sample_near_surface / estimate_sup_diff / verify_nesting,
 * nesting.cpp:131-361) through the drop-in library; neural fields evaluate on the device
 * FP64 path.  A field source is "weights:<file.sdfnet>" or an analytic spec
 * ("torus:R=0.6,r=0.3").
 *   sample_near_surface: out = count x 3 doubles; gaussian != 0 selects gaussian noise.
 *   sup_diff: f's domain is set to g's; out = {eps, raw_max, argmax x, y, z, samples}.
 *   verify_nesting: counts = {samples_total, checked, violation_count, n_recorded};
 *                   recorded = n_recorded x {x, y, z, pair, f_coarse, f_fine}. */
int nsdf_host_sample_near_surface(const char* field, uint64_t count, int gaussian, double amount,
                                  uint64_t seed, double* out);
int nsdf_host_sup_diff(const char* f_src, const char* g_src, uint64_t n_uniform, uint64_t n_surface,
                       double margin, double noise_halfwidth, uint64_t seed, double* out);
int nsdf_host_verify_nesting(const char* manifest, double time, uint64_t samples, uint64_t seed,
                             uint64_t max_recorded, uint64_t* counts, double* recorded);

/* Training (trainer::sample_training_set / fit_mlp / backprop_sine_mlp) through the drop-in
 * library: sampling on the host, backprop and the fit loop on the device in FP64.
 *   sample: oracle source as above; points_out 3 x (n_uniform + n_surface), targets_out,
 *           val_points_out 3 x n_validation, val_targets_out.
 *   fit: arch "WxK" (parse_architecture); params_out has parameter_count() entries (packed
 *        per layer W then b); epoch_loss has cfg->epochs entries; report as nsdf_train_report.
 *   backprop: grads_out packed like params; *loss = mean squared error. */
int nsdf_host_sample_training_set(const char* oracle, uint64_t n_uniform, uint64_t n_surface, double sigma,
                                  uint64_t n_validation, uint64_t seed, double* points_out,
                                  double* targets_out, double* val_points_out, double* val_targets_out);
int nsdf_host_fit_mlp(const char* arch, int input_dim, double omega0, uint64_t seed,
                      const nsdf_train_config* cfg, const double* points, const double* targets, int n,
                      const double* val_points, const double* val_targets, int n_val, double* params_out,
                      double* epoch_loss, nsdf_train_report* report);
int nsdf_host_backprop(const char* arch, int input_dim, double omega0, uint64_t seed,
                       const double* points, const double* targets, int k, double* params_out,
                       double* grads_out, double* loss);

#ifdef __cplusplus
}
#endif

#endif /* NSDF_HOST_H_ */
