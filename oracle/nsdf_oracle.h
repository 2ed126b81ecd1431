/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle of the parity suite.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the product
 * (libnsdf_cuda.so and the host library) never does.
 *
 * A plain-C restatement of the reference's f32 render path (AVX2 backend arithmetic),
 * operation for operation.  Pinned bit-for-bit against the reference library compiled
 * from /root/reference (oracle/_ref/libnsdf_ref.so) and its golden vectors by
 * tests/test_oracle.py.
 */
#ifndef NSDF_ORACLE_H_
#define NSDF_ORACLE_H_

#include <stdint.h>

#include "../include/nsdf_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* A field as the oracle sees it.  kind 0 = MLP (packed doubles as in nsdf_cuda.h,
 * cast to f32 on use like NeuralField, field.cpp:150), else nsdf_analytic_kind. */
typedef struct {
  int kind;
  int n_layers;
  const int32_t* rows;
  const int32_t* cols;
  const double* packed;
  int activation;
  double omega0;
  int input_dim;
  double analytic[4];
} orc_field;

typedef struct {
  orc_field field;
  float time;
  double delta;
} orc_level;

void orc_sincos(float x, float* s, float* c);
void orc_sine(const float* x, float* out, int64_t n, float omega, int derivative);

/* mode 0 fwd, 1 grad, 2 fused; points rows x k (rows = input_dim, or 3 + time). */
int orc_mlp(const orc_field* f, int mode, const float* points, int rows, int k, float time,
            float* dist, float* grad);
int orc_field_eval(const orc_field* f, const float* points, int k, float time, float* dist,
                   float* grad);

void orc_generate_rays(const nsdf_camera* cam, float* rays);
int orc_trace_rays(const orc_level* levels, int m, const nsdf_trace_config* cfg, const float* rays,
                   int64_t n, nsdf_hit_record* out);
int orc_normal_map(const orc_field* f, float time, const float* points, int k, double delta,
                   const float* fallback, float* normals, uint64_t* outside, uint64_t* fallbacks);
int orc_shade(const float* points, const float* normals, int k, const nsdf_shade_config* cfg,
              const nsdf_camera* cam, float* rgb);
int orc_render(const orc_level* levels, int m, const nsdf_camera* cam,
               const nsdf_trace_config* trace, const nsdf_shade_config* shade, int normal_source,
               int fine_index, float* rgb, float* depth, uint8_t* mask);
/* Render only rows [row_lo, row_hi) of the image (bounded CPU-baseline samples). */
int orc_render_rows(const orc_level* levels, int m, const nsdf_camera* cam,
                    const nsdf_trace_config* trace, const nsdf_shade_config* shade,
                    int normal_source, int fine_index, int row_lo, int row_hi, float* rgb,
                    float* depth, uint8_t* mask);

#ifdef __cplusplus
}
#endif
#endif
