/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the parity suite (see nsdf_oracle.h).
 *
 * Plain-C restatement of the reference's float render path.  Built with
 * -ffp-contract=off (as the reference, proj/CMakeLists.txt:15) so every a*b+c below is
 * a separately rounded multiply and add; the only fused operations are the explicit
 * fmaf() calls that mirror _mm256_fmadd_ps in the AVX2 GEMM.  Citations are to
 * /root/reference/proj.
 *
 * Parity status: pinned bit-for-bit to the reference library (oracle/_ref/libnsdf_ref.so,
 * AVX2 backend) by tests/test_oracle.py — forward, gradient, rays, trace records,
 * normals and whole renders — and to the reference's own KATs (tests/golden/).
 */
#include "nsdf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------
 * sin / cos: Cephes scheme of src/tensor/sincos_poly.hpp:13-22 (constants) and
 * eval_scalar (sincos_poly.hpp:90-133), which replicates the AVX2 lanes
 * (kernels_avx2.cpp:203-257) operation for operation.
 * --------------------------------------------------------------------------------- */
static const float kFourOverPi = 1.27323954473516f;
static const float kDp1 = -0.78515625f;
static const float kDp2 = -2.4187564849853515625e-4f;
static const float kDp3 = -3.77489497744594108e-8f;
static const float kSin0 = -1.9515295891e-4f;
static const float kSin1 = 8.3321608736e-3f;
static const float kSin2 = -1.6666654611e-1f;
static const float kCos0 = 2.443315711809948e-5f;
static const float kCos1 = -1.388731625493765e-3f;
static const float kCos2 = 4.166664568298827e-2f;

static inline uint32_t f2u(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
static inline float u2f(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

void orc_sincos(float x, float* s, float* c) {
  uint32_t bits = f2u(x);
  uint32_t sign_sin = bits & 0x80000000u;
  float ax = u2f(bits & 0x7fffffffu);
  float y = ax * kFourOverPi;
  int32_t q = (int32_t)y; /* cvttps: truncation */
  q = (q + 1) & ~1;
  y = (float)q;
  uint32_t swap_sign = (uint32_t)(q & 4) << 29;
  int poly_sin = (q & 2) == 0;
  float r = ax;
  r = r + y * kDp1;
  r = r + y * kDp2;
  r = r + y * kDp3;
  float z = r * r;
  float pc = kCos0;
  pc = pc * z + kCos1;
  pc = pc * z + kCos2;
  pc = pc * z * z;
  pc = pc - z * 0.5f;
  pc = pc + 1.0f;
  float ps = kSin0;
  ps = ps * z + kSin1;
  ps = ps * z + kSin2;
  ps = ps * z * r;
  ps = ps + r;
  float ysin = poly_sin ? ps : pc;
  ysin = u2f(f2u(ysin) ^ sign_sin ^ swap_sign);
  int32_t qc = q - 2;
  uint32_t cos_sign = (uint32_t)(~qc & 4) << 29;
  int cos_poly_sin = (qc & 2) == 0;
  float ycos = cos_poly_sin ? ps : pc;
  ycos = u2f(f2u(ycos) ^ cos_sign);
  *s = ysin;
  *c = ycos;
}

/* sine_f32_avx2 (kernels_avx2.cpp:259-275): arg = omega*x rounded first. */
void orc_sine(const float* x, float* out, int64_t n, float omega, int derivative) {
  for (int64_t i = 0; i < n; ++i) {
    float s, c;
    orc_sincos(omega * x[i], &s, &c);
    out[i] = derivative ? omega * c : s;
  }
}

/* ---------------------------------------------------------------------------------
 * MLP: evaluate_network (src/mlp/mlp.cpp:104-167), one column at a time (the
 * per-column arithmetic does not depend on the batch, kernels_avx2.cpp:1-4).
 * GEMM element: acc = bias (or 0); acc = fma(a[i,kk], b[kk,j], acc), kk ascending
 * (kernels_avx2.cpp:30-54, tail :78-86).
 * --------------------------------------------------------------------------------- */
typedef struct {
  int n_layers, input_dim, activation, max_width;
  float omega;
  const int32_t* rows;
  const int32_t* cols;
  float** w; /* f32 casts, field.cpp:150 */
  float** b;
} orc_net;

static int net_init(orc_net* net, const orc_field* f) {
  net->n_layers = f->n_layers;
  net->input_dim = f->input_dim;
  net->activation = f->activation;
  net->omega = (float)f->omega0;
  net->rows = f->rows;
  net->cols = f->cols;
  net->w = (float**)calloc((size_t)f->n_layers, sizeof(float*));
  net->b = (float**)calloc((size_t)f->n_layers, sizeof(float*));
  net->max_width = f->input_dim;
  size_t off = 0;
  for (int l = 0; l < f->n_layers; ++l) {
    size_t nw = (size_t)f->rows[l] * (size_t)f->cols[l];
    net->w[l] = (float*)malloc(nw * sizeof(float));
    net->b[l] = (float*)malloc((size_t)f->rows[l] * sizeof(float));
    for (size_t i = 0; i < nw; ++i) net->w[l][i] = (float)f->packed[off + i];
    off += nw;
    for (int i = 0; i < f->rows[l]; ++i) net->b[l][i] = (float)f->packed[off + i];
    off += (size_t)f->rows[l];
    if (f->rows[l] > net->max_width) net->max_width = f->rows[l];
  }
  return 0;
}

static void net_free(orc_net* net) {
  for (int l = 0; l < net->n_layers; ++l) {
    free(net->w[l]);
    free(net->b[l]);
  }
  free(net->w);
  free(net->b);
}

/* out[i] = (bias ? bias[i] : 0) + sum_kk W[i,kk] x[kk], as a k-sequential fma chain. */
static void gemv(const float* W, const float* bias, const float* x, int m, int k, float* out) {
  for (int i = 0; i < m; ++i) {
    float acc = bias ? bias[i] : 0.0f;
    const float* wr = W + (size_t)i * (size_t)k;
    for (int kk = 0; kk < k; ++kk) acc = fmaf(wr[kk], x[kk], acc);
    out[i] = acc;
  }
}

/* One column of evaluate_network with gradient_coords = 3 when grad != NULL. */
static void net_column(const orc_net* net, const float* x_in, float* dist, float* grad,
                       float* scratch) {
  const int L = net->n_layers;
  const int W = net->max_width;
  if (L == 1) { /* mlp.cpp:115-126 */
    if (dist) gemv(net->w[0], net->b[0], x_in, 1, net->cols[0], dist);
    if (grad)
      for (int c = 0; c < 3; ++c) grad[c] = net->w[0][c];
    return;
  }
  float* cur = scratch;          /* W */
  float* pre = cur + W;          /* W */
  float* dphi = pre + W;         /* W */
  float* G = dphi + W;           /* 3 x W */
  float* Gn = G + 3 * W;         /* 3 x W */
  memcpy(cur, x_in, sizeof(float) * (size_t)net->input_dim);
  for (int li = 0; li < L; ++li) {
    const int m = net->rows[li], k = net->cols[li];
    const float* Wl = net->w[li];
    if (li + 1 == L) { /* mlp.cpp:129-135 */
      if (grad)
        for (int c = 0; c < 3; ++c) gemv(Wl, NULL, G + c * W, 1, k, grad + c);
      if (dist) gemv(Wl, net->b[li], cur, 1, k, dist);
      break;
    }
    gemv(Wl, net->b[li], cur, m, k, pre); /* mlp.cpp:137 */
    if (grad) {
      for (int i = 0; i < m; ++i) { /* activate(derivative) mlp.cpp:139 */
        if (net->activation == NSDF_ACT_SINE) {
          float s, c;
          orc_sincos(net->omega * pre[i], &s, &c);
          dphi[i] = net->omega * c;
        } else {
          dphi[i] = 1.0f;
        }
      }
      if (li == 0) { /* scale_rows, mlp.cpp:140-145; kernels_avx2.cpp:166-176 */
        for (int c = 0; c < 3; ++c)
          for (int i = 0; i < m; ++i) G[c * W + i] = Wl[(size_t)i * (size_t)k + c] * dphi[i];
      } else { /* hadamard(gemm(W, G), dphi), mlp.cpp:146-148 */
        for (int c = 0; c < 3; ++c) {
          gemv(Wl, NULL, G + c * W, m, k, Gn + c * W);
          for (int i = 0; i < m; ++i) Gn[c * W + i] = Gn[c * W + i] * dphi[i];
        }
        float* t = G;
        G = Gn;
        Gn = t;
      }
    }
    for (int i = 0; i < m; ++i) { /* activate(value), mlp.cpp:153-154 */
      if (net->activation == NSDF_ACT_SINE) {
        float s, c;
        orc_sincos(net->omega * pre[i], &s, &c);
        cur[i] = s;
      } else {
        cur[i] = pre[i];
      }
    }
  }
}

int orc_mlp(const orc_field* f, int mode, const float* points, int rows, int k, float time,
            float* dist, float* grad) {
  if (f->kind != 0) return NSDF_ERR_CONTRACT;
  if (rows != f->input_dim && !(rows == 3 && f->input_dim == 4)) return NSDF_ERR_CONTRACT;
  orc_net net;
  net_init(&net, f);
  float* scratch = (float*)malloc(sizeof(float) * 9 * (size_t)net.max_width + 64);
  float x[4];
  for (int j = 0; j < k; ++j) {
    for (int r = 0; r < f->input_dim; ++r)
      x[r] = r < rows ? points[(size_t)r * (size_t)k + j] : time; /* with_time_row, field.cpp:213-220 */
    float d = 0, g[3] = {0, 0, 0};
    net_column(&net, x, mode == 1 ? NULL : &d, mode == 0 ? NULL : g, scratch);
    if (mode != 1) dist[j] = d;
    if (mode != 0)
      for (int c = 0; c < 3; ++c) grad[(size_t)c * (size_t)k + j] = g[c];
  }
  free(scratch);
  net_free(&net);
  return 0;
}

/* ---------------------------------------------------------------------------------
 * Analytic fields: double eval, cast to float (Field::eval_batch default,
 * field.cpp:11-29; shapes field.cpp:57-124).
 * --------------------------------------------------------------------------------- */
static double an_eval(const orc_field* f, double x, double y, double z) {
  const double* a = f->analytic;
  if (f->kind == NSDF_FIELD_SPHERE) {
    double dx = x - a[0], dy = y - a[1], dz = z - a[2];
    return sqrt(dx * dx + dy * dy + dz * dz) - a[3];
  }
  if (f->kind == NSDF_FIELD_TORUS) {
    double s = hypot(x, z);
    return hypot(s - a[0], y) - a[1];
  }
  double qx = fabs(x) - a[0], qy = fabs(y) - a[1], qz = fabs(z) - a[2];
  double px = fmax(qx, 0.0), py = fmax(qy, 0.0), pz = fmax(qz, 0.0);
  double outside = sqrt(px * px + py * py + pz * pz);
  double inside = fmin(fmax(qx, fmax(qy, qz)), 0.0);
  return outside + inside;
}

static double sgn(double v) { return v < 0 ? -1.0 : 1.0; }

static void an_grad(const orc_field* f, double x, double y, double z, double* g) {
  const double* a = f->analytic;
  g[0] = g[1] = g[2] = 0;
  if (f->kind == NSDF_FIELD_SPHERE) {
    double dx = x - a[0], dy = y - a[1], dz = z - a[2];
    double n = sqrt(dx * dx + dy * dy + dz * dz);
    if (n == 0) return;
    g[0] = dx / n;
    g[1] = dy / n;
    g[2] = dz / n;
    return;
  }
  if (f->kind == NSDF_FIELD_TORUS) {
    double s = hypot(x, z);
    double q = s - a[0];
    double d = hypot(q, y);
    if (d == 0) return;
    if (s == 0) {
      g[1] = y / d;
      return;
    }
    double ff = q / (d * s);
    g[0] = x * ff;
    g[1] = y / d;
    g[2] = z * ff;
    return;
  }
  double qx = fabs(x) - a[0], qy = fabs(y) - a[1], qz = fabs(z) - a[2];
  if (qx > 0 || qy > 0 || qz > 0) {
    double px = fmax(qx, 0.0), py = fmax(qy, 0.0), pz = fmax(qz, 0.0);
    double n = sqrt(px * px + py * py + pz * pz);
    if (n == 0) return;
    g[0] = sgn(x) * px / n;
    g[1] = sgn(y) * py / n;
    g[2] = sgn(z) * pz / n;
    return;
  }
  if (qx >= qy && qx >= qz) g[0] = sgn(x);
  else if (qy >= qz) g[1] = sgn(y);
  else g[2] = sgn(z);
}

int orc_field_eval(const orc_field* f, const float* points, int k, float time, float* dist,
                   float* grad) {
  if (f->kind == 0) {
    int mode = dist && grad ? 2 : (grad ? 1 : 0);
    return orc_mlp(f, mode, points, 3, k, time, dist, grad);
  }
  for (int j = 0; j < k; ++j) {
    double x = points[j], y = points[k + j], z = points[2 * (size_t)k + j];
    if (dist) dist[j] = (float)an_eval(f, x, y, z);
    if (grad) {
      double g[3];
      an_grad(f, x, y, z, g);
      for (int c = 0; c < 3; ++c) grad[(size_t)c * (size_t)k + j] = (float)g[c];
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------------------
 * Rays: generate_rays (src/tracer/camera.cpp:20-43), double math, no contraction.
 * --------------------------------------------------------------------------------- */
typedef struct {
  double x, y, z;
} v3;
static v3 v3_sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static double v3_norm(v3 a) { return sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
static v3 v3_normalized(v3 a) {
  double n = v3_norm(a);
  v3 z = {0, 0, 0};
  if (!(n > 0)) return z;
  v3 r = {a.x / n, a.y / n, a.z / n};
  return r;
}
static v3 v3_cross(v3 a, v3 o) {
  v3 r = {a.y * o.z - a.z * o.y, a.z * o.x - a.x * o.z, a.x * o.y - a.y * o.x};
  return r;
}

static int camera_validate(const nsdf_camera* c) { /* camera.cpp:7-18 */
  if (c->width <= 0 || c->height <= 0) return NSDF_ERR_CONFIG;
  if (!(c->vertical_fov_deg > 0) || !(c->vertical_fov_deg < 180)) return NSDF_ERR_CONFIG;
  v3 pos = {c->position[0], c->position[1], c->position[2]};
  v3 at = {c->look_at[0], c->look_at[1], c->look_at[2]};
  v3 up = {c->up[0], c->up[1], c->up[2]};
  v3 fwd = v3_normalized(v3_sub(at, pos));
  if (v3_norm(fwd) == 0) return NSDF_ERR_CONFIG;
  if (v3_norm(v3_cross(fwd, up)) < 1e-9) return NSDF_ERR_CONFIG;
  return 0;
}

static void ray_rows(const nsdf_camera* c, int row_lo, int row_hi, float* rays) {
  v3 pos = {c->position[0], c->position[1], c->position[2]};
  v3 at = {c->look_at[0], c->look_at[1], c->look_at[2]};
  v3 up0 = {c->up[0], c->up[1], c->up[2]};
  v3 fwd = v3_normalized(v3_sub(at, pos));
  v3 right = v3_normalized(v3_cross(fwd, up0));
  v3 up = v3_cross(right, fwd);
  double half_h = tan(c->vertical_fov_deg * M_PI / 360.0);
  double half_w = half_h * (double)c->width / (double)c->height;
  size_t o = 0;
  for (int py = row_lo; py < row_hi; ++py) {
    double v = (py + 0.5) / c->height;
    double sy = (1.0 - 2.0 * v) * half_h;
    for (int px = 0; px < c->width; ++px) {
      double u = (px + 0.5) / c->width;
      double sx = (2.0 * u - 1.0) * half_w;
      /* (forward + sx * right + sy * up).normalized(), Vec3 ops core.hpp:30-45 */
      v3 d = {(fwd.x + right.x * sx) + up.x * sy, (fwd.y + right.y * sx) + up.y * sy,
              (fwd.z + right.z * sx) + up.z * sy};
      d = v3_normalized(d);
      rays[o + 0] = (float)pos.x;
      rays[o + 1] = (float)pos.y;
      rays[o + 2] = (float)pos.z;
      rays[o + 3] = (float)d.x;
      rays[o + 4] = (float)d.y;
      rays[o + 5] = (float)d.z;
      o += 6;
    }
  }
}

void orc_generate_rays(const nsdf_camera* c, float* rays) { ray_rows(c, 0, c->height, rays); }

/* ---------------------------------------------------------------------------------
 * Multiscale sphere tracing: trace_level / trace_rays (src/tracer/trace.cpp:39-132),
 * per ray (results do not depend on batching, trace.hpp:69-70).
 * --------------------------------------------------------------------------------- */
typedef struct {
  orc_net net;
  int is_net;
  float* scratch;
} orc_eval_ctx;

static float eval_point(const orc_field* f, orc_eval_ctx* ec, float time, float px, float py,
                        float pz) {
  if (f->kind == 0) {
    float x[4] = {px, py, pz, time};
    float d;
    net_column(&ec->net, x, &d, NULL, ec->scratch);
    return d;
  }
  return (float)an_eval(f, px, py, pz);
}

static void ec_init(orc_eval_ctx* ec, const orc_field* f) {
  ec->is_net = f->kind == 0;
  if (ec->is_net) {
    net_init(&ec->net, f);
    ec->scratch = (float*)malloc(sizeof(float) * 9 * (size_t)ec->net.max_width + 64);
  }
}
static void ec_free(orc_eval_ctx* ec) {
  if (ec->is_net) {
    net_free(&ec->net);
    free(ec->scratch);
  }
}

static int trace_validate(const orc_level* levels, int m, const nsdf_trace_config* cfg) {
  if (m < 1) return NSDF_ERR_VALIDATION;
  for (int j = 0; j < m; ++j)
    if (!(levels[j].delta > 0)) return NSDF_ERR_VALIDATION; /* nesting.cpp:56-69 */
  if (cfg->n_levels != m) return NSDF_ERR_CONFIG;             /* trace.cpp:10-23 */
  if (m > NSDF_MAX_LEVELS) return NSDF_ERR_CONFIG;
  int any = 0;
  for (int j = 0; j < m; ++j) {
    if (cfg->budgets[j] < 0) return NSDF_ERR_CONFIG;
    if (cfg->budgets[j] > 0) any = 1;
  }
  if (!any) return NSDF_ERR_CONFIG;
  if (!(cfg->eps_stop > 0)) return NSDF_ERR_CONFIG;
  return 0;
}

static void trace_one(const orc_level* levels, orc_eval_ctx* ecs, int m,
                      const nsdf_trace_config* cfg, const float* ray, nsdf_hit_record* rec) {
  memset(rec, 0, sizeof(*rec));
  rec->level_reached = -1;
  int effective_final = -1;
  for (int j = 0; j < m; ++j)
    if (cfg->budgets[j] > 0) effective_final = j;
  float px = ray[0], py = ray[1], pz = ray[2], t = 0.0f;
  const float dx = ray[3], dy = ray[4], dz = ray[5];
  int active = 1;
  for (int j = 0; j <= effective_final; ++j) {
    if (cfg->budgets[j] == 0) continue;
    if (!active) break;
    const int final_level = j == effective_final;
    const float delta = final_level ? 0.0f : (float)levels[j].delta;
    int advanced = 0;
    for (int iter = 0; iter < cfg->budgets[j]; ++iter) {
      float f = eval_point(&levels[j].field, &ecs[j], levels[j].time, px, py, pz);
      rec->level_reached = j;
      rec->iterations_used[j]++;
      float fd = f - delta;
      rec->final_distance = fabsf(fd);
      int converged = final_level ? fabsf(fd) <= cfg->eps_stop : fd <= cfg->eps_stop;
      if (converged) {
        advanced = 1;
        break;
      }
      float step = fd;
      if (final_level && step < 0) step = 0;
      px += step * dx;
      py += step * dy;
      pz += step * dz;
      t += step;
      if (t > cfg->t_max) break; /* miss: flew past the far clip */
    }
    active = advanced;
  }
  rec->hit = active;
  rec->point[0] = px;
  rec->point[1] = py;
  rec->point[2] = pz;
  rec->t = t;
}

int orc_trace_rays(const orc_level* levels, int m, const nsdf_trace_config* cfg, const float* rays,
                   int64_t n, nsdf_hit_record* out) {
  int st = trace_validate(levels, m, cfg);
  if (st) return st;
  orc_eval_ctx ecs[NSDF_MAX_LEVELS];
  for (int j = 0; j < m; ++j) ec_init(&ecs[j], &levels[j].field);
  for (int64_t i = 0; i < n; ++i) trace_one(levels, ecs, m, cfg, rays + 6 * i, out + i);
  for (int j = 0; j < m; ++j) ec_free(&ecs[j]);
  return 0;
}

/* ---------------------------------------------------------------------------------
 * Normals and shading: neural_normal_map (shade.cpp:8-42), shade (shade.cpp:44-93).
 * --------------------------------------------------------------------------------- */
int orc_normal_map(const orc_field* f, float time, const float* points, int k, double delta,
                   const float* fallback, float* normals, uint64_t* outside, uint64_t* fallbacks) {
  float* vals = (float*)malloc(sizeof(float) * (size_t)(k > 0 ? k : 1));
  int st = orc_field_eval(f, points, k, time, vals, normals);
  if (st) {
    free(vals);
    return st;
  }
  uint64_t out_n = 0, fb_n = 0;
  for (int j = 0; j < k; ++j) {
    if (fabs((double)vals[j]) > delta) ++out_n;
    float gx = normals[j], gy = normals[k + j], gz = normals[2 * (size_t)k + j];
    float n2 = gx * gx + gy * gy + gz * gz;
    if (n2 < 1e-16f) {
      ++fb_n;
      if (fallback) {
        normals[j] = fallback[j];
        normals[k + j] = fallback[k + j];
        normals[2 * (size_t)k + j] = fallback[2 * (size_t)k + j];
      } else {
        normals[j] = 0;
        normals[k + j] = 1;
        normals[2 * (size_t)k + j] = 0;
      }
      continue;
    }
    float inv = 1.0f / sqrtf(n2);
    normals[j] = gx * inv;
    normals[k + j] = gy * inv;
    normals[2 * (size_t)k + j] = gz * inv;
  }
  if (outside) *outside = out_n;
  if (fallbacks) *fallbacks = fb_n;
  free(vals);
  return 0;
}

static float clamp01(float v) { return v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v); }

int orc_shade(const float* points, const float* normals, int k, const nsdf_shade_config* cfg,
              const nsdf_camera* cam, float* rgb) {
  if (cfg->n_lights < 1 || cfg->n_lights > NSDF_MAX_LIGHTS) return NSDF_ERR_CONTRACT;
  float L[NSDF_MAX_LIGHTS][4];
  for (int i = 0; i < cfg->n_lights; ++i) {
    const float* d = cfg->light_direction[i];
    float n = sqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (n == 0) return NSDF_ERR_CONTRACT;
    L[i][0] = d[0] / n;
    L[i][1] = d[1] / n;
    L[i][2] = d[2] / n;
    L[i][3] = cfg->light_intensity[i];
  }
  const float cx = (float)cam->position[0], cy = (float)cam->position[1],
              cz = (float)cam->position[2];
  for (int j = 0; j < k; ++j) {
    float nx = normals[j], ny = normals[k + j], nz = normals[2 * (size_t)k + j];
    float lit = cfg->ambient;
    float spec = 0.0f;
    for (int i = 0; i < cfg->n_lights; ++i) {
      float ndotl = nx * L[i][0] + ny * L[i][1] + nz * L[i][2];
      if (ndotl > 0) lit += cfg->diffuse * L[i][3] * ndotl;
      if (cfg->specular > 0 && ndotl > 0) {
        float vx = cx - points[j], vy = cy - points[k + j], vz = cz - points[2 * (size_t)k + j];
        float vn = sqrtf(vx * vx + vy * vy + vz * vz);
        if (vn > 0) {
          float hx = L[i][0] + vx / vn, hy = L[i][1] + vy / vn, hz = L[i][2] + vz / vn;
          float hn = sqrtf(hx * hx + hy * hy + hz * hz);
          if (hn > 0) {
            float ndoth = (nx * hx + ny * hy + nz * hz) / hn;
            if (ndoth > 0) spec += cfg->specular * L[i][3] * powf(ndoth, cfg->shininess);
          }
        }
      }
    }
    rgb[j] = clamp01(cfg->albedo[0] * lit + spec);
    rgb[k + j] = clamp01(cfg->albedo[1] * lit + spec);
    rgb[2 * (size_t)k + j] = clamp01(cfg->albedo[2] * lit + spec);
  }
  return 0;
}

/* render (src/shading/render.cpp:12-82) restricted to image rows [row_lo, row_hi). */
int orc_render_rows(const orc_level* levels, int m, const nsdf_camera* cam,
                    const nsdf_trace_config* trace, const nsdf_shade_config* shade,
                    int normal_source, int fine_index, int row_lo, int row_hi, float* rgb,
                    float* depth, uint8_t* mask) {
  int st = trace_validate(levels, m, trace);
  if (st) return st;
  st = camera_validate(cam);
  if (st) return st;
  int effective_final = 0;
  for (int j = 0; j < m; ++j)
    if (trace->budgets[j] > 0) effective_final = j;
  int fine = fine_index < 0 ? m - 1 : fine_index;
  if (normal_source == NSDF_NORMALS_MAPPED && fine >= m) return NSDF_ERR_CONFIG;
  const int W = cam->width;
  const int64_t n = (int64_t)W * (row_hi - row_lo);
  float* rays = (float*)malloc(sizeof(float) * 6 * (size_t)(n > 0 ? n : 1));
  nsdf_hit_record* recs = (nsdf_hit_record*)malloc(sizeof(nsdf_hit_record) * (size_t)(n > 0 ? n : 1));
  ray_rows(cam, row_lo, row_hi, rays);
  orc_trace_rays(levels, m, trace, rays, n, recs);
  for (int64_t p = 0; p < n; ++p) {
    rgb[3 * p + 0] = shade->background[0];
    rgb[3 * p + 1] = shade->background[1];
    rgb[3 * p + 2] = shade->background[2];
    depth[p] = 0.0f;
    mask[p] = 0;
  }
  int64_t nh = 0;
  for (int64_t p = 0; p < n; ++p) nh += recs[p].hit;
  if (nh > 0) {
    const int mapped = normal_source == NSDF_NORMALS_MAPPED;
    const orc_level* own = &levels[effective_final];
    const orc_level* nf = mapped ? &levels[fine] : own;
    const double nd = levels[mapped ? fine : effective_final].delta;
    float* pts = (float*)malloc(sizeof(float) * 3 * (size_t)nh);
    float* nrm = (float*)malloc(sizeof(float) * 3 * (size_t)nh);
    float* col = (float*)malloc(sizeof(float) * 3 * (size_t)nh);
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)nh);
    int64_t h = 0;
    for (int64_t p = 0; p < n; ++p)
      if (recs[p].hit) idx[h++] = p;
    for (h = 0; h < nh; ++h)
      for (int c = 0; c < 3; ++c) pts[c * nh + h] = recs[idx[h]].point[c];
    /* chunks of 8192 (render.cpp:9) only partition the work: per-point results are
     * independent, so one batch gives the same bits. */
    if (mapped && fine != effective_final) {
      float* ownn = (float*)malloc(sizeof(float) * 3 * (size_t)nh);
      orc_normal_map(&own->field, own->time, pts, (int)nh, levels[effective_final].delta, NULL,
                     ownn, NULL, NULL);
      orc_normal_map(&nf->field, nf->time, pts, (int)nh, nd, ownn, nrm, NULL, NULL);
      free(ownn);
    } else {
      orc_normal_map(&nf->field, nf->time, pts, (int)nh, nd, NULL, nrm, NULL, NULL);
    }
    orc_shade(pts, nrm, (int)nh, shade, cam, col);
    for (h = 0; h < nh; ++h) {
      int64_t p = idx[h];
      rgb[3 * p + 0] = col[h];
      rgb[3 * p + 1] = col[nh + h];
      rgb[3 * p + 2] = col[2 * nh + h];
      depth[p] = recs[p].t;
      mask[p] = 1;
    }
    free(pts);
    free(nrm);
    free(col);
    free(idx);
  }
  free(rays);
  free(recs);
  return 0;
}

int orc_render(const orc_level* levels, int m, const nsdf_camera* cam,
               const nsdf_trace_config* trace, const nsdf_shade_config* shade, int normal_source,
               int fine_index, float* rgb, float* depth, uint8_t* mask) {
  return orc_render_rows(levels, m, cam, trace, shade, normal_source, fine_index, 0, cam->height,
                         rgb, depth, mask);
}
