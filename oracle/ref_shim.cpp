// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A C shim over the UNMODIFIED reference library (compiled from /root/reference/proj/src by
// oracle/Makefile) so the parity suite, the fixture generator and bench.py's reference arm
// can drive the reference CPU path through ctypes.  Every call goes through the
// reference's own public API (include/nsdf/*.hpp); nothing here re-implements arithmetic.
// PODs are the ones of our C ABI (include/nsdf_cuda.h) so results compare field by field.

#include <chrono>
#include <cstring>
#include <filesystem>
#include <memory>
#include <string>
#include <vector>

#include "nsdf/core.hpp"
#include "nsdf/fields/field.hpp"
#include "nsdf/fields/nesting.hpp"
#include "nsdf/mlp/mlp.hpp"
#include "nsdf/shading/shading.hpp"
#include "nsdf/tensor/kernels.hpp"
#include "nsdf/tracer/trace.hpp"
#include "nsdf_cuda.h"
#include "nsdf/trainer/trainer.hpp"

using namespace nsdf;

namespace {

thread_local std::string g_error;

int fail(const std::exception& e) {
  g_error = e.what();
  if (auto* ne = dynamic_cast<const Error*>(&e)) return 1 + int(ne->kind());
  return 3;
}

#define SHIM_TRY try {
#define SHIM_CATCH                    \
  }                                   \
  catch (const std::exception& e) {   \
    return fail(e);                   \
  }                                   \
  return 0;

mlp::MlpParams<double> unpack(int n_layers, const int32_t* rows, const int32_t* cols,
                              const double* packed, int activation, double omega0,
                              int input_dim) {
  mlp::MlpParams<double> p;
  p.input_dim = input_dim;
  p.activation = activation == NSDF_ACT_SINE ? tensor::ActivationSpec::sine(omega0)
                                             : tensor::ActivationSpec::identity();
  size_t off = 0;
  for (int l = 0; l < n_layers; ++l) {
    std::vector<double> w(packed + off, packed + off + size_t(rows[l]) * cols[l]);
    off += size_t(rows[l]) * cols[l];
    std::vector<double> b(packed + off, packed + off + rows[l]);
    off += rows[l];
    p.layers.push_back({tensor::Matrix<double>(rows[l], cols[l], std::move(w)),
                        tensor::Matrix<double>(rows[l], 1, std::move(b))});
  }
  return p;
}

tracer::Camera to_camera(const nsdf_camera* c) {
  tracer::Camera cam;
  cam.position = {c->position[0], c->position[1], c->position[2]};
  cam.look_at = {c->look_at[0], c->look_at[1], c->look_at[2]};
  cam.up = {c->up[0], c->up[1], c->up[2]};
  cam.vertical_fov_deg = c->vertical_fov_deg;
  cam.width = c->width;
  cam.height = c->height;
  return cam;
}

tracer::TraceConfig to_trace(const nsdf_trace_config* t) {
  tracer::TraceConfig cfg;
  cfg.budgets.assign(t->budgets, t->budgets + t->n_levels);
  cfg.eps_stop = t->eps_stop;
  cfg.t_max = t->t_max;
  return cfg;
}

shading::ShadeConfig to_shade(const nsdf_shade_config* s) {
  shading::ShadeConfig cfg;
  cfg.material.albedo = {s->albedo[0], s->albedo[1], s->albedo[2]};
  cfg.material.ambient = s->ambient;
  cfg.material.diffuse = s->diffuse;
  cfg.material.specular = s->specular;
  cfg.material.shininess = s->shininess;
  cfg.lights.clear();
  for (int i = 0; i < s->n_lights; ++i)
    cfg.lights.push_back({{s->light_direction[i][0], s->light_direction[i][1],
                           s->light_direction[i][2]},
                          s->light_intensity[i]});
  cfg.background = {s->background[0], s->background[1], s->background[2]};
  return cfg;
}

void to_pod(const tracer::HitRecord& r, nsdf_hit_record* o) {
  o->hit = r.hit ? 1 : 0;
  o->point[0] = r.point.x;
  o->point[1] = r.point.y;
  o->point[2] = r.point.z;
  o->t = r.t;
  o->level_reached = r.level_reached;
  for (int i = 0; i < NSDF_MAX_LEVELS; ++i) o->iterations_used[i] = r.iterations_used[i];
  o->final_distance = r.final_distance;
}

fields::NestedSequence load_sequence(const char* manifest, double time) {
  fields::SequenceManifest m = fields::load_manifest(manifest);
  return m.time_dependent ? m.animated.slice(time) : m.sequence;
}

tensor::Matrix<float> points_matrix(const float* pts, int rows, int k) {
  return tensor::Matrix<float>(rows, k, std::vector<float>(pts, pts + size_t(rows) * k));
}

}  // namespace

// tensor::gemm / hadamard / activate(sine) / scale_rows (ops.cpp:24-95) through the reference's
// active kernel backend; dtype 0 = float, 1 = double; op 0 gemm (a m x k, b k x n, bias m or
// null -> c m x n), 1 hadamard (a, b: m x n), 2 sine (a m x n, omega, derivative), 3
// scale_rows (a = col m x 1, b m x n).
namespace {
template <typename T>
int ref_tensor(int op, const T* a, const T* b, const T* bias, T* out, int m, int n, int k, double omega,
               int derivative) {
  auto mat = [](const T* p, int r, int c) { return tensor::Matrix<T>(r, c, std::vector<T>(p, p + size_t(r) * c)); };
  tensor::Matrix<T> res;
  if (op == 0) {
    tensor::Matrix<T> bm;
    if (bias) bm = mat(bias, m, 1);
    res = tensor::gemm(mat(a, m, k), mat(b, k, n), bias ? &bm : nullptr);
  } else if (op == 1) {
    res = tensor::hadamard(mat(a, m, n), mat(b, m, n));
  } else if (op == 2) {
    res = tensor::activate(mat(a, m, n), tensor::ActivationSpec::sine(omega), derivative != 0);
  } else {
    res = tensor::scale_rows(mat(a, m, 1), mat(b, m, n));
  }
  std::copy(res.data(), res.data() + res.size(), out);
  return 0;
}
}  // namespace

extern "C" {

const char* nsdf_ref_last_error(void) { return g_error.c_str(); }

int nsdf_ref_worker_threads(void) { return worker_thread_count(); }

int nsdf_ref_set_backend(const char* name) {
  SHIM_TRY
  std::string n(name);
  tensor::set_backend(n == "scalar" ? tensor::Backend::scalar
                                    : n == "neon" ? tensor::Backend::neon : tensor::Backend::avx2);
  SHIM_CATCH
}

const char* nsdf_ref_backend(void) { return tensor::backend_name(tensor::active_backend()); }


int nsdf_ref_tensor(int op, int dtype, const void* a, const void* b, const void* bias, void* out, int m, int n, int k,
                    double omega, int derivative) {
  SHIM_TRY
  if (dtype == 1)
    ref_tensor<double>(op, static_cast<const double*>(a), static_cast<const double*>(b),
                       static_cast<const double*>(bias), static_cast<double*>(out), m, n, k, omega, derivative);
  else
    ref_tensor<float>(op, static_cast<const float*>(a), static_cast<const float*>(b), static_cast<const float*>(bias),
                      static_cast<float*>(out), m, n, k, omega, derivative);
  SHIM_CATCH
}

// mlp::random_init (mlp.cpp:63-88) with Rng(seed); writes the packed layout.
int nsdf_ref_random_init(int width, int hidden, int input_dim, double omega0, uint64_t seed,
                         double* packed, int32_t* rows, int32_t* cols) {
  SHIM_TRY
  Rng rng(seed);
  mlp::Architecture arch{width, hidden, input_dim};
  auto p = mlp::random_init(arch, omega0, rng);
  size_t off = 0;
  for (size_t l = 0; l < p.layers.size(); ++l) {
    const auto& L = p.layers[l];
    rows[l] = L.weights.rows();
    cols[l] = L.weights.cols();
    std::memcpy(packed + off, L.weights.data(), L.weights.size() * sizeof(double));
    off += L.weights.size();
    std::memcpy(packed + off, L.bias.data(), L.bias.size() * sizeof(double));
    off += L.bias.size();
  }
  SHIM_CATCH
}

// mode 0: forward_batch, 1: gradient_batch (spatial for 4-input nets), 2: fused.
// f32 path exactly as NeuralField (params cast once, field.cpp:150).
int nsdf_ref_mlp(int mode, int n_layers, const int32_t* rows, const int32_t* cols,
                 const double* packed, int activation, double omega0, int input_dim,
                 const float* pts, int k, float* dist, float* grad) {
  SHIM_TRY
  auto p64 = unpack(n_layers, rows, cols, packed, activation, omega0, input_dim);
  auto p = p64.cast<float>();
  auto P = points_matrix(pts, input_dim, k);
  if (mode == 0) {
    auto d = mlp::forward_batch(p, P);
    std::memcpy(dist, d.data(), sizeof(float) * k);
  } else if (mode == 1) {
    auto g = input_dim == 4 ? mlp::spatial_gradient_batch(p, P) : mlp::gradient_batch(p, P);
    std::memcpy(grad, g.data(), sizeof(float) * 3 * k);
  } else {
    auto [d, g] = mlp::forward_and_gradient_batch(p, P);
    std::memcpy(dist, d.data(), sizeof(float) * k);
    std::memcpy(grad, g.data(), sizeof(float) * 3 * k);
  }
  SHIM_CATCH
}

int nsdf_ref_mlp_f64(int mode, int n_layers, const int32_t* rows, const int32_t* cols,
                     const double* packed, int activation, double omega0, int input_dim,
                     const double* pts, int k, double* dist, double* grad) {
  SHIM_TRY
  auto p = unpack(n_layers, rows, cols, packed, activation, omega0, input_dim);
  tensor::Matrix<double> P(input_dim, k, std::vector<double>(pts, pts + size_t(input_dim) * k));
  if (mode == 0 || mode == 2) {
    auto d = mlp::forward_batch(p, P);
    std::memcpy(dist, d.data(), sizeof(double) * k);
  }
  if (mode == 1 || mode == 2) {
    auto g = input_dim == 4 ? mlp::spatial_gradient_batch(p, P) : mlp::gradient_batch(p, P);
    std::memcpy(grad, g.data(), sizeof(double) * 3 * k);
  }
  SHIM_CATCH
}

int nsdf_ref_save_params(int n_layers, const int32_t* rows, const int32_t* cols,
                         const double* packed, int activation, double omega0, int input_dim,
                         const char* path) {
  SHIM_TRY
  mlp::save_params(unpack(n_layers, rows, cols, packed, activation, omega0, input_dim), path);
  SHIM_CATCH
}

int nsdf_ref_generate_rays(const nsdf_camera* camera, float* rays) {
  SHIM_TRY
  auto rs = tracer::generate_rays(to_camera(camera));
  for (size_t i = 0; i < rs.size(); ++i) {
    rays[6 * i + 0] = rs[i].origin.x;
    rays[6 * i + 1] = rs[i].origin.y;
    rays[6 * i + 2] = rs[i].origin.z;
    rays[6 * i + 3] = rs[i].direction.x;
    rays[6 * i + 4] = rs[i].direction.y;
    rays[6 * i + 5] = rs[i].direction.z;
  }
  SHIM_CATCH
}

// Field batch evaluation of one member of a manifest (eval_batch / grad_batch, f32).
int nsdf_ref_field_eval(const char* manifest, double time, int index, const float* pts, int k,
                        float* dist, float* grad) {
  SHIM_TRY
  auto seq = load_sequence(manifest, time);
  auto P = points_matrix(pts, 3, k);
  if (dist) {
    auto d = seq.field(index).eval_batch(P);
    std::memcpy(dist, d.data(), sizeof(float) * k);
  }
  if (grad) {
    auto g = seq.field(index).grad_batch(P);
    std::memcpy(grad, g.data(), sizeof(float) * 3 * k);
  }
  SHIM_CATCH
}

int nsdf_ref_trace_image(const char* manifest, double time, const nsdf_camera* camera,
                         const nsdf_trace_config* config, nsdf_hit_record* out) {
  SHIM_TRY
  auto seq = load_sequence(manifest, time);
  auto recs = tracer::trace_image(seq, to_camera(camera), to_trace(config));
  for (size_t i = 0; i < recs.size(); ++i) to_pod(recs[i], out + i);
  SHIM_CATCH
}

// Per-ray multiscale_sphere_trace (trace.cpp:162-169).
int nsdf_ref_trace_rays(const char* manifest, double time, const nsdf_trace_config* config,
                        const float* rays, int n, nsdf_hit_record* out) {
  SHIM_TRY
  auto seq = load_sequence(manifest, time);
  auto cfg = to_trace(config);
  for (int i = 0; i < n; ++i) {
    tracer::Ray r{{rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]},
                  {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]}};
    to_pod(tracer::multiscale_sphere_trace(seq, r, cfg), out + i);
  }
  SHIM_CATCH
}

// Classic sphere_trace of one member (trace.cpp:136-160).
int nsdf_ref_sphere_trace(const char* manifest, double time, int index, float delta,
                          float eps_stop, int max_iters, float t_max, const float* rays, int n,
                          nsdf_hit_record* out) {
  SHIM_TRY
  auto seq = load_sequence(manifest, time);
  for (int i = 0; i < n; ++i) {
    tracer::Ray r{{rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]},
                  {rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5]}};
    to_pod(tracer::sphere_trace(seq.field(index), r, delta, eps_stop, max_iters, t_max), out + i);
  }
  SHIM_CATCH
}

int nsdf_ref_normal_map(const char* manifest, double time, int index, const float* pts, int k,
                        double delta, const float* fallback, float* normals,
                        uint64_t* outside, uint64_t* fallbacks) {
  SHIM_TRY
  auto seq = load_sequence(manifest, time);
  auto P = points_matrix(pts, 3, k);
  std::unique_ptr<tensor::Matrix<float>> fb;
  if (fallback) fb = std::make_unique<tensor::Matrix<float>>(points_matrix(fallback, 3, k));
  auto r = shading::neural_normal_map(seq.field(index), P, delta, fb.get());
  std::memcpy(normals, r.normals.data(), sizeof(float) * 3 * k);
  *outside = r.outside_count;
  *fallbacks = r.fallback_count;
  SHIM_CATCH
}

// shading::map_normals_to_mesh (mesh.cpp:122-156) on a Mesh built from k x 3 double
// vertices and (has_normals) k x 3 double normals; normals_out receives mesh.normals after
// the call (k x 3, or untouched when the mesh ends without normals); counts {mapped,
// violators, fallbacks}; *out_has = whether the mesh has normals afterwards.
int nsdf_ref_map_normals_mesh(const char* manifest, double time, int index, const double* verts, int k,
                              const double* normals_in, int has_normals, double delta, double* normals_out,
                              uint64_t* counts, int* out_has) {
  SHIM_TRY
  auto seq = load_sequence(manifest, time);
  shading::Mesh mesh;
  for (int j = 0; j < k; ++j) mesh.vertices.push_back({verts[3 * j], verts[3 * j + 1], verts[3 * j + 2]});
  if (has_normals)
    for (int j = 0; j < k; ++j)
      mesh.normals.push_back({normals_in[3 * j], normals_in[3 * j + 1], normals_in[3 * j + 2]});
  auto r = shading::map_normals_to_mesh(mesh, seq.field(index), delta);
  counts[0] = r.mapped;
  counts[1] = r.violators;
  counts[2] = r.fallbacks;
  *out_has = mesh.has_normals() ? 1 : 0;
  for (size_t j = 0; j < mesh.normals.size(); ++j) {
    normals_out[3 * j] = mesh.normals[j].x;
    normals_out[3 * j + 1] = mesh.normals[j].y;
    normals_out[3 * j + 2] = mesh.normals[j].z;
  }
  SHIM_CATCH
}

// The reference CLI's train flow (nsdf_main.cpp:163-258: fit_sequence(_4d) -> save_params,
// report.write, save_manifest) through the reference library, minus the config echo.
int nsdf_ref_train(const char* shape, const char* archs_csv, int epochs, const char* epochs_list, double lr,
                   double omega0, uint64_t seed, uint64_t n_uniform, uint64_t n_surface, double sigma,
                   uint64_t sup_uniform, uint64_t sup_surface, uint64_t verify_samples, double domain_half,
                   const char* out_dir, const char* name) {
  SHIM_TRY
  auto split = [](const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    for (char ch : s + ",") {
      if (ch == ',') {
        if (!cur.empty()) out.push_back(cur);
        cur.clear();
      } else {
        cur += ch;
      }
    }
    return out;
  };
  fields::AnalyticSpec spec = fields::parse_field_spec(shape);
  const bool td = spec.name == "blend";
  std::vector<mlp::Architecture> archs;
  for (const auto& a : split(archs_csv)) archs.push_back(mlp::parse_architecture(a, td ? 4 : 3));
  std::filesystem::path dir(out_dir);
  std::filesystem::create_directories(dir);
  trainer::SequenceFitConfig config;
  config.train.epochs = epochs;
  config.train.learning_rate = lr;
  config.train.omega0 = omega0;
  config.train.seed = seed;
  config.samples = {n_uniform, n_surface, sigma, 10000, seed};
  config.sup.n_uniform = sup_uniform;
  config.sup.n_surface = sup_surface;
  config.sup.seed = seed + 1;
  config.verify.samples = verify_samples;
  config.verify.seed = seed + 2;
  for (const auto& e : split(epochs_list)) config.epochs_per_arch.push_back(std::stoi(e));
  auto save = [&](size_t i, const mlp::MlpParams<double>& p, const trainer::TrainReport& r) {
    std::string stem = std::string(name) + "_" + archs[i].name();
    mlp::save_params(p, dir / (stem + ".sdfnet"));
    r.write(dir / (stem + ".report.txt"));
    return stem + ".sdfnet";
  };
  if (td) {
    auto oracle = std::const_pointer_cast<fields::TimeVaryingField>(
        std::shared_ptr<const fields::TimeVaryingField>(fields::make_analytic_time_field(spec)));
    oracle->set_domain(Aabb::cube(domain_half));
    auto fit = trainer::fit_sequence_4d(archs, *oracle, config);
    for (size_t i = 0; i < archs.size(); ++i)
      fit.sequence.entries[i].source = {fields::FieldSource::Kind::weights, {}, save(i, fit.params[i], fit.reports[i])};
    fields::save_manifest(fit.sequence, dir / (std::string(name) + ".nest"));
  } else {
    auto oracle = std::const_pointer_cast<fields::Field>(fields::make_analytic_field(spec));
    oracle->set_domain(Aabb::cube(domain_half));
    auto fit = trainer::fit_sequence(archs, *oracle, config);
    for (size_t i = 0; i < archs.size(); ++i)
      fit.sequence.entries[i].source = {fields::FieldSource::Kind::weights, {}, save(i, fit.params[i], fit.reports[i])};
    fields::save_manifest(fit.sequence, dir / (std::string(name) + ".nest"));
  }
  SHIM_CATCH
}

int nsdf_ref_write_image(const char* path, int width, int height, const float* rgb) {
  SHIM_TRY
  shading::ImageBuffer img(width, height);
  std::memcpy(img.rgb.data(), rgb, sizeof(float) * img.rgb.size());
  const std::filesystem::path p(path);
  if (p.extension() == ".png")
    shading::write_png(img, p);
  else
    shading::write_ppm(img, p);
  SHIM_CATCH
}

int nsdf_ref_shade(const float* pts, const float* normals, int k, const nsdf_shade_config* shade,
                   const nsdf_camera* camera, float* rgb) {
  SHIM_TRY
  auto r = shading::shade(points_matrix(pts, 3, k), points_matrix(normals, 3, k),
                          to_shade(shade), to_camera(camera));
  std::memcpy(rgb, r.data(), sizeof(float) * 3 * k);
  SHIM_CATCH
}

// shading::render of a manifest (sliced at `time` when time-dependent), timed with
// steady_clock like `nsdf bench` (nsdf_main.cpp:466-470); `seconds` gets the wall time
// of the render call alone (manifest loading excluded).
int nsdf_ref_render(const char* manifest, double time, const nsdf_camera* camera,
                    const nsdf_trace_config* trace, const nsdf_shade_config* shade,
                    int normal_source, int fine_index, float* rgb, float* depth, uint8_t* mask,
                    double* seconds) {
  SHIM_TRY
  auto seq = load_sequence(manifest, time);
  shading::RenderConfig cfg;
  cfg.trace = to_trace(trace);
  cfg.shade = to_shade(shade);
  cfg.normal_source =
      normal_source == NSDF_NORMALS_MAPPED ? shading::NormalSource::mapped : shading::NormalSource::own;
  cfg.mapped_fine_index = fine_index;
  auto t0 = std::chrono::steady_clock::now();
  auto img = shading::render(seq, to_camera(camera), cfg);
  auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  std::memcpy(rgb, img.rgb.data(), sizeof(float) * img.rgb.size());
  std::memcpy(depth, img.depth.data(), sizeof(float) * img.depth.size());
  std::memcpy(mask, img.mask.data(), img.mask.size());
  SHIM_CATCH
}

// Fixture certification (fit.cpp:262-298 minus the fitting): eps_i = estimate_sup_diff
// of each weight file against the analytic reference shape, Prop-2 thresholds, empirical
// verify_nesting, save_manifest.  Returns eps/deltas and the violation count.
int nsdf_ref_certify(const char* const* weight_paths, const char* const* labels, int m,
                     const char* analytic_spec, uint64_t n_uniform, uint64_t n_surface,
                     double margin, uint64_t sup_seed, uint64_t verify_samples,
                     const char* out_manifest, double* eps_out, double* deltas_out,
                     uint64_t* violations) {
  SHIM_TRY
  auto oracle = fields::make_analytic_field(fields::parse_field_spec(analytic_spec));
  fields::NestedSequence seq;
  std::vector<double> eps;
  for (int i = 0; i < m; ++i) {
    auto params = mlp::load_params(weight_paths[i]);
    size_t count = params.parameter_count();
    auto field = std::make_shared<fields::NeuralField>(std::move(params));
    field->set_domain(oracle->domain());
    fields::SupSamplerConfig sup;
    sup.n_uniform = n_uniform;
    sup.n_surface = n_surface;
    sup.margin = margin;
    sup.seed = sup_seed + 31 * i;
    eps.push_back(fields::estimate_sup_diff(*field, *oracle, sup).eps);
    fields::FieldSource src;
    src.kind = fields::FieldSource::Kind::weights;
    std::string wp(weight_paths[i]);
    src.weights_path = wp.substr(wp.find_last_of('/') + 1);
    seq.entries.push_back({field, src, labels[i], count});
  }
  seq.deltas = m == 1 ? std::vector<double>{eps[0] + margin} : fields::thresholds_prop2(eps);
  seq.provenance.proposition = m == 1 ? 0 : 2;
  seq.provenance.eps = eps;
  seq.provenance.margin = margin;
  seq.provenance.sampler_seed = sup_seed;
  seq.provenance.n_uniform = n_uniform;
  seq.provenance.n_surface = n_surface;
  fields::VerifyConfig vc;
  vc.samples = verify_samples;
  auto report = fields::verify_nesting(seq, vc);
  seq.provenance.verify_samples = verify_samples;
  seq.provenance.verify_violations = report.violation_count;
  if (!report.ok()) seq.provenance.note = "empirical nesting violations recorded";
  fields::save_manifest(seq, out_manifest);
  for (int i = 0; i < m; ++i) {
    eps_out[i] = eps[i];
    deltas_out[i] = seq.deltas[i];
  }
  *violations = report.violation_count;
  SHIM_CATCH
}

// ---- certification (nesting.cpp:131-361), same signatures as nsdf_host.h ----
static fields::FieldPtr ref_field(const char* src, const Aabb* domain = nullptr) {
  const std::string s(src);
  if (s.rfind("weights:", 0) == 0) {
    auto f = std::make_shared<fields::NeuralField>(mlp::load_params(s.substr(8)));
    if (domain) f->set_domain(*domain);
    return f;
  }
  return fields::make_analytic_field(fields::parse_field_spec(s));
}

int nsdf_ref_sample_near_surface(const char* field, uint64_t count, int gaussian, double amount, uint64_t seed,
                                 double* out) {
  SHIM_TRY
  auto f = ref_field(field);
  Rng rng(seed);
  fields::SurfaceNoise noise;
  noise.kind = gaussian ? fields::SurfaceNoise::Kind::gaussian : fields::SurfaceNoise::Kind::uniform;
  noise.amount = amount;
  auto pts = fields::sample_near_surface(*f, size_t(count), noise, rng);
  for (size_t i = 0; i < pts.size(); ++i) {
    out[3 * i] = pts[i].x;
    out[3 * i + 1] = pts[i].y;
    out[3 * i + 2] = pts[i].z;
  }
  SHIM_CATCH
}

int nsdf_ref_sup_diff(const char* f_src, const char* g_src, uint64_t n_uniform, uint64_t n_surface, double margin,
                      double noise_halfwidth, uint64_t seed, double* out) {
  SHIM_TRY
  auto g = ref_field(g_src);
  auto f = ref_field(f_src, &g->domain());
  fields::SupSamplerConfig cfg;
  cfg.n_uniform = size_t(n_uniform);
  cfg.n_surface = size_t(n_surface);
  cfg.margin = margin;
  cfg.noise_halfwidth = noise_halfwidth;
  cfg.seed = seed;
  auto r = fields::estimate_sup_diff(*f, *g, cfg);
  out[0] = r.eps;
  out[1] = r.raw_max;
  out[2] = r.argmax.x;
  out[3] = r.argmax.y;
  out[4] = r.argmax.z;
  out[5] = double(r.samples);
  SHIM_CATCH
}

int nsdf_ref_verify_nesting(const char* manifest, double time, uint64_t samples, uint64_t seed, uint64_t max_recorded,
                            uint64_t* counts, double* recorded) {
  SHIM_TRY
  auto seq = load_sequence(manifest, time);
  fields::VerifyConfig cfg;
  cfg.samples = size_t(samples);
  cfg.seed = seed;
  cfg.max_recorded_violations = size_t(max_recorded);
  auto r = fields::verify_nesting(seq, cfg);
  counts[0] = r.samples_total;
  counts[1] = r.checked;
  counts[2] = r.violation_count;
  counts[3] = r.violations.size();
  for (size_t i = 0; i < r.violations.size(); ++i) {
    double* o = recorded + 6 * i;
    o[0] = r.violations[i].point.x;
    o[1] = r.violations[i].point.y;
    o[2] = r.violations[i].point.z;
    o[3] = double(r.violations[i].pair_index);
    o[4] = r.violations[i].f_coarse;
    o[5] = r.violations[i].f_fine;
  }
  SHIM_CATCH
}

// ---- training (trainer::sample_training_set / fit_mlp / backprop_sine_mlp) ----
int nsdf_ref_sample_training_set(const char* oracle, uint64_t n_uniform, uint64_t n_surface, double sigma,
                                 uint64_t n_validation, uint64_t seed, double* points_out, double* targets_out,
                                 double* val_points_out, double* val_targets_out) {
  SHIM_TRY
  auto f = ref_field(oracle);
  trainer::SampleConfig sc;
  sc.n_uniform = size_t(n_uniform);
  sc.n_surface = size_t(n_surface);
  sc.sigma = sigma;
  sc.n_validation = size_t(n_validation);
  sc.seed = seed;
  auto set = trainer::sample_training_set(*f, sc);
  std::memcpy(points_out, set.points.data(), sizeof(double) * set.points.size());
  std::memcpy(targets_out, set.targets.data(), sizeof(double) * set.targets.size());
  std::memcpy(val_points_out, set.val_points.data(), sizeof(double) * set.val_points.size());
  std::memcpy(val_targets_out, set.val_targets.data(), sizeof(double) * set.val_targets.size());
  SHIM_CATCH
}

static void ref_put_params(const mlp::MlpParams<double>& p, double* out) {
  size_t o = 0;
  for (const auto& l : p.layers) {
    std::memcpy(out + o, l.weights.data(), sizeof(double) * l.weights.size());
    o += l.weights.size();
    std::memcpy(out + o, l.bias.data(), sizeof(double) * l.bias.size());
    o += l.bias.size();
  }
}

int nsdf_ref_fit_mlp(const char* arch, int input_dim, double omega0, uint64_t seed, const nsdf_train_config* cfg,
                     const double* points, const double* targets, int n, const double* val_points,
                     const double* val_targets, int n_val, double* params_out, double* epoch_loss,
                     nsdf_train_report* report) {
  SHIM_TRY
  trainer::TrainConfig tc;
  tc.arch = mlp::parse_architecture(arch, input_dim);
  tc.epochs = cfg->epochs;
  tc.batch_size = cfg->batch_size;
  tc.learning_rate = cfg->learning_rate;
  tc.momentum = cfg->momentum;
  tc.omega0 = omega0;
  tc.seed = seed;
  tc.warmup_epochs = cfg->warmup_epochs;
  tc.plateau_patience = cfg->plateau_patience;
  tc.plateau_threshold = cfg->plateau_threshold;
  tc.min_learning_rate = cfg->min_learning_rate;
  trainer::TrainingSet set;
  set.input_dim = input_dim;
  set.points = tensor::Matrix<double>(input_dim, n, std::vector<double>(points, points + size_t(input_dim) * n));
  set.targets = tensor::Matrix<double>(1, n, std::vector<double>(targets, targets + n));
  set.val_points = tensor::Matrix<double>(input_dim, n_val,
                                          std::vector<double>(val_points, val_points + size_t(input_dim) * n_val));
  set.val_targets = tensor::Matrix<double>(1, n_val, std::vector<double>(val_targets, val_targets + n_val));
  auto fit = trainer::fit_mlp(tc, set);
  ref_put_params(fit.params, params_out);
  std::memset(report, 0, sizeof(*report));
  for (size_t i = 0; i < fit.report.epoch_loss.size(); ++i) epoch_loss[i] = fit.report.epoch_loss[i];
  report->epochs_recorded = int(fit.report.epoch_loss.size());
  report->final_loss = fit.report.final_loss;
  report->validation_mse = fit.report.validation_mse;
  report->validation_max_error = fit.report.validation_max_error;
  report->final_learning_rate = fit.report.final_learning_rate;
  report->diverged = fit.report.diverged ? 1 : 0;
  report->halvings = fit.report.halvings;
  SHIM_CATCH
}

int nsdf_ref_backprop(const char* arch, int input_dim, double omega0, uint64_t seed, const double* points,
                      const double* targets, int k, double* params_out, double* grads_out, double* loss) {
  SHIM_TRY
  Rng rng(seed);
  auto params = mlp::random_init(mlp::parse_architecture(arch, input_dim), omega0, rng);
  ref_put_params(params, params_out);
  auto g = trainer::backprop_sine_mlp(
      params, tensor::Matrix<double>(input_dim, k, std::vector<double>(points, points + size_t(input_dim) * k)),
      tensor::Matrix<double>(1, k, std::vector<double>(targets, targets + k)), loss);
  size_t o = 0;
  for (const auto& l : g.layers) {
    std::memcpy(grads_out + o, l.weights.data(), sizeof(double) * l.weights.size());
    o += l.weights.size();
    std::memcpy(grads_out + o, l.bias.data(), sizeof(double) * l.bias.size());
    o += l.bias.size();
  }
  SHIM_CATCH
}

}  // extern "C"
