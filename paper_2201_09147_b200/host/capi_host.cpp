// extern "C" entry points into the drop-in C++ API, so tests and bench.py can drive the
// reference-shaped call chain (load_manifest -> shading::render / tracer::trace_image ->
// C ABI -> B200) in-process through ctypes.  Declared in include/nsdf_host.h.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <filesystem>
#include <string>

#include "device_seq.hpp"
#include "nsdf_host.h"
#include "nsdf/trainer/trainer.hpp"

using namespace nsdf;

namespace {
thread_local std::string g_err;

int fail_from(const std::exception& e) {
  g_err = e.what();
  if (auto* ne = dynamic_cast<const Error*>(&e)) return 1 + int(ne->kind());
  return NSDF_ERR_VALIDATION;
}

fields::NestedSequence sequence_of(const char* manifest, double time) {
  auto m = fields::load_manifest(manifest);
  return m.time_dependent ? m.animated.slice(time) : m.sequence;
}

tracer::Camera camera_of(const nsdf_camera* c) {
  tracer::Camera cam;
  cam.position = {c->position[0], c->position[1], c->position[2]};
  cam.look_at = {c->look_at[0], c->look_at[1], c->look_at[2]};
  cam.up = {c->up[0], c->up[1], c->up[2]};
  cam.vertical_fov_deg = c->vertical_fov_deg;
  cam.width = c->width;
  cam.height = c->height;
  return cam;
}

tracer::TraceConfig trace_of(const nsdf_trace_config* t) {
  tracer::TraceConfig cfg;
  cfg.budgets.assign(t->budgets, t->budgets + t->n_levels);
  cfg.eps_stop = t->eps_stop;
  cfg.t_max = t->t_max;
  return cfg;
}

// "weights:<file.sdfnet>" -> NeuralField; anything else is an analytic spec ("torus:R=0.6,r=0.3").
// A neural field takes `domain` when given (as the reference's certify flow does, fit.cpp).
fields::FieldPtr field_of(const char* src, const Aabb* domain = nullptr) {
  const std::string s(src);
  if (s.rfind("weights:", 0) == 0) {
    auto f = std::make_shared<fields::NeuralField>(mlp::load_params(s.substr(8)));
    if (domain) f->set_domain(*domain);
    return f;
  }
  return fields::make_analytic_field(fields::parse_field_spec(s));
}

void put_vec(const Vec3& v, double* out) {
  out[0] = v.x;
  out[1] = v.y;
  out[2] = v.z;
}

shading::ShadeConfig shade_of(const nsdf_shade_config* s) {
  shading::ShadeConfig cfg;
  cfg.material.albedo = {s->albedo[0], s->albedo[1], s->albedo[2]};
  cfg.material.ambient = s->ambient;
  cfg.material.diffuse = s->diffuse;
  cfg.material.specular = s->specular;
  cfg.material.shininess = s->shininess;
  cfg.lights.clear();
  for (int i = 0; i < s->n_lights; ++i)
    cfg.lights.push_back({{s->light_direction[i][0], s->light_direction[i][1], s->light_direction[i][2]},
                          s->light_intensity[i]});
  cfg.background = {s->background[0], s->background[1], s->background[2]};
  return cfg;
}
}  // namespace

extern "C" {

const char* nsdf_host_last_error(void) { return g_err.c_str(); }

int nsdf_host_render_manifest(const char* manifest, double time, const nsdf_camera* camera,
                              const nsdf_trace_config* trace, const nsdf_shade_config* shade, int normal_source,
                              int fine_index, float* rgb, float* depth, uint8_t* mask) {
  try {
    const auto seq = sequence_of(manifest, time);
    shading::RenderConfig cfg;
    cfg.trace = trace_of(trace);
    cfg.shade = shade_of(shade);
    cfg.normal_source = normal_source == NSDF_NORMALS_MAPPED ? shading::NormalSource::mapped : shading::NormalSource::own;
    cfg.mapped_fine_index = fine_index;
    const auto img = shading::render(seq, camera_of(camera), cfg);
    std::memcpy(rgb, img.rgb.data(), img.rgb.size() * sizeof(float));
    std::memcpy(depth, img.depth.data(), img.depth.size() * sizeof(float));
    std::memcpy(mask, img.mask.data(), img.mask.size());
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

int nsdf_host_bench_render(const char* manifest, double time, const nsdf_camera* camera,
                           const nsdf_trace_config* trace, const nsdf_shade_config* shade, int normal_source,
                           int fine_index, int warmup, int repeats, double* seconds_per_frame) {
  try {
    const auto seq = sequence_of(manifest, time);
    shading::RenderConfig cfg;
    cfg.trace = trace_of(trace);
    cfg.shade = shade_of(shade);
    cfg.normal_source = normal_source == NSDF_NORMALS_MAPPED ? shading::NormalSource::mapped : shading::NormalSource::own;
    cfg.mapped_fine_index = fine_index;
    const tracer::Camera cam = camera_of(camera);
    for (int i = 0; i < warmup; ++i) (void)shading::render(seq, cam, cfg);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < repeats; ++i) (void)shading::render(seq, cam, cfg);
    *seconds_per_frame =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / std::max(repeats, 1);
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

int nsdf_host_trace_image_manifest(const char* manifest, double time, const nsdf_camera* camera,
                                   const nsdf_trace_config* trace, nsdf_hit_record* out) {
  try {
    const auto recs = tracer::trace_image(sequence_of(manifest, time), camera_of(camera), trace_of(trace));
    for (size_t i = 0; i < recs.size(); ++i) {
      const auto& r = recs[i];
      nsdf_hit_record& o = out[i];
      o.hit = r.hit ? 1 : 0;
      o.point[0] = r.point.x;
      o.point[1] = r.point.y;
      o.point[2] = r.point.z;
      o.t = r.t;
      o.level_reached = r.level_reached;
      for (int j = 0; j < NSDF_MAX_LEVELS; ++j) o.iterations_used[j] = r.iterations_used[j];
      o.final_distance = r.final_distance;
    }
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

int nsdf_host_forward_and_gradient(const char* sdfnet, const float* points, int k, float* dist, float* grad) {
  try {
    const auto p = mlp::load_params(sdfnet).cast<float>();
    tensor::Matrix<float> pts(3, k, std::vector<float>(points, points + size_t(3) * k));
    auto [d, g] = mlp::forward_and_gradient_batch(p, pts);
    std::memcpy(dist, d.data(), sizeof(float) * size_t(k));
    std::memcpy(grad, g.data(), sizeof(float) * size_t(3) * k);
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

int nsdf_host_write_image(const char* path, int width, int height, const float* rgb) {
  try {
    shading::ImageBuffer img(width, height);
    std::memcpy(img.rgb.data(), rgb, sizeof(float) * img.rgb.size());
    const std::filesystem::path p(path);
    if (p.extension() == ".png")
      shading::write_png(img, p);
    else
      shading::write_ppm(img, p);
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

int nsdf_host_read_ppm(const char* path, int* width, int* height, float* rgb, size_t capacity) {
  try {
    const auto img = shading::read_ppm(path);
    *width = img.width;
    *height = img.height;
    if (rgb && capacity >= img.rgb.size()) std::memcpy(rgb, img.rgb.data(), sizeof(float) * img.rgb.size());
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

}  // extern "C"

extern "C" {

int nsdf_host_sample_near_surface(const char* field, uint64_t count, int gaussian, double amount, uint64_t seed,
                                  double* out) {
  try {
    auto f = field_of(field);
    Rng rng(seed);
    fields::SurfaceNoise noise;
    noise.kind = gaussian ? fields::SurfaceNoise::Kind::gaussian : fields::SurfaceNoise::Kind::uniform;
    noise.amount = amount;
    const auto pts = fields::sample_near_surface(*f, size_t(count), noise, rng);
    for (size_t i = 0; i < pts.size(); ++i) put_vec(pts[i], out + 3 * i);
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

int nsdf_host_sup_diff(const char* f_src, const char* g_src, uint64_t n_uniform, uint64_t n_surface, double margin,
                       double noise_halfwidth, uint64_t seed, double* out) {
  try {
    auto g = field_of(g_src);
    auto f = field_of(f_src, &g->domain());
    fields::SupSamplerConfig cfg;
    cfg.n_uniform = size_t(n_uniform);
    cfg.n_surface = size_t(n_surface);
    cfg.margin = margin;
    cfg.noise_halfwidth = noise_halfwidth;
    cfg.seed = seed;
    const auto r = fields::estimate_sup_diff(*f, *g, cfg);
    out[0] = r.eps;
    out[1] = r.raw_max;
    put_vec(r.argmax, out + 2);
    out[5] = double(r.samples);
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

int nsdf_host_verify_nesting(const char* manifest, double time, uint64_t samples, uint64_t seed,
                             uint64_t max_recorded, uint64_t* counts, double* recorded) {
  try {
    const auto seq = sequence_of(manifest, time);
    fields::VerifyConfig cfg;
    cfg.samples = size_t(samples);
    cfg.seed = seed;
    cfg.max_recorded_violations = size_t(max_recorded);
    const auto r = fields::verify_nesting(seq, cfg);
    counts[0] = r.samples_total;
    counts[1] = r.checked;
    counts[2] = r.violation_count;
    counts[3] = r.violations.size();
    for (size_t i = 0; i < r.violations.size(); ++i) {
      double* o = recorded + 6 * i;
      put_vec(r.violations[i].point, o);
      o[3] = double(r.violations[i].pair_index);
      o[4] = r.violations[i].f_coarse;
      o[5] = r.violations[i].f_fine;
    }
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

}  // extern "C"

extern "C" {

int nsdf_host_sample_training_set(const char* oracle, uint64_t n_uniform, uint64_t n_surface, double sigma,
                                  uint64_t n_validation, uint64_t seed, double* points_out, double* targets_out,
                                  double* val_points_out, double* val_targets_out) {
  try {
    auto f = field_of(oracle);
    trainer::SampleConfig sc;
    sc.n_uniform = size_t(n_uniform);
    sc.n_surface = size_t(n_surface);
    sc.sigma = sigma;
    sc.n_validation = size_t(n_validation);
    sc.seed = seed;
    const auto set = trainer::sample_training_set(*f, sc);
    std::memcpy(points_out, set.points.data(), set.points.size() * 8);
    std::memcpy(targets_out, set.targets.data(), set.targets.size() * 8);
    std::memcpy(val_points_out, set.val_points.data(), set.val_points.size() * 8);
    std::memcpy(val_targets_out, set.val_targets.data(), set.val_targets.size() * 8);
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

static trainer::TrainingSet training_set(int input_dim, const double* points, const double* targets, int n,
                                         const double* val_points, const double* val_targets, int n_val) {
  trainer::TrainingSet set;
  set.input_dim = input_dim;
  set.points = tensor::Matrix<double>(input_dim, n, std::vector<double>(points, points + size_t(input_dim) * n));
  set.targets = tensor::Matrix<double>(1, n, std::vector<double>(targets, targets + n));
  set.val_points = tensor::Matrix<double>(input_dim, n_val,
                                          std::vector<double>(val_points, val_points + size_t(input_dim) * n_val));
  set.val_targets = tensor::Matrix<double>(1, n_val, std::vector<double>(val_targets, val_targets + n_val));
  return set;
}

static void put_params(const mlp::MlpParams<double>& p, double* out) {
  size_t o = 0;
  for (const auto& l : p.layers) {
    std::memcpy(out + o, l.weights.data(), l.weights.size() * 8);
    o += l.weights.size();
    std::memcpy(out + o, l.bias.data(), l.bias.size() * 8);
    o += l.bias.size();
  }
}

int nsdf_host_fit_mlp(const char* arch, int input_dim, double omega0, uint64_t seed, const nsdf_train_config* cfg,
                      const double* points, const double* targets, int n, const double* val_points,
                      const double* val_targets, int n_val, double* params_out, double* epoch_loss,
                      nsdf_train_report* report) {
  try {
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
    const auto fit = trainer::fit_mlp(tc, training_set(input_dim, points, targets, n, val_points, val_targets, n_val));
    put_params(fit.params, params_out);
    std::memset(report, 0, sizeof(*report));
    for (size_t i = 0; i < fit.report.epoch_loss.size(); ++i) epoch_loss[i] = fit.report.epoch_loss[i];
    report->epochs_recorded = int(fit.report.epoch_loss.size());
    report->final_loss = fit.report.final_loss;
    report->validation_mse = fit.report.validation_mse;
    report->validation_max_error = fit.report.validation_max_error;
    report->final_learning_rate = fit.report.final_learning_rate;
    report->diverged = fit.report.diverged ? 1 : 0;
    report->halvings = fit.report.halvings;
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

int nsdf_host_backprop(const char* arch, int input_dim, double omega0, uint64_t seed, const double* points,
                       const double* targets, int k, double* params_out, double* grads_out, double* loss) {
  try {
    Rng rng(seed);
    const auto params = mlp::random_init(mlp::parse_architecture(arch, input_dim), omega0, rng);
    put_params(params, params_out);
    const auto g = trainer::backprop_sine_mlp(
        params, tensor::Matrix<double>(input_dim, k, std::vector<double>(points, points + size_t(input_dim) * k)),
        tensor::Matrix<double>(1, k, std::vector<double>(targets, targets + k)), loss);
    size_t o = 0;
    for (const auto& l : g.layers) {
      std::memcpy(grads_out + o, l.weights.data(), l.weights.size() * 8);
      o += l.weights.size();
      std::memcpy(grads_out + o, l.bias.data(), l.bias.size() * 8);
      o += l.bias.size();
    }
    return NSDF_OK;
  } catch (const std::exception& e) {
    return fail_from(e);
  }
}

}  // extern "C"
