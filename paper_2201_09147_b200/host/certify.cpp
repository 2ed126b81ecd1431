// Certification on the B200: near-surface sampling, sup-norm
// deviation estimation and empirical nesting verification (nesting.cpp:96-361).
//
// The reference evaluates these in double precision, 16384 points per chunk on its CPU
// thread pool.  Here every Field batch call covers a whole sample set at once, so a neural
// field's FP64 evaluation is one device launch (mlp_f64.cu, bit-exact with the reference's
// double kernels); analytic fields evaluate on the host exactly as in the reference.  Every
// per-point quantity is independent of the chunking, and the chunk-ordered reductions of the
// reference (first maximum in chunk order, violations recorded in chunk order) are the same
// as a single in-order scan, so the results — sample sets, maxima, argmax, counts, recorded
// violations — are identical to the reference's for the same seeds.
#include <algorithm>
#include <cmath>

#include "nsdf/fields/nesting.hpp"

namespace nsdf::fields {

namespace {

constexpr int kProjectionSteps = 4;  // nesting.cpp:94

Matrix<double> as_matrix(const std::vector<Vec3>& pts, size_t lo, size_t hi) {
  Matrix<double> p(3, int(hi - lo));
  for (size_t j = lo; j < hi; ++j) {
    p(0, int(j - lo)) = pts[j].x;
    p(1, int(j - lo)) = pts[j].y;
    p(2, int(j - lo)) = pts[j].z;
  }
  return p;
}

// Newton projection onto the zero set along the gradient, then the acceptance test
// (project_chunk, nesting.cpp:98-127).  Accepted points keep the input order.
void project(const Field& field, std::vector<Vec3>& pts, double keep_tol) {
  const int k = int(pts.size());
  Matrix<double> p = as_matrix(pts, 0, pts.size());
  for (int step = 0; step < kProjectionSteps; ++step) {
    const Matrix<double> d = field.eval_batch(p);
    const Matrix<double> g = field.grad_batch(p);
    for (int j = 0; j < k; ++j) {
      const double gx = g(0, j), gy = g(1, j), gz = g(2, j);
      const double n2 = gx * gx + gy * gy + gz * gz;
      if (n2 < 1e-16) continue;
      const double s = d(0, j) / n2;
      p(0, j) -= s * gx;
      p(1, j) -= s * gy;
      p(2, j) -= s * gz;
    }
  }
  const Matrix<double> d = field.eval_batch(p);
  std::vector<Vec3> accepted;
  accepted.reserve(pts.size());
  for (int j = 0; j < k; ++j)
    if (std::abs(d(0, j)) <= keep_tol) accepted.push_back({p(0, j), p(1, j), p(2, j)});
  pts = std::move(accepted);
}

}  // namespace

std::vector<Vec3> sample_near_surface(const Field& field, size_t count, SurfaceNoise noise, Rng& rng) {
  // nesting.cpp:131-200
  std::vector<Vec3> result;
  result.reserve(count);
  const Aabb& box = field.domain();
  const double keep_tol = 2e-3 * box.diameter();
  int empty_rounds = 0;
  while (result.size() < count && empty_rounds < 8) {
    const size_t want = count - result.size();
    const size_t batch = std::min<size_t>(std::max<size_t>(want + want / 4, 4096), size_t(1) << 20);
    std::vector<Vec3> surface(batch);
    for (auto& c : surface) c = rng.uniform_in_box(box);
    project(field, surface, keep_tol);
    if (surface.empty()) {
      ++empty_rounds;
      continue;
    }
    const Matrix<double> grads = field.grad_batch(as_matrix(surface, 0, surface.size()));
    for (size_t j = 0; j < surface.size() && result.size() < count; ++j) {
      const Vec3 g{grads(0, int(j)), grads(1, int(j)), grads(2, int(j))};
      const double n = g.norm();
      if (n < 1e-12) continue;
      const double offset = noise.kind == SurfaceNoise::Kind::uniform ? rng.uniform(-noise.amount, noise.amount)
                                                                       : rng.normal(0.0, noise.amount);
      result.push_back(surface[j] + g * (offset / n));
    }
  }
  if (result.size() < count)
    throw Error(ErrorKind::divergence, "surface sampling kept only " + std::to_string(result.size()) + " of " +
                                           std::to_string(count) + " requested points for " + field.describe());
  return result;
}

SupDiffResult estimate_sup_diff(const Field& f, const Field& g, const SupSamplerConfig& config) {
  // nesting.cpp:235-260 (+ max_abs_diff, :206-231)
  if (config.n_uniform + config.n_surface < 1000)
    throw Error(ErrorKind::config, "sup-norm estimation needs at least 1000 samples, got " +
                                       std::to_string(config.n_uniform + config.n_surface));
  Rng rng(config.seed);
  std::vector<Vec3> pts;
  pts.reserve(config.n_uniform + config.n_surface);
  const Aabb& box = g.domain();
  for (size_t i = 0; i < config.n_uniform; ++i) pts.push_back(rng.uniform_in_box(box));
  if (config.n_surface) {
    try {
      auto near = sample_near_surface(g, config.n_surface, {SurfaceNoise::Kind::uniform, config.noise_halfwidth}, rng);
      pts.insert(pts.end(), near.begin(), near.end());
    } catch (const Error&) {
      for (size_t i = 0; i < config.n_surface; ++i) pts.push_back(rng.uniform_in_box(box));
    }
  }
  SupDiffResult result;
  result.samples = pts.size();
  double best = -1.0;
  Vec3 arg;
  if (!pts.empty()) {
    const Matrix<double> p = as_matrix(pts, 0, pts.size());
    const Matrix<double> df = f.eval_batch(p);
    const Matrix<double> dg = g.eval_batch(p);
    for (size_t j = 0; j < pts.size(); ++j) {
      const double d = std::abs(df(0, int(j)) - dg(0, int(j)));
      if (d > best) {
        best = d;
        arg = pts[j];
      }
    }
  }
  result.raw_max = std::max(best, 0.0);
  result.argmax = arg;
  result.eps = result.raw_max + config.margin;
  return result;
}

NestingReport verify_nesting(const NestedSequence& seq, const VerifyConfig& config) {
  // nesting.cpp:266-361
  seq.validate();
  if (config.samples < 100000)
    throw Error(ErrorKind::contract,
                "nesting verification needs at least 1e5 samples, got " + std::to_string(config.samples));
  const size_t m = seq.size();
  NestingReport report;
  report.samples_total = config.samples;
  if (m < 2) return report;

  Rng rng(config.seed);
  std::vector<Vec3> pts;
  pts.reserve(config.samples);
  const Aabb& box = seq.field(m - 1).domain();
  const size_t n_uniform = config.samples / 2;
  for (size_t i = 0; i < n_uniform; ++i) pts.push_back(rng.uniform_in_box(box));
  const size_t n_surface = config.samples - n_uniform;
  const size_t per_field = n_surface / m;
  for (size_t fi = 0; fi < m; ++fi) {
    const size_t quota = fi + 1 == m ? n_surface - per_field * (m - 1) : per_field;
    try {
      auto near = sample_near_surface(seq.field(fi), quota, {SurfaceNoise::Kind::uniform, 0.1}, rng);
      pts.insert(pts.end(), near.begin(), near.end());
    } catch (const Error&) {
      for (size_t i = 0; i < quota; ++i) pts.push_back(rng.uniform_in_box(box));
    }
  }

  const Matrix<double> p = as_matrix(pts, 0, pts.size());
  for (size_t pair = 0; pair + 1 < m; ++pair) {
    const Field& coarse = seq.field(pair);
    const Field& fine = seq.field(pair + 1);
    const double delta_coarse = seq.deltas[pair];
    const double delta_fine = seq.deltas[pair + 1];
    const Matrix<double> df = fine.eval_batch(p);
    std::vector<int> inside;
    for (int j = 0; j < p.cols(); ++j)
      if (std::abs(df(0, j)) <= delta_fine) inside.push_back(j);
    report.checked += inside.size();
    if (inside.empty()) continue;
    Matrix<double> q(3, int(inside.size()));
    for (size_t jj = 0; jj < inside.size(); ++jj)
      for (int r = 0; r < 3; ++r) q(r, int(jj)) = p(r, inside[jj]);
    const Matrix<double> dc = coarse.eval_batch(q);
    for (size_t jj = 0; jj < inside.size(); ++jj) {
      if (std::abs(dc(0, int(jj))) > delta_coarse) {
        ++report.violation_count;
        if (report.violations.size() < config.max_recorded_violations)
          report.violations.push_back({pts[size_t(inside[jj])], pair, dc(0, int(jj)), df(0, inside[jj])});
      }
    }
  }
  return report;
}

}  // namespace nsdf::fields
