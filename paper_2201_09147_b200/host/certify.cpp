// Certification on the B200: near-surface sampling, sup-norm
// deviation estimation and empirical nesting verification (reference: nesting.cpp:96-361).
//
// Device-resident where the work is: the Newton projection of sample_near_surface keeps the
// candidate points on the GPU for all its steps (nsdf_cuda_project_to_surface: one H2D of
// the candidates, one D2H of the kept points and their gradients per round); sup-norm and
// nesting checks evaluate whole sample sets in single FP64 device launches.  The host keeps
// only what is inherently sequential: the RNG stream (xoshiro256++, consumed in the
// reference's order) and the in-order reductions.  Every per-point quantity is independent
// of how points are batched, and a single in-order scan equals the reference's chunk-ordered
// merges (first maximum, violations in order), so every result — sample sets, maxima,
// argmax, counts, recorded violations — is bit-identical to the reference's.
#include <algorithm>
#include <cmath>

#include "engine.hpp"
#include "nsdf/fields/nesting.hpp"

namespace nsdf::fields {

namespace {

constexpr int kNewtonSteps = 4;  // nesting.cpp:94

// 3 x n column matrix of a point list (one point per column, matrix.hpp:32-33)
Matrix<double> columns_of(const std::vector<Vec3>& v) {
  Matrix<double> m(3, int(v.size()));
  for (int j = 0; j < int(v.size()); ++j) {
    m(0, j) = v[size_t(j)].x;
    m(1, j) = v[size_t(j)].y;
    m(2, j) = v[size_t(j)].z;
  }
  return m;
}

Vec3 column(const Matrix<double>& m, int j) { return {m(0, j), m(1, j), m(2, j)}; }

// Projected candidates that passed the acceptance test, with the field gradient at each.
struct Surface {
  std::vector<Vec3> points, grads;
};

Surface project_on_device(const DeviceBinding& b, const std::vector<Vec3>& cand, double tol) {
  static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");
  Surface s;
  s.points.resize(cand.size());
  s.grads.resize(cand.size());
  int kept = 0;
  engine::check(nsdf_cuda_project_to_surface(engine::context(), b.handle, b.time64,
                                             reinterpret_cast<const double*>(cand.data()), int(cand.size()), tol,
                                             kNewtonSteps, reinterpret_cast<double*>(s.points.data()),
                                             reinterpret_cast<double*>(s.grads.data()), &kept));
  s.points.resize(size_t(kept));
  s.grads.resize(size_t(kept));
  return s;
}

// Fields without a device binding (user subclasses): the same steps through the field's own
// batch evaluation — Newton updates p -= (f / |g|^2) g, separately rounded, skipped where
// |g|^2 < 1e-16; acceptance |f| <= tol; the gradient at the accepted points.
Surface project_on_host(const Field& field, const std::vector<Vec3>& cand, double tol) {
  Matrix<double> p = columns_of(cand);
  for (int step = 0; step < kNewtonSteps; ++step) {
    const Matrix<double> f = field.eval_batch(p);
    const Matrix<double> g = field.grad_batch(p);
    for (int j = 0; j < p.cols(); ++j) {
      const Vec3 gj = column(g, j);
      const double n2 = gj.x * gj.x + gj.y * gj.y + gj.z * gj.z;
      if (n2 < 1e-16) continue;
      const double s = f(0, j) / n2;
      p(0, j) -= s * gj.x;
      p(1, j) -= s * gj.y;
      p(2, j) -= s * gj.z;
    }
  }
  const Matrix<double> f = field.eval_batch(p);
  Surface out;
  for (int j = 0; j < p.cols(); ++j)
    if (std::abs(f(0, j)) <= tol) out.points.push_back(column(p, j));
  if (!out.points.empty()) {
    const Matrix<double> g = field.grad_batch(columns_of(out.points));
    for (int j = 0; j < g.cols(); ++j) out.grads.push_back(column(g, j));
  }
  return out;
}

// uniform draws in a box, appended in RNG order
void draw_uniform(Rng& rng, const Aabb& box, size_t n, std::vector<Vec3>& out) {
  for (size_t i = 0; i < n; ++i) out.push_back(rng.uniform_in_box(box));
}

// near-surface samples of `field`, or uniform ones if its zero set cannot be sampled
// (estimate_sup_diff / verify_nesting, nesting.cpp:243-250, 283-294)
void draw_near_or_uniform(const Field& field, size_t n, double amount, Rng& rng, const Aabb& box,
                          std::vector<Vec3>& out) {
  try {
    const auto near = sample_near_surface(field, n, {SurfaceNoise::Kind::uniform, amount}, rng);
    out.insert(out.end(), near.begin(), near.end());
  } catch (const Error&) {
    draw_uniform(rng, box, n, out);
  }
}

}  // namespace

std::vector<Vec3> sample_near_surface(const Field& field, size_t count, SurfaceNoise noise, Rng& rng) {
  const Aabb& box = field.domain();
  const double tol = 2e-3 * box.diameter();
  DeviceBinding b;
  const bool on_device = field.device_binding(b);
  std::vector<Vec3> out;
  out.reserve(count);
  // rounds of uniform candidates, each projected and offset along the gradient; eight rounds
  // in a row without a single accepted point end the search
  for (int barren = 0; out.size() < count && barren < 8;) {
    const size_t need = count - out.size();
    const size_t batch = std::min<size_t>(std::max<size_t>(need + need / 4, 4096), size_t(1) << 20);
    std::vector<Vec3> cand;
    cand.reserve(batch);
    draw_uniform(rng, box, batch, cand);
    const Surface s = on_device ? project_on_device(b, cand, tol) : project_on_host(field, cand, tol);
    if (s.points.empty()) {
      ++barren;
      continue;
    }
    for (size_t j = 0; j < s.points.size() && out.size() < count; ++j) {
      const double len = s.grads[j].norm();
      if (len < 1e-12) continue;
      const double offset = noise.kind == SurfaceNoise::Kind::uniform ? rng.uniform(-noise.amount, noise.amount)
                                                                       : rng.normal(0.0, noise.amount);
      out.push_back(s.points[j] + s.grads[j] * (offset / len));
    }
  }
  if (out.size() < count)
    throw Error(ErrorKind::divergence, "surface sampling kept only " + std::to_string(out.size()) + " of " +
                                           std::to_string(count) + " requested points for " + field.describe());
  return out;
}

SupDiffResult estimate_sup_diff(const Field& f, const Field& g, const SupSamplerConfig& config) {
  if (config.n_uniform + config.n_surface < 1000)
    throw Error(ErrorKind::config, "sup-norm estimation needs at least 1000 samples, got " +
                                       std::to_string(config.n_uniform + config.n_surface));
  Rng rng(config.seed);
  const Aabb& box = g.domain();
  std::vector<Vec3> pts;
  pts.reserve(config.n_uniform + config.n_surface);
  draw_uniform(rng, box, config.n_uniform, pts);
  if (config.n_surface > 0) draw_near_or_uniform(g, config.n_surface, config.noise_halfwidth, rng, box, pts);
  SupDiffResult r;
  r.samples = pts.size();
  // the FIRST point attaining max |f - g| (strict > in point order; NaNs never win)
  double best = -1.0;
  size_t at = pts.size();
  if (!pts.empty()) {
    const Matrix<double> p = columns_of(pts);
    const Matrix<double> df = f.eval_batch(p), dg = g.eval_batch(p);
    for (int j = 0; j < p.cols(); ++j)
      if (const double d = std::abs(df(0, j) - dg(0, j)); d > best) {
        best = d;
        at = size_t(j);
      }
  }
  r.raw_max = std::max(best, 0.0);
  r.argmax = at < pts.size() ? pts[at] : Vec3{};
  r.eps = r.raw_max + config.margin;
  return r;
}

NestingReport verify_nesting(const NestedSequence& seq, const VerifyConfig& config) {
  seq.validate();
  if (config.samples < 100000)
    throw Error(ErrorKind::contract,
                "nesting verification needs at least 1e5 samples, got " + std::to_string(config.samples));
  NestingReport report;
  report.samples_total = config.samples;
  const size_t m = seq.size();
  if (m < 2) return report;
  // one shared sample set: half uniform in the finest member's box, half near the members'
  // zero sets (an equal quota each, the remainder to the finest)
  Rng rng(config.seed);
  const Aabb& box = seq.field(m - 1).domain();
  std::vector<Vec3> pts;
  pts.reserve(config.samples);
  const size_t n_uniform = config.samples / 2, n_surface = config.samples - n_uniform, quota = n_surface / m;
  draw_uniform(rng, box, n_uniform, pts);
  for (size_t i = 0; i < m; ++i)
    draw_near_or_uniform(seq.field(i), i + 1 == m ? n_surface - quota * (m - 1) : quota, 0.1, rng, box, pts);
  const Matrix<double> p = columns_of(pts);
  for (size_t pair = 0; pair + 1 < m; ++pair) {
    // points inside the fine member's delta-neighbourhood must lie inside the coarse one's
    const Matrix<double> df = seq.field(pair + 1).eval_batch(p);
    std::vector<int> inside;
    for (int j = 0; j < p.cols(); ++j)
      if (std::abs(df(0, j)) <= seq.deltas[pair + 1]) inside.push_back(j);
    report.checked += inside.size();
    if (inside.empty()) continue;
    Matrix<double> q(3, int(inside.size()));
    for (int jj = 0; jj < q.cols(); ++jj)
      for (int r = 0; r < 3; ++r) q(r, jj) = p(r, inside[size_t(jj)]);
    const Matrix<double> dc = seq.field(pair).eval_batch(q);
    for (int jj = 0; jj < q.cols(); ++jj) {
      if (std::abs(dc(0, jj)) <= seq.deltas[pair]) continue;
      ++report.violation_count;
      if (report.violations.size() < config.max_recorded_violations) {
        const int j = inside[size_t(jj)];
        report.violations.push_back({pts[size_t(j)], pair, dc(0, jj), df(0, j)});
      }
    }
  }
  return report;
}

}  // namespace nsdf::fields
