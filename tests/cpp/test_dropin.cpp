// Reference-style checks of the drop-in C++ API (include/nsdf/*.hpp) running on the B200.
// Cases follow the reference's own suites (proj/tests/test_mlp.cpp, test_tracer.cpp,
// test_shading.cpp); file:line of the originals is given per case.  Run with
// NSDF_MODE=oracle for the bit-exact assertions.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <filesystem>
#include <map>

#include "check.hpp"
#include "nsdf/shading/shading.hpp"
#include "nsdf/tensor/ops.hpp"
#include "nsdf/fields/nesting.hpp"

using namespace nsdf;
using fields::NestedSequence;
using fields::SphereField;
using tensor::Matrix;
using namespace nsdf::tracer;

namespace {

mlp::MlpParams<double> linear(std::vector<double> w, double b) {
  mlp::MlpParams<double> p;
  p.input_dim = int(w.size());
  p.activation = tensor::ActivationSpec::identity();
  p.layers.push_back({Matrix<double>(1, int(w.size()), w), Matrix<double>(1, 1, {b})});
  return p;
}

Ray axis_ray(Vec3 origin, Vec3 toward) { return {Vec3f::from(origin), Vec3f::from((toward - origin).normalized())}; }

NestedSequence spheres(std::vector<double> radii, std::vector<double> deltas) {
  NestedSequence s;
  for (double r : radii) s.entries.push_back({std::make_shared<SphereField>(Vec3{0, 0, 0}, r), {}, "s", 0});
  s.deltas = std::move(deltas);
  return s;
}

Matrix<float> random_points(int k, uint64_t seed) {
  Rng rng(seed);
  Matrix<float> m(3, k);
  for (auto& v : m.storage()) v = float(rng.uniform(-1, 1));
  return m;
}

}  // namespace

TEST_CASE("forward: single affine layer picks out a coordinate (test_mlp.cpp:64-68)") {
  auto p = linear({1, 0, 0}, 0.0).cast<float>();
  CHECK(mlp::forward_batch(p, Matrix<float>(3, 1, {2, 0, 0}))(0, 0) == 2.0f);
}

TEST_CASE("gradient of a linear network is its weight row (test_mlp.cpp:82-91)") {
  auto p = linear({0.5, -2.0, 3.25}, 1.0).cast<float>();
  auto g = mlp::gradient_batch(p, random_points(7, 8));
  for (int j = 0; j < 7; ++j) CHECK(g(0, j) == 0.5f && g(1, j) == -2.0f && g(2, j) == 3.25f);
}

TEST_CASE("hand-sized sine network gradient at the origin (test_mlp.cpp:93-111)") {
  mlp::MlpParams<double> p;
  p.activation = tensor::ActivationSpec::sine(2.0);
  p.layers.push_back({Matrix<double>{{1, 2, 3}, {4, 5, 6}}, Matrix<double>{{0.1}, {-0.2}}});
  p.layers.push_back({Matrix<double>{{0.5, -1.5}}, Matrix<double>{{0.3}}});
  auto g = mlp::gradient_batch(p.cast<float>(), Matrix<float>(3, 1));
  for (int c = 0; c < 3; ++c) {
    const double want = 0.5 * 2 * std::cos(0.2) * p.layers[0].weights(0, c) +
                        (-1.5) * 2 * std::cos(-0.4) * p.layers[0].weights(1, c);
    CHECK_NEAR(g(c, 0), want, 2e-5 * std::abs(want) + 1e-6);
  }
}

TEST_CASE("fused evaluation is bitwise equal to the separate calls (test_mlp.cpp:128-137)") {
  for (int it = 0; it < 12; ++it) {
    Rng rng(300 + it);
    auto net = mlp::random_init({4 + (it % 3) * 4, 1 + it % 2, 3}, 30.0, rng).cast<float>();
    auto pts = random_points(1 + it % 5, 400 + it);
    auto [d, g] = mlp::forward_and_gradient_batch(net, pts);
    CHECK(d == mlp::forward_batch(net, pts));
    CHECK(g == mlp::gradient_batch(net, pts));
  }
}

TEST_CASE("batch width invariance and single point == batch (test_tensor.cpp:283-309, test_mlp.cpp:182-202)") {
  Rng rng(9);
  auto net = mlp::random_init({128, 2, 3}, 30.0, rng).cast<float>();
  auto pts = random_points(300, 10);
  auto all = mlp::forward_batch(net, pts);
  for (int j = 0; j < 300; j += 37) {
    Matrix<float> one(3, 1, {pts(0, j), pts(1, j), pts(2, j)});
    CHECK(mlp::forward_batch(net, one)(0, 0) == all(0, j));
  }
}

TEST_CASE("validation and contract errors") {
  mlp::MlpParams<float> empty;
  CHECK_THROWS(mlp::forward_batch(empty, Matrix<float>(3, 1)));
  auto p = linear({1, 0, 0}, 0).cast<float>();
  CHECK_THROWS(mlp::forward_batch(p, Matrix<float>(2, 1)));
  CHECK_THROWS(mlp::parse_architecture("64"));
  CHECK(mlp::parse_architecture("256x3").parameter_count() == 198657u);
  // f64 batches run on the device FP64 path (certification): a linear net is exact
  CHECK(mlp::forward_batch(linear({1, 0, 0}, 0), Matrix<double>(3, 1, {2.0, 0.0, 0.0}))(0, 0) == 2.0);
  CHECK_THROWS(mlp::forward_batch(linear({1, 0, 0}, 0), Matrix<double>(2, 1)));
}

TEST_CASE("classic sphere tracing hits the surface and the offset surface (test_tracer.cpp:74-87)") {
  SphereField sphere({0, 0, 0}, 1.0);
  const Ray ray = axis_ray({3, 0, 0}, {-1, 0, 0});
  HitRecord hit = sphere_trace(sphere, ray, 0.0f, 1e-3f, 100);
  CHECK(hit.hit);
  CHECK_NEAR(hit.point.x, 1.0, 2e-3);
  CHECK_NEAR(hit.t, 2.0, 4e-3);
  CHECK(hit.final_distance <= 1e-3f);
  HitRecord off = sphere_trace(sphere, ray, 0.1f, 1e-3f, 100);
  CHECK(off.hit);
  CHECK_NEAR(off.point.x, 1.1, 2.2e-3);
}

TEST_CASE("multiscale trace on certified concentric spheres (test_tracer.cpp:104-121)") {
  auto seq = spheres({1.0, 0.95}, {0.1, 0.05});
  TraceConfig cfg;
  cfg.budgets = {50, 50};
  HitRecord hit = multiscale_sphere_trace(seq, axis_ray({3, 0, 0}, {0, 0, 0}), cfg);
  CHECK(hit.hit);
  CHECK(hit.level_reached == 1);
  CHECK_NEAR(hit.point.x, 0.95, 2e-3);
  CHECK(hit.iterations_used[0] > 0 && hit.iterations_used[1] > 0);
}

TEST_CASE("a single-level sequence is classic sphere tracing bit for bit (test_tracer.cpp:123-141)") {
  auto seq = spheres({0.8}, {0.05});
  TraceConfig cfg;
  cfg.budgets = {60};
  Rng rng(5);
  for (int i = 0; i < 20; ++i) {
    const Vec3 o{rng.uniform(2, 3), rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5)};
    const Vec3 to{rng.uniform(-0.2, 0.2), rng.uniform(-0.2, 0.2), rng.uniform(-0.2, 0.2)};
    const Ray ray = axis_ray(o, to);
    HitRecord a = multiscale_sphere_trace(seq, ray, cfg);
    HitRecord b = sphere_trace(seq.field(0), ray, 0.0f, cfg.eps_stop, 60);
    CHECK(a.hit == b.hit && a.point.x == b.point.x && a.point.y == b.point.y && a.point.z == b.point.z);
    CHECK(a.t == b.t && a.final_distance == b.final_distance);
  }
}

TEST_CASE("budget exhaustion, trailing zero budget, origin inside the shell (test_tracer.cpp:185-192, 281-307)") {
  auto one = spheres({1.0}, {0.05});
  TraceConfig b1;
  b1.budgets = {1};
  HitRecord miss = multiscale_sphere_trace(one, axis_ray({4, 0.3, 0}, {0, 0.3, 0}), b1);
  CHECK(!miss.hit && miss.iterations_used[0] == 1 && miss.t > 0);
  auto con = spheres({1.0, 0.95}, {0.1, 0.05});
  TraceConfig trailing;
  trailing.budgets = {50, 0};
  HitRecord h = multiscale_sphere_trace(con, axis_ray({3, 0, 0}, {0, 0, 0}), trailing);
  CHECK(h.hit && h.iterations_used[1] == 0);
  CHECK_NEAR(h.point.x, 1.0, 2e-3);
  TraceConfig zero;
  zero.budgets = {0, 0};
  CHECK_THROWS(multiscale_sphere_trace(con, axis_ray({3, 0, 0}, {0, 0, 0}), zero));
  TraceConfig c30;
  c30.budgets = {30, 30};
  HitRecord in = multiscale_sphere_trace(con, axis_ray({1.05, 0, 0}, {-1, 0, 0}), c30);
  CHECK(in.hit && in.iterations_used[0] == 1);
  CHECK_NEAR(in.point.x, 0.95, 2e-3);
}

TEST_CASE("trace_image: empty view, filled disc, per-ray equivalence (test_tracer.cpp:194-244)") {
  auto seq = spheres({0.7}, {0.05});
  TraceConfig cfg;
  cfg.budgets = {60};
  Camera away;
  away.position = {0, 0, 3};
  away.look_at = {0, 0, 6};
  away.width = away.height = 32;
  for (const auto& r : trace_image(seq, away, cfg)) CHECK(!r.hit);
  Camera cam;
  cam.position = {0, 0, 3};
  cam.width = cam.height = 129;
  cam.vertical_fov_deg = 40;
  auto recs = trace_image(seq, cam, cfg);
  const double screen = std::tan(std::asin(0.7 / 3.0)) / std::tan(cam.vertical_fov_deg * M_PI / 360.0);
  int first = -1, last = -1;
  for (int x = 0; x < cam.width; ++x)
    if (recs[size_t(64) * cam.width + x].hit) {
      if (first < 0) first = x;
      last = x;
    }
  CHECK(first >= 0);
  CHECK(std::abs((last - first + 1) / 2.0 - screen * cam.height / 2.0) <= 1.0);
  auto rays = generate_rays(cam);
  for (size_t i = 0; i < recs.size(); i += 37) {
    HitRecord one = multiscale_sphere_trace(seq, rays[i], cfg);
    CHECK(one.hit == recs[i].hit);
    if (one.hit) CHECK(one.point.x == recs[i].point.x && one.t == recs[i].t);
  }
}

TEST_CASE("ray generation geometry (test_tracer.cpp:38-72)") {
  Camera cam;
  cam.width = cam.height = 101;
  auto rays = generate_rays(cam);
  CHECK(rays.size() == 101u * 101u);
  const auto& c = rays[50 * 101 + 50].direction;
  CHECK(std::abs(c.x) < 1e-6 && std::abs(c.y) < 1e-6 && std::abs(c.z + 1) < 1e-6);
  Camera bad = cam;
  bad.width = 0;
  CHECK_THROWS(generate_rays(bad));
}

TEST_CASE("analytic-sphere render: unit normals, parallel level sets (test_shading.cpp:142-165, 197-213)") {
  auto seq = spheres({0.7}, {0.05});
  Camera cam;
  cam.width = cam.height = 64;
  shading::RenderConfig cfg;
  cfg.trace.budgets = {80};
  auto img = shading::render(seq, cam, cfg);
  size_t hits = 0;
  for (auto m : img.mask) hits += m;
  CHECK(hits > 300);
  Matrix<float> pts(3, 4, {0.7f, 0, 0, -0.8f, 0, 0.7f, 0, 0, 0, 0, 0.7f, 0});
  auto r = shading::neural_normal_map(seq.field(0), pts, 0.05);
  for (int j = 0; j < 4; ++j) {
    const double n = std::sqrt(double(r.normals(0, j)) * r.normals(0, j) + double(r.normals(1, j)) * r.normals(1, j) +
                               double(r.normals(2, j)) * r.normals(2, j));
    CHECK_NEAR(n, 1.0, 1e-6);
  }
  CHECK(r.normals(0, 0) > 0.999f);
  CHECK(r.outside_count == 1);  // (-0.8, 0, 0): |f| = 0.1 > delta
}

TEST_CASE("self-mapped normals reproduce the own-normal render exactly (test_shading.cpp:332-349)") {
  auto seq = spheres({0.7}, {0.05});
  Camera cam;
  cam.width = cam.height = 48;
  shading::RenderConfig own;
  own.trace.budgets = {60};
  shading::RenderConfig mapped = own;
  mapped.normal_source = shading::NormalSource::mapped;
  CHECK(shading::image_mse(shading::render(seq, cam, own), shading::render(seq, cam, mapped)) == 0.0);
}

// The reference test suite's icosphere builder (test_shading.cpp:74-112), restated.
shading::Mesh test_icosphere(int subdivisions, double radius) {
  const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
  std::vector<Vec3> v = {{-1, phi, 0}, {1, phi, 0}, {-1, -phi, 0}, {1, -phi, 0}, {0, -1, phi}, {0, 1, phi},
                         {0, -1, -phi}, {0, 1, -phi}, {phi, 0, -1}, {phi, 0, 1}, {-phi, 0, -1}, {-phi, 0, 1}};
  for (auto& x : v) x = x.normalized();
  std::vector<std::array<int, 3>> f = {{0, 11, 5}, {0, 5, 1},  {0, 1, 7},   {0, 7, 10}, {0, 10, 11},
                                       {1, 5, 9},  {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
                                       {3, 9, 4},  {3, 4, 2},  {3, 2, 6},   {3, 6, 8},  {3, 8, 9},
                                       {4, 9, 5},  {2, 4, 11}, {6, 2, 10},  {8, 6, 7},  {9, 8, 1}};
  for (int s = 0; s < subdivisions; ++s) {
    std::map<std::pair<int, int>, int> memo;
    auto mid = [&](int a, int b) {
      const auto key = std::minmax(a, b);
      auto it = memo.find(key);
      if (it != memo.end()) return it->second;
      v.push_back(((v[a] + v[b]) * 0.5).normalized());
      return memo[key] = int(v.size()) - 1;
    };
    std::vector<std::array<int, 3>> next;
    for (const auto& t : f) {
      const int a = mid(t[0], t[1]), b = mid(t[1], t[2]), c = mid(t[2], t[0]);
      next.push_back({t[0], a, c});
      next.push_back({t[1], b, a});
      next.push_back({t[2], c, b});
      next.push_back({a, b, c});
    }
    f = std::move(next);
  }
  shading::Mesh m;
  m.triangles = f;
  for (const auto& x : v) {
    m.normals.push_back(x);
    m.vertices.push_back(x * radius);
  }
  return m;
}

TEST_CASE("mesh normal mapping on the device (test_shading.cpp:215-261)") {
  auto mesh = test_icosphere(2, 1.0);
  SphereField sphere({0, 0, 0}, 1.0);
  auto rep = shading::map_normals_to_mesh(mesh, sphere, 0.05);
  CHECK(rep.violators == 0 && rep.mapped == mesh.vertices.size());
  for (size_t i = 0; i < mesh.vertices.size(); ++i) CHECK((mesh.normals[i] - mesh.vertices[i].normalized()).norm() < 1e-6);
  auto small = test_icosphere(1, 1.0);
  const auto original = small.normals;
  fields::TorusField far_torus(0.2, 0.05);
  rep = shading::map_normals_to_mesh(small, far_torus, 0.01);
  CHECK(rep.mapped == 0 && rep.violators == small.vertices.size());
  for (size_t i = 0; i < original.size(); ++i) CHECK((small.normals[i] - original[i]).norm() == 0);
  auto a = test_icosphere(2, 1.02), b = test_icosphere(2, 1.02);
  std::reverse(b.triangles.begin(), b.triangles.end());
  shading::map_normals_to_mesh(a, sphere, 0.1);
  shading::map_normals_to_mesh(b, sphere, 0.1);
  for (size_t i = 0; i < a.normals.size(); ++i)
    CHECK(a.normals[i].x == b.normals[i].x && a.normals[i].y == b.normals[i].y && a.normals[i].z == b.normals[i].z);
  shading::Mesh empty;
  CHECK_THROWS(shading::map_normals_to_mesh(empty, sphere, 0.1));
}

TEST_CASE("manifest + sdfnet round trip and image / mesh I/O") {
  const auto dir = std::filesystem::temp_directory_path() / "nsdf_dropin_test";
  std::filesystem::create_directories(dir);
  Rng rng(3);
  auto p = mlp::random_init({16, 1, 3}, 30.0, rng);
  mlp::save_params(p, dir / "n.sdfnet");
  auto q = mlp::load_params(dir / "n.sdfnet");
  CHECK(q.layers[1].weights == p.layers[1].weights);
  NestedSequence seq;
  fields::FieldSource src;
  src.kind = fields::FieldSource::Kind::weights;
  src.weights_path = "n.sdfnet";
  seq.entries.push_back({std::make_shared<fields::NeuralField>(p), src, "16x1", p.parameter_count()});
  seq.deltas = {0.1};
  fields::save_manifest(seq, dir / "s.nest");
  auto m = fields::load_manifest(dir / "s.nest");
  CHECK(!m.time_dependent && m.sequence.size() == 1 && m.sequence.deltas[0] == 0.1);
  shading::ImageBuffer img(4, 3);
  for (size_t i = 0; i < img.rgb.size(); ++i) img.rgb[i] = float(i % 256) / 255.0f;
  shading::write_ppm(img, dir / "a.ppm");
  CHECK(shading::image_mse(img, shading::read_ppm(dir / "a.ppm")) < 1e-10);
  shading::write_png(img, dir / "a.png");
  CHECK(std::filesystem::file_size(dir / "a.png") > 40);
  CHECK(fields::thresholds_prop2({0.3, 0.1, 0.05})[2] == 0.1 + 0.05);
}

TEST_CASE("gemm identity and hand examples (test_tensor.cpp:31-48)") {
  const Matrix<float> a{{1, 2}, {3, 4}};
  const Matrix<float> ones{{1}, {1}};
  const Matrix<float> bias{{10}, {10}};
  const Matrix<float> c = tensor::gemm(a, ones, &bias);
  CHECK(c.rows() == 2 && c.cols() == 1 && c(0, 0) == 13.0f && c(1, 0) == 17.0f);
  const Matrix<double> id{{1, 0}, {0, 1}};
  const Matrix<double> ad{{1, 2}, {3, 4}};
  const Matrix<double> r = tensor::gemm(id, ad);
  CHECK(r(0, 0) == 1.0 && r(0, 1) == 2.0 && r(1, 0) == 3.0 && r(1, 1) == 4.0);
}

TEST_CASE("tensor ops: shape errors name both shapes, sine basics, flops, backends (test_tensor.cpp:84-177, 311-323)") {
  const Matrix<float> a(2, 3), b(2, 3);
  bool named = false;
  try {
    tensor::gemm(a, b);
  } catch (const Error& e) {
    named = e.kind() == ErrorKind::contract && std::string(e.what()).find("2x3") != std::string::npos;
  }
  CHECK(named);
  CHECK_THROWS(tensor::hadamard(a, Matrix<float>(3, 2)));
  CHECK_THROWS(tensor::scale_rows(Matrix<float>(3, 1), a));
  const Matrix<float> z(1, 1);
  CHECK(tensor::activate(z, tensor::ActivationSpec::sine(1.0))(0, 0) == 0.0f);
  CHECK(tensor::activate(z, tensor::ActivationSpec::sine(1.0), true)(0, 0) == 1.0f);
  const Matrix<float> h = tensor::hadamard(Matrix<float>{{1, 2, 3}}, Matrix<float>{{4, 5, 6}});
  CHECK(h(0, 0) == 4.0f && h(0, 1) == 10.0f && h(0, 2) == 18.0f);
  const Matrix<double> s = tensor::scale_rows(Matrix<double>{{2}, {3}}, Matrix<double>{{1, 2}, {3, 4}});
  CHECK(s(0, 1) == 4.0 && s(1, 0) == 9.0);
  tensor::reset_flops();
  tensor::gemm(Matrix<float>(4, 8), Matrix<float>(8, 16));
  CHECK(tensor::flops_performed() == 2ull * 4 * 16 * 8);
  CHECK(tensor::active_backend() == tensor::Backend::b200 && tensor::backend_available(tensor::Backend::b200));
  CHECK(!tensor::backend_available(tensor::Backend::neon));
  CHECK_THROWS(tensor::set_backend(tensor::Backend::neon));
}

TEST_CASE("backend loop of the reference suite: scalar / avx2 / b200 (test_tensor.cpp:17-28, 230-280)") {
  // the reference's available_backends(): scalar always, then the SIMD backends present
  std::vector<tensor::Backend> backends{tensor::Backend::scalar};
  for (auto b : {tensor::Backend::avx2, tensor::Backend::neon})
    if (tensor::backend_available(b)) backends.push_back(b);
  CHECK(backends.size() == 2);
  const tensor::Backend saved = tensor::active_backend();
  Rng rng(77);
  Matrix<float> a(37, 29), b(29, 41), bias(37, 1);
  for (auto* m : {&a, &b, &bias})
    for (auto& v : m->storage()) v = float(rng.uniform(-1, 1));
  tensor::set_backend(tensor::Backend::scalar);
  const Matrix<float> want = tensor::gemm(a, b, &bias);
  const Matrix<float> sw = tensor::activate(a, tensor::ActivationSpec::sine(30.0));
  for (auto be : backends) {
    tensor::set_backend(be);
    CHECK(tensor::active_backend() == be);
    CHECK(std::string(tensor::kernels::active().name) == tensor::backend_name(be));
    const Matrix<float> got = tensor::gemm(a, b, &bias);
    const Matrix<float> s = tensor::activate(a, tensor::ActivationSpec::sine(30.0));
    double worst = 0, worst_s = 0;
    for (size_t i = 0; i < got.storage().size(); ++i)
      worst = std::max(worst, double(std::abs(got.storage()[i] - want.storage()[i])));
    for (size_t i = 0; i < s.storage().size(); ++i)
      worst_s = std::max(worst_s, double(std::abs(s.storage()[i] - sw.storage()[i])));
    CHECK(worst < 1e-5 && worst_s < 1e-5);  // the SIMD variants agree with scalar up to rounding
    const Matrix<float> ten{{10}, {10}};
    const Matrix<float> hand = tensor::gemm(Matrix<float>{{1, 2}, {3, 4}}, Matrix<float>{{1}, {1}}, &ten);
    CHECK(hand(0, 0) == 13.0f && hand(1, 0) == 17.0f);
  }
  // the avx2 table IS the device table's arithmetic
  tensor::set_backend(tensor::Backend::avx2);
  const Matrix<float> x = tensor::gemm(a, b, &bias);
  tensor::set_backend(tensor::Backend::b200);
  CHECK(x.storage() == tensor::gemm(a, b, &bias).storage());
  tensor::set_backend(saved);
}

template <typename T>
Matrix<T> rand_mat(int r, int c, Rng& rng) {
  Matrix<T> m(r, c);
  for (auto& v : m.storage()) v = T(rng.uniform(-1, 1));
  return m;
}

TEST_CASE("acceptance 1: f64 analytic gradients vs central differences (acceptance_main.cpp:30-71)") {
  const double h = 1e-4;
  const int points = 1000;
  double worst = 0;
  for (auto arch : {mlp::Architecture{16, 1, 3}, {64, 1, 3}, {256, 1, 3}, {256, 3, 3}}) {
    for (uint64_t seed = 1; seed <= 3; ++seed) {
      Rng rng(seed * 7919 + arch.width);
      auto net = mlp::random_init(arch, 30.0, rng);
      Matrix<double> pts = rand_mat<double>(3, points, rng);
      Matrix<double> grad = mlp::gradient_batch(net, pts);
      Matrix<double> fd(3, points);
      for (int c = 0; c < 3; ++c) {
        Matrix<double> hi = pts, lo = pts;
        for (int j = 0; j < points; ++j) {
          hi(c, j) += h;
          lo(c, j) -= h;
        }
        auto up = mlp::forward_batch(net, hi);
        auto dn = mlp::forward_batch(net, lo);
        for (int j = 0; j < points; ++j) fd(c, j) = (up(0, j) - dn(0, j)) / (2 * h);
      }
      for (int j = 0; j < points; ++j) {
        const double dx = grad(0, j) - fd(0, j), dy = grad(1, j) - fd(1, j), dz = grad(2, j) - fd(2, j);
        const double scale =
            std::max(std::sqrt(fd(0, j) * fd(0, j) + fd(1, j) * fd(1, j) + fd(2, j) * fd(2, j)), 1e-9);
        worst = std::max(worst, std::sqrt(dx * dx + dy * dy + dz * dz) / scale);
      }
    }
  }
  CHECK(worst < 1e-4);
}

TEST_CASE("acceptance 2: commutation identity behind the cheap gradient form (acceptance_main.cpp:74-98)") {
  Rng rng(1234);
  const tensor::ActivationSpec spec = tensor::ActivationSpec::sine(30.0);
  double worst = 0;
  for (int iter = 0; iter < 20; ++iter) {
    const int n = 2 + int(rng.next_u64() % 63);
    const int k = 1 + int(rng.next_u64() % 32);
    auto w = rand_mat<double>(n, n, rng);
    auto g = rand_mat<double>(n, k, rng);
    auto a = rand_mat<double>(n, 1, rng);
    Matrix<double> a_cols(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) a_cols(i, j) = a(i, 0);
    auto lhs = tensor::gemm(tensor::hadamard(w, tensor::activate(a_cols, spec, true)), g);
    auto rhs = tensor::scale_rows(tensor::activate(a, spec, true), tensor::gemm(w, g));
    double scale = 0;  // max-abs-scaled error (oracles.hpp:39-48)
    for (size_t i = 0; i < rhs.size(); ++i) scale = std::max(scale, std::fabs(rhs.data()[i]));
    if (scale == 0) scale = 1;
    for (size_t i = 0; i < lhs.size(); ++i) worst = std::max(worst, std::fabs(lhs.data()[i] - rhs.data()[i]) / scale);
  }
  CHECK(worst < 1e-10);
}

TEST_CASE("acceptance 3: threshold recurrences reproduce the hand tables (acceptance_main.cpp:100-121)") {
  auto near = [](double a, double b) { return std::fabs(a - b) <= 1e-15; };
  auto p2 = fields::thresholds_prop2({0.01, 0.02, 0.03});
  CHECK(near(p2[0], 0.13) && near(p2[1], 0.10) && near(p2[2], 0.05));
  auto p1 = fields::thresholds_prop1({0.02, 0.03});
  CHECK(near(p1[2], 0.03) && near(p1[1], 0.06) && near(p1[0], 0.08));
  auto p1e = fields::thresholds_prop1({0.01, 0.01, 0.01});
  for (size_t i = 0; i < p1e.size(); ++i) CHECK(near(p1e[i], 0.01 * double(4 - i)));
  auto p3 = fields::thresholds_prop3({0.05}, 0.01);
  CHECK(near(p3[1], 0.01) && near(p3[0], 0.08));
}

TEST_CASE("acceptance 4: exact concentric pair certifies, halved threshold violates (acceptance_main.cpp:123-150)") {
  NestedSequence seq = spheres({1.0, 0.95}, fields::thresholds_prop1({0.05}));
  fields::VerifyConfig cfg;
  cfg.samples = 200000;
  cfg.seed = 99;
  auto good = fields::verify_nesting(seq, cfg);
  auto again = fields::verify_nesting(seq, cfg);
  NestedSequence bad = seq;
  bad.deltas[0] *= 0.5;
  bad.deltas[1] = std::min(bad.deltas[1], bad.deltas[0] * 0.98);
  auto violated = fields::verify_nesting(bad, cfg);
  CHECK(good.violation_count == 0 && violated.violation_count >= 1);
  CHECK(good.checked == again.checked && good.violation_count == again.violation_count);
}

int main() { return chk::run_all(); }
