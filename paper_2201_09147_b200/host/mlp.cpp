// nsdf::mlp over the C ABI: parameter validation and init on the host, float batch
// evaluation on the B200 (nsdf_cuda_eval_grad), .sdfnet JSON I/O (reference io.cpp schema).
#include <cstring>
#include <fstream>
#include <list>
#include <mutex>

#include <json.hpp>

#include "engine.hpp"
#include "nsdf/mlp/mlp.hpp"

namespace nsdf {

namespace tensor {

ActivationSpec parse_activation(const std::string& name, double omega0) {
  if (name == "sine") return ActivationSpec::sine(omega0);
  if (name == "identity") return ActivationSpec::identity();
  throw Error(ErrorKind::config, "unknown activation kind '" + name + "' (expected sine or identity)");
}

std::string activation_name(const ActivationSpec& spec) {
  return spec.kind == Activation::sine ? "sine" : "identity";
}

}  // namespace tensor

namespace mlp {

template <typename T>
void MlpParams<T>::validate() const {
  if (layers.empty()) throw Error(ErrorKind::validation, "network has no layers");
  if (input_dim != 3 && input_dim != 4)
    throw Error(ErrorKind::validation, "input_dim must be 3 or 4, got " + std::to_string(input_dim));
  if (layers.front().weights.cols() != input_dim)
    throw Error(ErrorKind::validation, "layer 0 expects input dim " + std::to_string(layers.front().weights.cols()) +
                                           " but network input_dim is " + std::to_string(input_dim));
  for (size_t i = 0; i < layers.size(); ++i) {
    const auto& l = layers[i];
    if (l.bias.cols() != 1 || l.bias.rows() != l.weights.rows())
      throw Error(ErrorKind::validation, "layer " + std::to_string(i) + " bias is " + l.bias.shape_str() +
                                             ", weights are " + l.weights.shape_str());
    if (i + 1 < layers.size() && layers[i + 1].weights.cols() != l.weights.rows())
      throw Error(ErrorKind::validation, "dimension chain broken between layers " + std::to_string(i) + "," +
                                             std::to_string(i + 1) + ": " + l.weights.shape_str() + " feeds " +
                                             layers[i + 1].weights.shape_str());
  }
  if (layers.back().weights.rows() != 1)
    throw Error(ErrorKind::validation,
                "output layer must have a single output, got " + std::to_string(layers.back().weights.rows()));
}

template void MlpParams<float>::validate() const;
template void MlpParams<double>::validate() const;

Architecture parse_architecture(const std::string& spec, int input_dim) {
  const auto x = spec.find('x');
  const auto bad = [&] {
    return Error(ErrorKind::config, "architecture '" + spec + "' does not match the WxK grammar (e.g. 64x1)");
  };
  if (x == std::string::npos || x == 0 || x + 1 >= spec.size()) throw bad();
  Architecture a;
  try {
    a.width = std::stoi(spec.substr(0, x));
    a.hidden_blocks = std::stoi(spec.substr(x + 1));
  } catch (const std::exception&) {
    throw bad();
  }
  a.input_dim = input_dim;
  if (a.width < 1 || a.hidden_blocks < 0)
    throw Error(ErrorKind::config, "architecture '" + spec + "' has non-positive dimensions");
  return a;
}

// SIREN initialisation (reference mlp.cpp:63-88): first layer U(+-1/fan_in), deeper layers
// U(+-sqrt(6/fan_in)/omega0), biases U(+-1/sqrt(fan_in)); weights then biases per layer.
MlpParams<double> random_init(const Architecture& arch, double omega0, Rng& rng) {
  MlpParams<double> p;
  p.input_dim = arch.input_dim;
  p.activation = ActivationSpec::sine(omega0);
  std::vector<std::pair<int, int>> shapes{{arch.width, arch.input_dim}};
  for (int i = 0; i < arch.hidden_blocks; ++i) shapes.push_back({arch.width, arch.width});
  shapes.push_back({1, arch.width});
  for (size_t li = 0; li < shapes.size(); ++li) {
    const auto [out, in] = shapes[li];
    const double wb = li == 0 ? 1.0 / in : std::sqrt(6.0 / in) / omega0;
    const double bb = 1.0 / std::sqrt(double(in));
    LayerParams<double> l{Matrix<double>(out, in), Matrix<double>(out, 1)};
    for (auto& w : l.weights.storage()) w = rng.uniform(-wb, wb);
    for (auto& b : l.bias.storage()) b = rng.uniform(-bb, bb);
    p.layers.push_back(std::move(l));
  }
  p.validate();
  return p;
}

namespace {

// Device copies of parameter sets used through the free functions, keyed by content.
struct UploadCache {
  std::mutex mu;
  std::list<std::pair<uint64_t, int>> entries;  // most recent first
};
UploadCache& cache() {
  static UploadCache c;
  return c;
}

template <typename T>
uint64_t content_hash(const MlpParams<T>& p) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* d, size_t n) {
    const auto* b = static_cast<const unsigned char*>(d);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  mix(&p.input_dim, sizeof(int));
  mix(&p.activation.kind, sizeof(p.activation.kind));
  mix(&p.activation.omega0, sizeof(double));
  for (const auto& l : p.layers) {
    const int r = l.weights.rows(), c = l.weights.cols();
    mix(&r, sizeof r);
    mix(&c, sizeof c);
    mix(l.weights.data(), l.weights.size() * sizeof(T));
    mix(l.bias.data(), l.bias.size() * sizeof(T));
  }
  return h;
}

}  // namespace

// Uploads (or finds) the device copy of a parameter set; shared with fields.cpp.
template <typename T>
int device_handle(const MlpParams<T>& p) {
  p.validate();
  const uint64_t key = content_hash(p);
  auto& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  for (auto it = c.entries.begin(); it != c.entries.end(); ++it)
    if (it->first == key) {
      c.entries.splice(c.entries.begin(), c.entries, it);
      return it->second;
    }
  std::vector<int32_t> rows, cols;
  std::vector<double> packed;
  for (const auto& l : p.layers) {
    rows.push_back(l.weights.rows());
    cols.push_back(l.weights.cols());
    for (T v : l.weights.storage()) packed.push_back(double(v));
    for (T v : l.bias.storage()) packed.push_back(double(v));
  }
  int h = 0;
  engine::check(nsdf_cuda_upload_mlp(engine::context(), int(rows.size()), rows.data(), cols.data(), packed.data(),
                                     p.activation.kind == tensor::Activation::sine ? NSDF_ACT_SINE : NSDF_ACT_IDENTITY,
                                     p.activation.omega0, p.input_dim, &h));
  c.entries.emplace_front(key, h);
  if (c.entries.size() > 16) {
    nsdf_cuda_release(engine::context(), c.entries.back().second);
    c.entries.pop_back();
  }
  return h;
}
template int device_handle(const MlpParams<float>&);
template int device_handle(const MlpParams<double>&);

namespace {

void check_points(int input_dim, const Matrix<float>& pts, int rows) {
  if (pts.rows() != rows)
    throw Error(ErrorKind::contract,
                "point batch is " + pts.shape_str() + " but " + std::to_string(rows) + " rows are required");
  (void)input_dim;
}

void eval_device(const MlpParams<float>& p, const Matrix<float>& pts, Matrix<float>* dist, Matrix<float>* grad) {
  const int h = device_handle(p);
  const int k = pts.cols();
  if (dist) *dist = Matrix<float>(1, k);
  if (grad) *grad = Matrix<float>(3, k);
  engine::check(nsdf_cuda_eval_grad(engine::context(), h, pts.data(), pts.rows(), k, 0.0f,
                                    dist ? dist->data() : nullptr, grad ? grad->data() : nullptr));
}

}  // namespace

template <>
Matrix<float> forward_batch(const MlpParams<float>& p, const Matrix<float>& points) {
  if (p.layers.empty()) throw Error(ErrorKind::contract, "network has no layers");
  check_points(p.input_dim, points, p.input_dim);
  Matrix<float> d;
  eval_device(p, points, &d, nullptr);
  return d;
}

template <>
Matrix<float> gradient_batch(const MlpParams<float>& p, const Matrix<float>& points) {
  if (p.input_dim != 3)
    throw Error(ErrorKind::contract,
                "gradient_batch expects a 3-input network; use spatial_gradient_batch for time-extended networks");
  check_points(3, points, 3);
  Matrix<float> g;
  eval_device(p, points, nullptr, &g);
  return g;
}

template <>
Matrix<float> spatial_gradient_batch(const MlpParams<float>& p, const Matrix<float>& points) {
  if (p.input_dim != 4) throw Error(ErrorKind::contract, "spatial_gradient_batch expects a 4-input network");
  check_points(4, points, 4);
  Matrix<float> g;
  eval_device(p, points, nullptr, &g);
  return g;
}

template <>
std::pair<Matrix<float>, Matrix<float>> forward_and_gradient_batch(const MlpParams<float>& p,
                                                                    const Matrix<float>& points) {
  if (p.input_dim != 3) throw Error(ErrorKind::contract, "forward_and_gradient_batch expects a 3-input network");
  check_points(3, points, 3);
  Matrix<float> d, g;
  eval_device(p, points, &d, &g);
  return {std::move(d), std::move(g)};
}

// f64 evaluation (certification: nesting.cpp:131-361) runs on the device FP64 path
// (mlp_f64.cu), bit-exact with the reference's double AVX2 kernels.
namespace {

void check_points_d(const Matrix<double>& pts, int rows) {
  if (pts.rows() != rows)
    throw Error(ErrorKind::contract,
                "point batch is " + pts.shape_str() + " but " + std::to_string(rows) + " rows are required");
}

void eval_device_d(const MlpParams<double>& p, const Matrix<double>& pts, Matrix<double>* dist, Matrix<double>* grad) {
  const int h = device_handle(p);
  const int k = pts.cols();
  if (dist) *dist = Matrix<double>(1, k);
  if (grad) *grad = Matrix<double>(3, k);
  engine::check(nsdf_cuda_eval_f64(engine::context(), h, pts.data(), pts.rows(), k, 0.0,
                                   dist ? dist->data() : nullptr, grad ? grad->data() : nullptr));
}

}  // namespace

template <>
Matrix<double> forward_batch(const MlpParams<double>& p, const Matrix<double>& points) {
  if (p.layers.empty()) throw Error(ErrorKind::contract, "network has no layers");
  check_points_d(points, p.input_dim);
  Matrix<double> d;
  eval_device_d(p, points, &d, nullptr);
  return d;
}
template <>
Matrix<double> gradient_batch(const MlpParams<double>& p, const Matrix<double>& points) {
  if (p.input_dim != 3)
    throw Error(ErrorKind::contract,
                "gradient_batch expects a 3-input network; use spatial_gradient_batch for time-extended networks");
  check_points_d(points, 3);
  Matrix<double> g;
  eval_device_d(p, points, nullptr, &g);
  return g;
}
template <>
Matrix<double> spatial_gradient_batch(const MlpParams<double>& p, const Matrix<double>& points) {
  if (p.input_dim != 4) throw Error(ErrorKind::contract, "spatial_gradient_batch expects a 4-input network");
  check_points_d(points, 4);
  Matrix<double> g;
  eval_device_d(p, points, nullptr, &g);
  return g;
}
template <>
std::pair<Matrix<double>, Matrix<double>> forward_and_gradient_batch(const MlpParams<double>& p,
                                                                      const Matrix<double>& points) {
  if (p.input_dim != 3) throw Error(ErrorKind::contract, "forward_and_gradient_batch expects a 3-input network");
  check_points_d(points, 3);
  Matrix<double> d, g;
  eval_device_d(p, points, &d, &g);
  return {std::move(d), std::move(g)};
}

// ---- .sdfnet: {activation, omega0, input_dim, layers[{rows, cols, weights_flat, bias}]} ----
using nlohmann::json;

void save_params(const MlpParams<double>& params, const std::filesystem::path& destination) {
  params.validate();
  json layers = json::array();
  for (const auto& l : params.layers)
    layers.push_back({{"rows", l.weights.rows()},
                      {"cols", l.weights.cols()},
                      {"weights_flat", l.weights.storage()},
                      {"bias", l.bias.storage()}});
  json j{{"activation", tensor::activation_name(params.activation)},
         {"omega0", params.activation.omega0},
         {"input_dim", params.input_dim},
         {"layers", std::move(layers)}};
  std::ofstream out(destination);
  if (!out) throw Error(ErrorKind::validation, "cannot write weight file " + destination.string());
  out << j.dump(1) << "\n";
}

MlpParams<double> load_params(const std::filesystem::path& source) {
  std::ifstream in(source);
  if (!in) throw Error(ErrorKind::parse, "cannot open weight file " + source.string());
  json j;
  try {
    in >> j;
  } catch (const json::parse_error& e) {
    throw Error(ErrorKind::parse, "malformed weight file " + source.string() + ": " + e.what());
  }
  MlpParams<double> p;
  try {
    p.activation = tensor::parse_activation(j.at("activation").get<std::string>(), j.at("omega0").get<double>());
    p.input_dim = j.at("input_dim").get<int>();
    const json& layers = j.at("layers");
    for (size_t i = 0; i < layers.size(); ++i) {
      const int r = layers[i].at("rows").get<int>(), c = layers[i].at("cols").get<int>();
      auto w = layers[i].at("weights_flat").get<std::vector<double>>();
      auto b = layers[i].at("bias").get<std::vector<double>>();
      if (w.size() != size_t(r) * size_t(c) || b.size() != size_t(r))
        throw Error(ErrorKind::parse, "layer " + std::to_string(i) + " of " + source.string() +
                                          " has inconsistent weight or bias length");
      p.layers.push_back({Matrix<double>(r, c, std::move(w)), Matrix<double>(r, 1, std::move(b))});
    }
  } catch (const json::exception& e) {
    throw Error(ErrorKind::parse, "weight file " + source.string() + " is malformed: " + e.what());
  }
  p.validate();
  return p;
}

}  // namespace mlp
}  // namespace nsdf
