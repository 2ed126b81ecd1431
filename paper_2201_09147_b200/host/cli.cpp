// The reference CLI's train / render / bench flows (proj/tools/nsdf_main.cpp) over the drop-in
// library, so a user of `nsdf train|render|bench` finds the same commands, flags, files and
// exit codes on the B200 build:
//   train   nsdf_main.cpp:141-258  fit_sequence(_4d) on the device, weights + reports +
//           manifest (+ .config echo) written next to each other
//   render  nsdf_main.cpp:260-340  one frame (or --time-steps frames of an animation)
//   bench   nsdf_main.cpp:344-502  rows of subsequences; CSV nets,iters,time_s,mem_kb,mse,
//           speedup with the MSE and speedup against the baseline row
// Exit codes as the reference: 0 ok, 1 usage/config, 2 validation or certification, 3
// divergence.  Entry point: nsdf_host_cli(argc, argv) (include/nsdf_host.h); tools/nsdf_b200
// is a main() around it.
#include <chrono>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <sstream>

#include "engine.hpp"
#include "nsdf/b200.hpp"
#include "nsdf/fields/nesting.hpp"
#include "nsdf/shading/shading.hpp"
#include "nsdf/trainer/trainer.hpp"
#include "nsdf_host.h"

namespace fs = std::filesystem;
using namespace nsdf;

namespace {

// --key value flags (repeatable keys keep every value, in order).
class Flags {
 public:
  Flags(int argc, const char* const* argv, int first) {
    for (int i = first; i < argc; ++i) {
      const std::string k = argv[i];
      if (k.rfind("--", 0) != 0 || i + 1 >= argc) throw Error(ErrorKind::config, "expected --flag value, got '" + k + "'");
      values_[k.substr(2)].push_back(argv[++i]);
    }
  }
  std::string str(const std::string& k, const std::string& def) {
    used_.push_back(k);
    auto it = values_.find(k);
    return it == values_.end() ? def : it->second.back();
  }
  std::vector<std::string> all(const std::string& k) {
    used_.push_back(k);
    auto it = values_.find(k);
    return it == values_.end() ? std::vector<std::string>{} : it->second;
  }
  double num(const std::string& k, double def) {
    const std::string v = str(k, "");
    if (v.empty()) return def;
    try {
      size_t n = 0;
      const double d = std::stod(v, &n);
      if (n != v.size()) throw std::invalid_argument(v);
      return d;
    } catch (const std::exception&) {
      throw Error(ErrorKind::config, "--" + k + " expects a number, got '" + v + "'");
    }
  }
  // unknown flags are usage errors, as CLI11 makes them in the reference
  void finish() const {
    for (const auto& [k, v] : values_)
      if (std::find(used_.begin(), used_.end(), k) == used_.end()) throw Error(ErrorKind::config, "unknown flag --" + k);
  }

 private:
  std::map<std::string, std::vector<std::string>> values_;
  std::vector<std::string> used_;
};

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  size_t start = 0;
  while (start <= s.size()) {
    const size_t end = std::min(s.find(sep, start), s.size());
    if (end > start) out.push_back(s.substr(start, end - start));
    start = end + 1;
  }
  return out;
}

std::vector<int> ints(const std::string& s) {
  std::vector<int> out;
  for (const auto& p : split(s, ',')) {
    try {
      out.push_back(std::stoi(p));
    } catch (const std::exception&) {
      throw Error(ErrorKind::config, "bad iteration budget '" + p + "'");
    }
  }
  return out;
}

std::string joined(const std::vector<int>& v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s;
}

Vec3 triple(const std::string& s) {
  const auto p = split(s, ',');
  try {
    if (p.size() == 3) return {std::stod(p[0]), std::stod(p[1]), std::stod(p[2])};
  } catch (const std::exception&) {
  }
  throw Error(ErrorKind::config, "expected x,y,z triple, got '" + s + "'");
}

// The reference's named shapes (nsdf_main.cpp resolve_shape); anything else is a field spec.
fields::AnalyticSpec shape_spec(const std::string& name) {
  static const std::map<std::string, std::string> named = {{"sphere", "sphere:r=0.7"},
                                                           {"sphere_unit", "sphere:r=1"},
                                                           {"torus", "torus:R=0.6,r=0.3"},
                                                           {"box", "box:hx=0.6,hy=0.45,hz=0.5"},
                                                           {"blend", "blend:r=0.7,R=0.6,rt=0.3"}};
  auto it = named.find(name);
  return fields::parse_field_spec(it == named.end() ? name : it->second);
}

using Echo = std::vector<std::pair<std::string, std::string>>;

// "# resolved configuration" block on stdout and in <file>.config
void echo(const std::string& command, const Echo& e, const fs::path& next_to) {
  std::ostringstream os;
  os << "# resolved configuration: " << command << "\n";
  for (const auto& [k, v] : e) os << k << " = " << v << "\n";
  std::cout << os.str();
  if (!next_to.empty()) std::ofstream(fs::path(next_to.string() + ".config")) << os.str();
}

struct CameraArgs {
  std::string pos, look, up;
  double fov;
  int width, height;
  explicit CameraArgs(Flags& f)
      : pos(f.str("cam-pos", "2,1.5,2")),
        look(f.str("look-at", "0,0,0")),
        up(f.str("up", "0,1,0")),
        fov(f.num("fov", 50.0)),
        width(int(f.num("width", 256))),
        height(int(f.num("height", 256))) {}
  tracer::Camera camera() const {
    tracer::Camera c;
    c.position = triple(pos);
    c.look_at = triple(look);
    c.up = triple(up);
    c.vertical_fov_deg = fov;
    c.width = width;
    c.height = height;
    return c;
  }
  void add_to(Echo& e) const {
    e.insert(e.end(), {{"cam-pos", pos}, {"look-at", look}, {"up", up}, {"fov", std::to_string(fov)},
                       {"width", std::to_string(width)}, {"height", std::to_string(height)}});
  }
};

void save_image(const shading::ImageBuffer& img, const fs::path& p) {
  if (p.extension() == ".png")
    shading::write_png(img, p);
  else
    shading::write_ppm(img, p);
}

// ---- train ----------------------------------------------------------------------------------
int cmd_train(Flags& f) {
  const std::string shape = f.str("shape", ""), archs_s = f.str("archs", "64x1"), out_dir_s = f.str("out-dir", ".");
  const std::string name_s = f.str("name", ""), epochs_list = f.str("epochs-list", "");
  const uint64_t seed = uint64_t(f.num("seed", 7));
  const int epochs = int(f.num("epochs", 800));
  const double lr = f.num("lr", 0.1), omega0 = f.num("omega0", 30.0), sigma = f.num("sigma", 0.01);
  const size_t n_uniform = size_t(f.num("uniform", 100000)), n_surface = size_t(f.num("surface", 100000));
  const size_t sup_u = size_t(f.num("sup-uniform", 500000)), sup_s = size_t(f.num("sup-surface", 500000));
  const size_t verify = size_t(f.num("verify-samples", 1000000));
  const double half = f.num("domain-half", 1.0);
  f.finish();
  if (shape.empty()) throw Error(ErrorKind::config, "--shape is required");
  const fields::AnalyticSpec spec = shape_spec(shape);
  const bool animated = spec.name == "blend";
  std::vector<mlp::Architecture> archs;
  for (const auto& a : split(archs_s, ',')) archs.push_back(mlp::parse_architecture(a, animated ? 4 : 3));
  if (archs.empty()) throw Error(ErrorKind::config, "--archs must list at least one WxK entry");
  const std::string name = name_s.empty() ? shape : name_s;
  const fs::path out_dir(out_dir_s);
  fs::create_directories(out_dir);
  const fs::path manifest = out_dir / (name + ".nest");

  trainer::SequenceFitConfig cfg;
  cfg.train.epochs = epochs;
  cfg.train.learning_rate = lr;
  cfg.train.omega0 = omega0;
  cfg.train.seed = seed;
  cfg.samples = {n_uniform, n_surface, sigma, 10000, seed};
  cfg.sup.n_uniform = sup_u;
  cfg.sup.n_surface = sup_s;
  cfg.sup.seed = seed + 1;
  cfg.verify.samples = verify;
  cfg.verify.seed = seed + 2;
  for (const auto& e : split(epochs_list, ',')) cfg.epochs_per_arch.push_back(std::stoi(e));

  Echo e{{"command", "train"},        {"shape", spec.text()},
         {"archs", archs_s},          {"seed", std::to_string(seed)},
         {"epochs", std::to_string(epochs)}, {"lr", std::to_string(lr)},
         {"omega0", std::to_string(omega0)}, {"uniform", std::to_string(n_uniform)},
         {"surface", std::to_string(n_surface)}, {"sigma", std::to_string(sigma)},
         {"sup-uniform", std::to_string(sup_u)}, {"sup-surface", std::to_string(sup_s)},
         {"verify-samples", std::to_string(verify)}, {"domain-half", std::to_string(half)},
         {"out-dir", out_dir_s},      {"name", name}};
  if (!epochs_list.empty()) e.push_back({"epochs-list", epochs_list});
  echo("train", e, manifest);

  auto write_member = [&](size_t i, const mlp::MlpParams<double>& p, const trainer::TrainReport& r) {
    const std::string stem = name + "_" + archs[i].name();
    mlp::save_params(p, out_dir / (stem + ".sdfnet"));
    r.write(out_dir / (stem + ".report.txt"));
    std::cout << archs[i].name() << ": " << r.summary() << "\n";
    return stem + ".sdfnet";
  };
  const Aabb domain = Aabb::cube(half);
  if (animated) {
    auto oracle = std::const_pointer_cast<fields::TimeVaryingField>(fields::make_analytic_time_field(spec));
    oracle->set_domain(domain);
    auto fit = trainer::fit_sequence_4d(archs, *oracle, cfg);
    for (size_t i = 0; i < archs.size(); ++i)
      fit.sequence.entries[i].source = {fields::FieldSource::Kind::weights, {}, write_member(i, fit.params[i], fit.reports[i])};
    fields::save_manifest(fit.sequence, manifest);
    std::cout << "certified per-slice with zero violations; manifest " << manifest << "\n";
    return 0;
  }
  auto oracle = std::const_pointer_cast<fields::Field>(fields::make_analytic_field(spec));
  oracle->set_domain(domain);
  auto fit = trainer::fit_sequence(archs, *oracle, cfg);
  for (size_t i = 0; i < archs.size(); ++i)
    fit.sequence.entries[i].source = {fields::FieldSource::Kind::weights, {}, write_member(i, fit.params[i], fit.reports[i])};
  fields::save_manifest(fit.sequence, manifest);
  std::cout << "eps:";
  for (double v : fit.eps) std::cout << " " << v;
  std::cout << "\ndeltas:";
  for (double v : fit.sequence.deltas) std::cout << " " << v;
  std::cout << "\ncertification: " << fit.certification.violation_count << " violations over "
            << fit.certification.checked << " checked samples\nmanifest " << manifest << "\n";
  return 0;
}

// ---- render ---------------------------------------------------------------------------------
shading::RenderConfig render_config(const std::string& budgets, size_t levels, const std::string& normals, int fine,
                                    double eps_stop, double t_max) {
  shading::RenderConfig c;
  c.trace.budgets = budgets.empty() ? std::vector<int>(levels, 40) : ints(budgets);
  c.trace.eps_stop = float(eps_stop);
  c.trace.t_max = float(t_max);
  if (normals != "own" && normals != "mapped") throw Error(ErrorKind::config, "--normals must be 'own' or 'mapped'");
  c.normal_source = normals == "mapped" ? shading::NormalSource::mapped : shading::NormalSource::own;
  c.mapped_fine_index = fine;
  return c;
}

int cmd_render(Flags& f) {
  const std::string path = f.str("manifest", ""), budgets = f.str("budgets", ""), normals = f.str("normals", "own");
  const int fine = int(f.num("fine", -1)), steps = int(f.num("time-steps", 0));
  const double eps_stop = f.num("eps-stop", 1e-3), t_max = f.num("t-max", 10.0), time = f.num("time", 0.0);
  const std::string out = f.str("out", "render.ppm");
  const CameraArgs cam(f);
  f.finish();
  if (path.empty()) throw Error(ErrorKind::config, "--manifest is required");
  const fields::SequenceManifest m = fields::load_manifest(path);
  const size_t levels = m.time_dependent ? m.animated.size() : m.sequence.size();
  const shading::RenderConfig cfg = render_config(budgets, levels, normals, fine, eps_stop, t_max);
  Echo e{{"command", "render"}, {"manifest", path},  {"budgets", joined(cfg.trace.budgets)},
         {"normals", normals},  {"fine", std::to_string(fine)}, {"eps-stop", std::to_string(eps_stop)},
         {"t-max", std::to_string(t_max)}, {"out", out}};
  if (m.time_dependent) e.insert(e.end(), {{"time-steps", std::to_string(steps)}, {"time", std::to_string(time)}});
  cam.add_to(e);
  echo("render", e, out);
  const tracer::Camera camera = cam.camera();
  if (m.time_dependent && steps > 0) {
    // the frame stream sharded across the engine's GPUs (NSDF_DEVICES): b200::render_frames
    const fs::path base(out);
    std::vector<double> times;
    for (int i = 0; i < steps; ++i) times.push_back(steps == 1 ? 0.0 : double(i) / double(steps - 1));
    const auto frames = b200::render_frames(m.animated, times, camera, cfg);
    for (int i = 0; i < steps; ++i) {
      std::ostringstream name;
      name << base.stem().string() << "_" << std::setw(3) << std::setfill('0') << i << base.extension().string();
      const fs::path frame = base.parent_path().empty() ? fs::path(name.str()) : base.parent_path() / name.str();
      save_image(frames[size_t(i)], frame);
      std::cout << "frame " << i << " (t=" << times[size_t(i)] << ") -> " << frame << "\n";
    }
    return 0;
  }
  const auto img = shading::render(m.time_dependent ? m.animated.slice(time) : m.sequence, camera, cfg);
  save_image(img, out);
  size_t hits = 0;
  for (uint8_t v : img.mask) hits += v;
  std::cout << "wrote " << out << " (" << hits << " hit pixels of " << img.pixel_count() << ")\n";
  return 0;
}

// ---- bench ----------------------------------------------------------------------------------
struct Row {
  std::vector<std::string> nets;
  std::vector<int> iters;
  std::string normals = "own";
  bool baseline = false;
};

Row parse_row(const std::string& text) {
  Row r;
  for (const auto& part : split(text, ';')) {
    const size_t eq = part.find('=');
    const std::string key = part.substr(0, eq), val = eq == std::string::npos ? "" : part.substr(eq + 1);
    if (key == "nets")
      r.nets = split(val, ',');
    else if (key == "iters")
      r.iters = ints(val);
    else if (key == "normals")
      r.normals = val;
    else if (key == "baseline")
      r.baseline = true;
    else
      throw Error(ErrorKind::config, "unknown bench row key '" + key + "' in '" + text + "'");
  }
  if (r.nets.empty() || r.iters.size() != r.nets.size())
    throw Error(ErrorKind::config, "bench row needs matching nets and iters lists: '" + text + "'");
  return r;
}

int cmd_bench(Flags& f) {
  const std::string path = f.str("manifest", ""), out = f.str("out", "bench.csv");
  const std::vector<std::string> row_texts = f.all("row");
  const int repeats = int(f.num("repeats", 1));
  const double eps_stop = f.num("eps-stop", 1e-3);
  const CameraArgs cam(f);
  f.finish();
  if (path.empty()) throw Error(ErrorKind::config, "--manifest is required");
  if (row_texts.empty()) throw Error(ErrorKind::config, "at least one --row is required");
  const fields::SequenceManifest m = fields::load_manifest(path);
  if (m.time_dependent) throw Error(ErrorKind::config, "bench expects a static manifest");
  const fields::NestedSequence& full = m.sequence;
  // a bare number selects by position, anything else matches a label
  auto index_of = [&](const std::string& label) -> size_t {
    if (!label.empty() && label.find_first_not_of("0123456789") == std::string::npos) {
      const size_t i = std::stoul(label);
      if (i >= full.size()) throw Error(ErrorKind::config, "field index " + label + " is out of range");
      return i;
    }
    for (size_t i = 0; i < full.size(); ++i)
      if (full.entries[i].label == label) return i;
    throw Error(ErrorKind::config, "manifest has no field labelled '" + label + "'");
  };
  std::vector<Row> rows;
  int base = -1;
  for (const auto& t : row_texts) {
    rows.push_back(parse_row(t));
    if (!rows.back().baseline) continue;
    if (base >= 0) throw Error(ErrorKind::config, "only one baseline row is allowed");
    base = int(rows.size()) - 1;
  }
  if (base < 0) throw Error(ErrorKind::config, "no baseline row configured (add ';baseline' to one row)");
  Echo e{{"command", "bench"}, {"manifest", path}, {"repeats", std::to_string(repeats)},
         {"eps-stop", std::to_string(eps_stop)}, {"out", out}};
  for (const auto& t : row_texts) e.push_back({"row", t});
  cam.add_to(e);
  echo("bench", e, out);
  const tracer::Camera camera = cam.camera();

  struct Result {
    std::string nets, iters;
    double seconds = 0;
    size_t mem_kb = 0;
    shading::ImageBuffer image;
  };
  std::vector<Result> res;
  for (const Row& r : rows) {
    // the traced subsequence; mapped normals come from the manifest's finest field, appended
    // with a zero budget when the row does not end with it
    fields::NestedSequence seq;
    std::vector<int> budgets = r.iters;
    for (const auto& label : r.nets) {
      const size_t i = index_of(label);
      seq.entries.push_back(full.entries[i]);
      seq.deltas.push_back(full.deltas[i]);
    }
    shading::RenderConfig cfg;
    cfg.shade.material.specular = 0.3f;
    cfg.trace.eps_stop = float(eps_stop);
    if (r.normals == "mapped") {
      cfg.normal_source = shading::NormalSource::mapped;
      const size_t finest = full.size() - 1;
      if (index_of(r.nets.back()) != finest) {
        seq.entries.push_back(full.entries[finest]);
        seq.deltas.push_back(full.deltas[finest]);
        budgets.push_back(0);
      }
      cfg.mapped_fine_index = int(seq.size()) - 1;
    } else if (r.normals != "own") {
      throw Error(ErrorKind::config, "row normals must be 'own' or 'mapped'");
    }
    cfg.trace.budgets = budgets;
    Result x;
    for (const auto& en : seq.entries) x.mem_kb += (en.param_count * 4 + 1023) / 1024;  // f32, ceil per net
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < repeats; ++k) x.image = shading::render(seq, camera, cfg);
    x.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / repeats;
    for (size_t i = 0; i < r.nets.size(); ++i) x.nets += (i ? ">" : "") + r.nets[i];
    if (r.normals == "mapped") x.nets += "+map";
    x.iters = joined(r.iters);
    res.push_back(std::move(x));
  }
  std::ofstream csv(out);
  if (!csv) throw Error(ErrorKind::validation, "cannot write " + out);
  csv << "nets,iters,time_s,mem_kb,mse,speedup\n";
  csv.precision(6);
  for (size_t i = 0; i < res.size(); ++i) {
    const Result& x = res[i];
    csv << "\"" << x.nets << "\",\"" << x.iters << "\"," << x.seconds << "," << x.mem_kb << ",";
    if (int(i) != base) csv << shading::image_mse(x.image, res[size_t(base)].image);
    csv << "," << (x.seconds > 0 ? res[size_t(base)].seconds / x.seconds : 0.0) << "\n";
  }
  std::cout << "wrote " << out << "\n";
  return 0;
}

int exit_code(const Error& e) {
  return e.kind() == ErrorKind::config ? 1 : e.kind() == ErrorKind::divergence ? 3 : 2;
}

}  // namespace

extern "C" int nsdf_host_cli(int argc, const char* const* argv) {
  if (argc < 2) {
    std::cerr << "usage: nsdf_b200 train|render|bench --flag value ...\n";
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    Flags f(argc, argv, 2);
    if (cmd == "train") return cmd_train(f);
    if (cmd == "render") return cmd_render(f);
    if (cmd == "bench") return cmd_bench(f);
    std::cerr << "error: unknown command '" << cmd << "' (train, render, bench)\n";
    return 1;
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return exit_code(e);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
