// nsdf::shading over the C ABI: neural normal mapping, shading and whole renders on the
// B200; image / mesh file I/O on the host.
#include <zlib.h>

#include <cstring>
#include <fstream>
#include <sstream>

#include <exception>
#include <thread>

#include "device_seq.hpp"
#include "nsdf/b200.hpp"
#include "engine.hpp"
#include "nsdf/shading/shading.hpp"

namespace nsdf::shading {

NormalMapResult neural_normal_map(const Field& fine, const Matrix<float>& points, double delta,
                                  const Matrix<float>* fallback_normals) {
  if (points.rows() != 3) throw Error(ErrorKind::contract, "points must be 3xk, got " + points.shape_str());
  if (fallback_normals && !fallback_normals->same_shape(points))
    throw Error(ErrorKind::contract, "fallback normals must match the point batch shape");
  const fields::DeviceBinding b = detail::bind(fine);
  NormalMapResult r;
  r.normals = Matrix<float>(3, points.cols());
  uint64_t outside = 0, fallbacks = 0;
  engine::check(nsdf_cuda_normal_map(engine::context(), b.handle, b.time, points.data(), points.cols(), delta,
                                     fallback_normals ? fallback_normals->data() : nullptr, r.normals.data(),
                                     &outside, &fallbacks));
  r.outside_count = size_t(outside);
  r.fallback_count = size_t(fallbacks);
  return r;
}

Matrix<float> shade(const Matrix<float>& points, const Matrix<float>& normals, const ShadeConfig& config,
                    const Camera& camera) {
  if (points.rows() != 3 || !points.same_shape(normals))
    throw Error(ErrorKind::contract, "points and normals must both be 3xk");
  if (config.lights.empty()) throw Error(ErrorKind::contract, "at least one directional light is required");
  const nsdf_shade_config sc = detail::to_pod(config);
  const nsdf_camera cam = detail::to_pod(camera);
  Matrix<float> rgb(3, points.cols());
  engine::check(nsdf_cuda_shade(engine::context(), points.data(), normals.data(), points.cols(), &sc, &cam, rgb.data()));
  return rgb;
}

ImageBuffer render(const NestedSequence& seq, const Camera& camera, const RenderConfig& config) {
  seq.validate();
  config.trace.validate(seq.size());
  camera.validate();
  const int fine = config.mapped_fine_index < 0 ? int(seq.size()) - 1 : config.mapped_fine_index;
  if (config.normal_source == NormalSource::mapped && fine >= int(seq.size()))
    throw Error(ErrorKind::config, "mapped-normal field index " + std::to_string(fine) + " is out of range");
  const auto levels = detail::levels_of(seq);
  const nsdf_camera cam = detail::to_pod(camera);
  const nsdf_trace_config tc = detail::to_pod(config.trace);
  const nsdf_shade_config sc = detail::to_pod(config.shade);
  const int src = config.normal_source == NormalSource::mapped ? NSDF_NORMALS_MAPPED : NSDF_NORMALS_OWN;
  const auto& ctxs = engine::contexts();
  if (ctxs.size() == 1) {
    // the frame renders while the ImageBuffer (35 MB at 1080p, value-initialised) is allocated
    engine::check(nsdf_cuda_render_begin(ctxs[0], levels.data(), int(levels.size()), &cam, &tc, &sc, src,
                                         config.mapped_fine_index));
    ImageBuffer img(camera.width, camera.height);
    engine::check(nsdf_cuda_render_end(ctxs[0], img.rgb.data(), img.depth.data(), img.mask.data(), nullptr));
    return img;
  }
  ImageBuffer img(camera.width, camera.height);
  // NSDF_DEVICES: the frame's tiles over every listed GPU (weights replicated once per field)
  std::vector<std::vector<nsdf_level>> per(ctxs.size(), levels);
  std::vector<const nsdf_level*> lp(ctxs.size());
  for (size_t i = 0; i < ctxs.size(); ++i) {
    for (nsdf_level& l : per[i]) l.field = engine::replica(i, l.field);
    lp[i] = per[i].data();
  }
  engine::check(nsdf_cuda_render_multi(ctxs.data(), int(ctxs.size()), lp.data(), int(levels.size()), &cam, &tc, &sc,
                                       src, config.mapped_fine_index, engine::tile_size(), img.rgb.data(),
                                       img.depth.data(), img.mask.data(), nullptr));
  return img;
}

}  // namespace nsdf::shading

namespace nsdf::b200 {

int context_count() { return int(engine::contexts().size()); }

std::vector<shading::ImageBuffer> render_frames(const fields::AnimatedSequence& anim, const std::vector<double>& times,
                                                const tracer::Camera& camera, const shading::RenderConfig& config) {
  anim.validate();
  camera.validate();
  const auto& ctxs = engine::contexts();
  const size_t n = ctxs.size();
  std::vector<shading::ImageBuffer> out(times.size());
  std::vector<std::exception_ptr> errors(n);
  const nsdf_camera cam = detail::to_pod(camera);
  const nsdf_trace_config tc = detail::to_pod(config.trace);
  const nsdf_shade_config sc = detail::to_pod(config.shade);
  const int src = config.normal_source == shading::NormalSource::mapped ? NSDF_NORMALS_MAPPED : NSDF_NORMALS_OWN;
  auto work = [&](size_t i) {
    try {
      for (size_t f = i; f < times.size(); f += n) {
        const fields::NestedSequence seq = anim.slice(times[f]);
        config.trace.validate(seq.size());
        auto levels = detail::levels_of(seq);
        for (nsdf_level& l : levels) l.field = engine::replica(i, l.field);
        engine::check(nsdf_cuda_render_begin(ctxs[i], levels.data(), int(levels.size()), &cam, &tc, &sc, src,
                                             config.mapped_fine_index));
        shading::ImageBuffer img(camera.width, camera.height);
        engine::check(nsdf_cuda_render_end(ctxs[i], img.rgb.data(), img.depth.data(), img.mask.data(), nullptr));
        out[f] = std::move(img);
      }
    } catch (...) {
      errors[i] = std::current_exception();
    }
  };
  std::vector<std::thread> threads;
  for (size_t i = 1; i < n; ++i) threads.emplace_back(work, i);
  work(0);
  for (auto& t : threads) t.join();
  for (const auto& e : errors)
    if (e) std::rethrow_exception(e);
  return out;
}

}  // namespace nsdf::b200

namespace nsdf::shading {

// Per-vertex normal mapping (reference mesh.cpp:122-156).  Fields with a device binding run
// entirely on the GPU (nsdf_cuda_map_normals_to_mesh: float cast, value + gradient tiles, the
// delta gate and the double normalisation in one device pass); other fields evaluate through
// their own eval_batch / grad_batch with the same gate on the host.
MeshMapReport map_normals_to_mesh(Mesh& mesh, const Field& fine, double delta) {
  if (mesh.vertices.empty()) throw Error(ErrorKind::contract, "mesh has no vertices");
  const int k = int(mesh.vertices.size());
  if (mesh.has_normals() && mesh.normals.size() != mesh.vertices.size())
    throw Error(ErrorKind::validation, "mesh has " + std::to_string(mesh.normals.size()) + " normals for " +
                                           std::to_string(mesh.vertices.size()) + " vertices");
  static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");
  fields::DeviceBinding b;
  if (fine.device_binding(b)) {
    std::vector<Vec3> updated = mesh.has_normals() ? mesh.normals : std::vector<Vec3>(mesh.vertices.size());
    uint64_t counts[3] = {0, 0, 0};
    engine::check(nsdf_cuda_map_normals_to_mesh(engine::context(), b.handle, b.time,
                                                reinterpret_cast<const double*>(mesh.vertices.data()), k, delta,
                                                reinterpret_cast<double*>(updated.data()), counts));
    MeshMapReport rep;
    rep.mapped = counts[0];
    rep.violators = counts[1];
    rep.fallbacks = counts[2];
    if (rep.mapped > 0) mesh.normals = std::move(updated);
    return rep;
  }
  Matrix<float> pts(3, k);
  for (int j = 0; j < k; ++j) {
    pts(0, j) = float(mesh.vertices[j].x);
    pts(1, j) = float(mesh.vertices[j].y);
    pts(2, j) = float(mesh.vertices[j].z);
  }
  const Matrix<float> vals = fine.eval_batch(pts);
  const Matrix<float> grads = fine.grad_batch(pts);
  MeshMapReport rep;
  std::vector<Vec3> updated = mesh.has_normals() ? mesh.normals : std::vector<Vec3>(mesh.vertices.size());
  for (int j = 0; j < k; ++j) {
    if (std::abs(double(vals(0, j))) > delta) {
      ++rep.violators;
      continue;
    }
    const Vec3 g{grads(0, j), grads(1, j), grads(2, j)};
    const double n = g.norm();
    if (n < 1e-8) {
      ++rep.fallbacks;
      continue;
    }
    updated[j] = g / n;
    ++rep.mapped;
  }
  if (rep.mapped > 0) mesh.normals = std::move(updated);
  return rep;
}

// ---- images ------------------------------------------------------------------------------------
double image_mse(const ImageBuffer& a, const ImageBuffer& b) {
  if (a.width != b.width || a.height != b.height)
    throw Error(ErrorKind::contract, "image sizes differ: " + std::to_string(a.width) + "x" +
                                         std::to_string(a.height) + " vs " + std::to_string(b.width) + "x" +
                                         std::to_string(b.height));
  if (a.rgb.empty()) return 0.0;
  double s = 0.0;
  for (size_t i = 0; i < a.rgb.size(); ++i) {
    const double d = double(a.rgb[i]) - double(b.rgb[i]);
    s += d * d;
  }
  return s / double(a.rgb.size());
}

namespace {
uint8_t to_byte(float v) {
  const float c = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
  return uint8_t(std::lround(c * 255.0f));
}
}  // namespace

void write_ppm(const ImageBuffer& img, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Error(ErrorKind::validation, "cannot write image " + path.string());
  out << "P6\n" << img.width << " " << img.height << "\n255\n";
  std::vector<uint8_t> px(img.rgb.size());
  for (size_t i = 0; i < px.size(); ++i) px[i] = to_byte(img.rgb[i]);
  out.write(reinterpret_cast<const char*>(px.data()), std::streamsize(px.size()));
}

ImageBuffer read_ppm(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Error(ErrorKind::parse, "cannot open image " + path.string());
  std::string magic;
  int w = 0, h = 0, maxv = 0;
  in >> magic >> w >> h >> maxv;
  if (magic != "P6" || w <= 0 || h <= 0 || maxv != 255)
    throw Error(ErrorKind::parse, path.string() + " is not an 8-bit binary PPM");
  in.get();
  ImageBuffer img(w, h);
  std::vector<uint8_t> px(img.rgb.size());
  in.read(reinterpret_cast<char*>(px.data()), std::streamsize(px.size()));
  if (!in) throw Error(ErrorKind::parse, path.string() + " is truncated");
  for (size_t i = 0; i < px.size(); ++i) img.rgb[i] = float(px[i]) / 255.0f;
  return img;
}

namespace {
void png_chunk(std::ofstream& out, const char* type, const std::vector<uint8_t>& data) {
  const uint32_t n = uint32_t(data.size());
  const uint8_t len[4] = {uint8_t(n >> 24), uint8_t(n >> 16), uint8_t(n >> 8), uint8_t(n)};
  out.write(reinterpret_cast<const char*>(len), 4);
  out.write(type, 4);
  if (n) out.write(reinterpret_cast<const char*>(data.data()), std::streamsize(n));
  uLong crc = crc32(0L, reinterpret_cast<const Bytef*>(type), 4);
  if (n) crc = crc32(crc, data.data(), n);
  const uint8_t c[4] = {uint8_t(crc >> 24), uint8_t(crc >> 16), uint8_t(crc >> 8), uint8_t(crc)};
  out.write(reinterpret_cast<const char*>(c), 4);
}
}  // namespace

void write_png(const ImageBuffer& img, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Error(ErrorKind::validation, "cannot write image " + path.string());
  static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
  out.write(reinterpret_cast<const char*>(sig), 8);
  std::vector<uint8_t> ihdr(13, 0);
  for (int i = 0; i < 4; ++i) {
    ihdr[i] = uint8_t(uint32_t(img.width) >> (24 - 8 * i));
    ihdr[4 + i] = uint8_t(uint32_t(img.height) >> (24 - 8 * i));
  }
  ihdr[8] = 8;  // bit depth
  ihdr[9] = 2;  // truecolor
  png_chunk(out, "IHDR", ihdr);
  std::vector<uint8_t> raw;
  raw.reserve(size_t(img.height) * (1 + size_t(img.width) * 3));
  for (int y = 0; y < img.height; ++y) {
    raw.push_back(0);  // filter: none
    for (int x = 0; x < img.width * 3; ++x) raw.push_back(to_byte(img.rgb[size_t(y) * img.width * 3 + x]));
  }
  uLongf zlen = compressBound(uLong(raw.size()));
  std::vector<uint8_t> z(zlen);
  if (compress2(z.data(), &zlen, raw.data(), uLong(raw.size()), 9) != Z_OK)
    throw Error(ErrorKind::validation, "zlib compression failed for " + path.string());
  z.resize(zlen);
  png_chunk(out, "IDAT", z);
  png_chunk(out, "IEND", {});
}

// ---- meshes (Wavefront OBJ v / vn / f) ---------------------------------------------------------
Mesh load_obj(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw Error(ErrorKind::parse, "cannot open mesh " + path.string());
  Mesh mesh;
  std::vector<Vec3> file_normals;
  std::vector<int> vn_of_vertex;
  std::string line;
  for (int line_no = 1; std::getline(in, line); ++line_no) {
    std::istringstream ss(line);
    std::string tag;
    ss >> tag;
    const std::string where = "line " + std::to_string(line_no) + ": ";
    if (tag == "v" || tag == "vn") {
      Vec3 v;
      if (!(ss >> v.x >> v.y >> v.z))
        throw Error(ErrorKind::parse, where + (tag == "v" ? "bad vertex record" : "bad normal record"));
      if (tag == "v") {
        mesh.vertices.push_back(v);
        vn_of_vertex.push_back(0);
      } else {
        file_normals.push_back(v);
      }
    } else if (tag == "f") {
      std::vector<int> corners;
      for (std::string tok; ss >> tok;) {
        int vi = 0, ni = 0;
        try {
          const auto s1 = tok.find('/');
          vi = std::stoi(tok.substr(0, s1));
          if (s1 != std::string::npos) {
            const auto s2 = tok.find('/', s1 + 1);
            if (s2 != std::string::npos && s2 + 1 < tok.size()) ni = std::stoi(tok.substr(s2 + 1));
          }
        } catch (const std::exception&) {
          throw Error(ErrorKind::parse, where + "bad face corner '" + tok + "'");
        }
        if (vi < 0) vi = int(mesh.vertices.size()) + 1 + vi;
        if (ni < 0) ni = int(file_normals.size()) + 1 + ni;
        if (vi < 1 || vi > int(mesh.vertices.size()))
          throw Error(ErrorKind::parse, where + "vertex index " + std::to_string(vi) + " out of range");
        if (ni != 0) {
          if (ni < 1 || ni > int(file_normals.size()))
            throw Error(ErrorKind::parse, where + "normal index " + std::to_string(ni) + " out of range");
          if (vn_of_vertex[vi - 1] == 0) vn_of_vertex[vi - 1] = ni;
        }
        corners.push_back(vi - 1);
      }
      if (corners.size() < 3) throw Error(ErrorKind::parse, where + "face needs at least 3 corners");
      for (size_t c = 1; c + 1 < corners.size(); ++c) mesh.triangles.push_back({corners[0], corners[c], corners[c + 1]});
    }
  }
  bool any = false;
  for (int n : vn_of_vertex) any = any || n != 0;
  if (any && !file_normals.empty()) {
    mesh.normals.assign(mesh.vertices.size(), Vec3{});
    for (size_t i = 0; i < mesh.vertices.size(); ++i)
      if (vn_of_vertex[i]) mesh.normals[i] = file_normals[size_t(vn_of_vertex[i] - 1)];
  }
  return mesh;
}

void save_obj(const Mesh& mesh, const std::filesystem::path& path) {
  std::ofstream out(path);
  if (!out) throw Error(ErrorKind::validation, "cannot write mesh " + path.string());
  if (mesh.has_normals() && mesh.normals.size() != mesh.vertices.size())
    throw Error(ErrorKind::validation, "mesh has " + std::to_string(mesh.normals.size()) + " normals for " +
                                           std::to_string(mesh.vertices.size()) + " vertices");
  out.precision(17);
  for (const auto& v : mesh.vertices) out << "v " << v.x << " " << v.y << " " << v.z << "\n";
  for (const auto& n : mesh.normals) out << "vn " << n.x << " " << n.y << " " << n.z << "\n";
  for (const auto& t : mesh.triangles) {
    out << "f";
    for (int c : t) {
      out << " " << c + 1;
      if (mesh.has_normals()) out << "//" << c + 1;
    }
    out << "\n";
  }
}

}  // namespace nsdf::shading
