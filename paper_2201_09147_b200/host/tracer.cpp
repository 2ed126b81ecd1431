// nsdf::tracer over the C ABI: rays, multiscale sphere tracing and whole-image traces all
// run on the B200 (nsdf_cuda_generate_rays / _trace_rays / _sphere_trace / _trace_image).
#include "device_seq.hpp"
#include "engine.hpp"
#include "nsdf/tracer/trace.hpp"

namespace nsdf::tracer {

void Camera::validate() const {
  if (width <= 0 || height <= 0)
    throw Error(ErrorKind::config,
                "image size must be positive, got " + std::to_string(width) + "x" + std::to_string(height));
  if (!(vertical_fov_deg > 0) || !(vertical_fov_deg < 180))
    throw Error(ErrorKind::config, "vertical fov must be in (0,180) degrees");
  const Vec3 fwd = (look_at - position).normalized();
  if (fwd.norm() == 0) throw Error(ErrorKind::config, "camera position and look_at coincide");
  if (fwd.cross(up).norm() < 1e-9) throw Error(ErrorKind::config, "up vector is parallel to the view direction");
}

void TraceConfig::validate(size_t n) const {
  if (budgets.size() != n)
    throw Error(ErrorKind::config,
                "got " + std::to_string(budgets.size()) + " budgets for " + std::to_string(n) + " levels");
  if (n > size_t(kMaxLevels)) throw Error(ErrorKind::config, "at most " + std::to_string(kMaxLevels) + " levels supported");
  bool any = false;
  for (int b : budgets) {
    if (b < 0) throw Error(ErrorKind::config, "iteration budgets must be non-negative");
    any = any || b > 0;
  }
  if (!any) throw Error(ErrorKind::config, "all iteration budgets are zero");
  if (!(eps_stop > 0)) throw Error(ErrorKind::config, "eps_stop must be positive");
}

std::vector<Ray> generate_rays(const Camera& camera) {
  camera.validate();
  const nsdf_camera cam = detail::to_pod(camera);
  const size_t n = size_t(camera.width) * camera.height;
  std::vector<float> buf(6 * n);
  engine::check(nsdf_cuda_generate_rays(engine::context(), &cam, buf.data()));
  std::vector<Ray> rays(n);
  for (size_t i = 0; i < n; ++i)
    rays[i] = {{buf[6 * i], buf[6 * i + 1], buf[6 * i + 2]}, {buf[6 * i + 3], buf[6 * i + 4], buf[6 * i + 5]}};
  return rays;
}

HitRecord sphere_trace(const Field& field, const Ray& ray, float delta, float eps_stop, int max_iters, float t_max) {
  if (!(eps_stop > 0)) throw Error(ErrorKind::config, "eps_stop must be positive");
  if (delta < 0) throw Error(ErrorKind::config, "offset must be non-negative");
  const fields::DeviceBinding b = detail::bind(field);
  const float r[6] = {ray.origin.x, ray.origin.y, ray.origin.z, ray.direction.x, ray.direction.y, ray.direction.z};
  nsdf_hit_record rec;
  engine::check(nsdf_cuda_sphere_trace(engine::context(), b.handle, b.time, delta, eps_stop, max_iters, t_max, r, 1,
                                       &rec));
  return detail::from_pod(rec);
}

HitRecord multiscale_sphere_trace(const NestedSequence& seq, const Ray& ray, const TraceConfig& config) {
  seq.validate();
  config.validate(seq.size());
  const auto levels = detail::levels_of(seq);
  const nsdf_trace_config cfg = detail::to_pod(config);
  const float r[6] = {ray.origin.x, ray.origin.y, ray.origin.z, ray.direction.x, ray.direction.y, ray.direction.z};
  nsdf_hit_record rec;
  engine::check(nsdf_cuda_trace_rays(engine::context(), levels.data(), int(levels.size()), &cfg, r, 1, &rec));
  return detail::from_pod(rec);
}

std::vector<HitRecord> trace_image(const NestedSequence& seq, const Camera& camera, const TraceConfig& config) {
  seq.validate();
  config.validate(seq.size());
  camera.validate();
  const auto levels = detail::levels_of(seq);
  const nsdf_trace_config cfg = detail::to_pod(config);
  const nsdf_camera cam = detail::to_pod(camera);
  std::vector<nsdf_hit_record> recs(size_t(camera.width) * camera.height);
  engine::check(nsdf_cuda_trace_image(engine::context(), levels.data(), int(levels.size()), &cam, &cfg, recs.data(),
                                      nullptr));
  std::vector<HitRecord> out(recs.size());
  for (size_t i = 0; i < recs.size(); ++i) out[i] = detail::from_pod(recs[i]);
  return out;
}

}  // namespace nsdf::tracer
