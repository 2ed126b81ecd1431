// Conversions between the drop-in C++ types and the C-ABI PODs.
#pragma once

#include <vector>

#include "engine.hpp"
#include "nsdf/shading/shading.hpp"

namespace nsdf::detail {

inline fields::DeviceBinding bind(const fields::Field& f) {
  fields::DeviceBinding b;
  if (!f.device_binding(b))
    throw Error(ErrorKind::config, "field " + f.describe() + " has no B200 device implementation");
  return b;
}

inline std::vector<nsdf_level> levels_of(const fields::NestedSequence& seq) {
  std::vector<nsdf_level> out;
  for (size_t i = 0; i < seq.size(); ++i) {
    const fields::DeviceBinding b = bind(seq.field(i));
    out.push_back({b.handle, b.time, seq.deltas[i]});
  }
  return out;
}

inline nsdf_camera to_pod(const tracer::Camera& c) {
  nsdf_camera p{};
  const Vec3* v[3] = {&c.position, &c.look_at, &c.up};
  double* d[3] = {p.position, p.look_at, p.up};
  for (int i = 0; i < 3; ++i) {
    d[i][0] = v[i]->x;
    d[i][1] = v[i]->y;
    d[i][2] = v[i]->z;
  }
  p.vertical_fov_deg = c.vertical_fov_deg;
  p.width = c.width;
  p.height = c.height;
  return p;
}

inline nsdf_trace_config to_pod(const tracer::TraceConfig& t) {
  nsdf_trace_config p{};
  p.n_levels = int(t.budgets.size());
  for (size_t i = 0; i < t.budgets.size() && i < size_t(NSDF_MAX_LEVELS); ++i) p.budgets[i] = t.budgets[i];
  p.eps_stop = t.eps_stop;
  p.t_max = t.t_max;
  return p;
}

inline nsdf_shade_config to_pod(const shading::ShadeConfig& s) {
  nsdf_shade_config p{};
  p.albedo[0] = s.material.albedo.x;
  p.albedo[1] = s.material.albedo.y;
  p.albedo[2] = s.material.albedo.z;
  p.ambient = s.material.ambient;
  p.diffuse = s.material.diffuse;
  p.specular = s.material.specular;
  p.shininess = s.material.shininess;
  if (s.lights.size() > size_t(NSDF_MAX_LIGHTS))
    throw Error(ErrorKind::config, "at most " + std::to_string(NSDF_MAX_LIGHTS) + " lights supported");
  p.n_lights = int(s.lights.size());
  for (size_t i = 0; i < s.lights.size(); ++i) {
    p.light_direction[i][0] = s.lights[i].direction.x;
    p.light_direction[i][1] = s.lights[i].direction.y;
    p.light_direction[i][2] = s.lights[i].direction.z;
    p.light_intensity[i] = s.lights[i].intensity;
  }
  p.background[0] = s.background.x;
  p.background[1] = s.background.y;
  p.background[2] = s.background.z;
  return p;
}

inline tracer::HitRecord from_pod(const nsdf_hit_record& r) {
  tracer::HitRecord h;
  h.hit = r.hit != 0;
  h.point = {r.point[0], r.point[1], r.point[2]};
  h.t = r.t;
  h.level_reached = r.level_reached;
  for (int i = 0; i < tracer::kMaxLevels; ++i) h.iterations_used[i] = r.iterations_used[i];
  h.final_distance = r.final_distance;
  return h;
}

}  // namespace nsdf::detail
