// Device operations shared by the FFMA (engine.cu) and tensor-core (mlp_tc.cu) kernels:
// the per-ray trace update, normal normalization and shading.  Every float operation is
// an explicit _rn intrinsic, so the arithmetic is the reference's -ffp-contract=off C++
// regardless of the translation unit's -fmad setting.
#pragma once

#include "engine.cuh"

namespace nsdf_b200 {

// ---------------------------------------------------------------------------------------
// Trace iteration (trace_level body, trace.cpp:46-82) for one compacted active list.
// ---------------------------------------------------------------------------------------
struct IterArgs {
  LevelDesc lv;
  float eps;
  float t_max;
  int iter;
  const int* in_list;
  const int* in_count;
  int* next_list;
  int* next_count;
  int* adv_list;
  int* adv_count;
  RayState st;
};

__device__ __forceinline__ void trace_update(const IterArgs& a, int slot, float f, bool& conv, bool& cont) {
  const RayState& st = a.st;
  const float fd = __fsub_rn(f, a.lv.delta);
  const float afd = fabsf(fd);
  conv = a.lv.final_level ? afd <= a.eps : fd <= a.eps;
  cont = false;
  if (a.iter == 0) st.level_reached[slot] = a.lv.level;
  if (!conv) {
    float step = fd;
    if (a.lv.final_level && step < 0.0f) step = 0.0f;  // trace.cpp:73
    st.px[slot] = __fadd_rn(st.px[slot], __fmul_rn(step, st.dx[slot]));
    st.py[slot] = __fadd_rn(st.py[slot], __fmul_rn(step, st.dy[slot]));
    st.pz[slot] = __fadd_rn(st.pz[slot], __fmul_rn(step, st.dz[slot]));
    const float t = __fadd_rn(st.t[slot], step);
    st.t[slot] = t;
    cont = !(t > a.t_max);  // trace.cpp:78
  }
  // Every ray in iteration `iter`'s list has made exactly iter evaluations at this level,
  // so the per-level counter is written once, when the ray leaves the level.
  if (!cont || a.iter == a.lv.budget - 1) {
    st.iters[size_t(slot) * kMaxLevels + a.lv.level] = uint16_t(a.iter + 1);
    st.final_dist[slot] = afd;
  }
}


// ---------------------------------------------------------------------------------------
// Shading (shade.cpp:44-93).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ float dot3_rn(float ax, float ay, float az, float bx, float by, float bz) {
  return __fadd_rn(__fadd_rn(__fmul_rn(ax, bx), __fmul_rn(ay, by)), __fmul_rn(az, bz));
}

__device__ __forceinline__ float clamp01(float v) { return v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v); }

__device__ __forceinline__ void shade_point(const ShadeParams& sp, float px, float py, float pz, float nx, float ny, float nz,
                            float rgb[3]) {
  float lit = sp.ambient;
  float spec = 0.0f;
  for (int i = 0; i < sp.n_lights; ++i) {
    const float lx = sp.light[i][0], ly = sp.light[i][1], lz = sp.light[i][2], li = sp.light[i][3];
    const float ndotl = dot3_rn(nx, ny, nz, lx, ly, lz);
    if (ndotl > 0) lit = __fadd_rn(lit, __fmul_rn(__fmul_rn(sp.diffuse, li), ndotl));
    if (sp.specular > 0 && ndotl > 0) {
      const float vx = __fsub_rn(sp.cam[0], px), vy = __fsub_rn(sp.cam[1], py), vz = __fsub_rn(sp.cam[2], pz);
      const float vn = __fsqrt_rn(dot3_rn(vx, vy, vz, vx, vy, vz));
      if (vn > 0) {
        const float hx = __fadd_rn(lx, __fdiv_rn(vx, vn)), hy = __fadd_rn(ly, __fdiv_rn(vy, vn)),
                    hz = __fadd_rn(lz, __fdiv_rn(vz, vn));
        const float hn = __fsqrt_rn(dot3_rn(hx, hy, hz, hx, hy, hz));
        if (hn > 0) {
          const float ndoth = __fdiv_rn(dot3_rn(nx, ny, nz, hx, hy, hz), hn);
          if (ndoth > 0) {
            // std::pow(float, float) (libm powf): CUDA's powf is within 2 ulp of it — with
            // specular * intensity <= 1 that is <= 2.4e-7 of the colour, inside the 1e-6 the
            // shading is compared at (it is not bitwise: libm's transcendentals are not
            // restated); NSDF_SHADE_POW_F64=1 evaluates in double and rounds once instead
#if NSDF_SHADE_POW_F64
            const float pw = __double2float_rn(pow(double(ndoth), double(sp.shininess)));
#else
            const float pw = powf(ndoth, sp.shininess);
#endif
            spec = __fadd_rn(spec, __fmul_rn(__fmul_rn(sp.specular, li), pw));
          }
        }
      }
    }
  }
  for (int c = 0; c < 3; ++c) rgb[c] = clamp01(__fadd_rn(__fmul_rn(sp.albedo[c], lit), spec));
}

// Normalization + zero-gradient fallback of neural_normal_map (shade.cpp:19-40).
__device__ __forceinline__ bool normalize_normal(float gx, float gy, float gz, float n[3]) {
  const float n2 = dot3_rn(gx, gy, gz, gx, gy, gz);
  if (n2 < 1e-16f) return false;
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(n2));
  n[0] = __fmul_rn(gx, inv);
  n[1] = __fmul_rn(gy, inv);
  n[2] = __fmul_rn(gz, inv);
  return true;
}


__device__ __forceinline__ void shade_and_write(const ShadeParams& sp, const RayState& st, int slot, const float n[3],
                                                float* rgb, float* depth, uint8_t* mask) {
  float c[3];
  shade_point(sp, st.px[slot], st.py[slot], st.pz[slot], n[0], n[1], n[2], c);
  const int p = st.pixel[slot];
  if (!in_bounds(p, st.n_pix, kChkPixel)) return;
  rgb[size_t(3) * p + 0] = c[0];
  rgb[size_t(3) * p + 1] = c[1];
  rgb[size_t(3) * p + 2] = c[2];
  depth[p] = st.t[slot];
  mask[p] = 1;
}

}  // namespace nsdf_b200
