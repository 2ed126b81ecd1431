// FP64 Cephes sin/cos shared by the device FP64 paths (mlp_f64.cu, train_f64.cu): the double
// scheme of the reference's AVX2 lanes (sincos_poly_avx2_d, kernels_avx2.cpp:284-333; constants
// sincos_poly.hpp:26-40) with every operation separately rounded; the quadrant uses the lanes'
// 32-bit truncation (cvttpd).  Include only from TUs compiled with -fmad=false.
#pragma once

namespace nsdf_b200 {

__device__ __forceinline__ void sincos_ref_d(double x, double& s, double& c) {
  const double kFourOverPiD = 1.2732395447351626862;
  const double kDp1D = -7.85398125648498535156e-1;
  const double kDp2D = -3.77489470793079817668e-8;
  const double kDp3D = -2.69515142907905952645e-15;
  const double kSinD[6] = {1.58962301576546568060e-10, -2.50507477628578072866e-8, 2.75573136213857245213e-6,
                           -1.98412698295895385996e-4, 8.33333333332211858878e-3,  -1.66666666666666307295e-1};
  const double kCosD[6] = {-1.13585365213876817300e-11, 2.08757008419747316778e-9, -2.75573141792967388112e-7,
                           2.48015872888517179954e-5,   -1.38888888888730564116e-3, 4.16666666666665929218e-2};
  const unsigned long long bits = __double_as_longlong(x);
  const unsigned long long sign_sin = bits & 0x8000000000000000ull;
  const double ax = __longlong_as_double(bits & 0x7fffffffffffffffull);
  double y = __dmul_rn(ax, kFourOverPiD);
  int q = __double2int_rz(y);  // _mm256_cvttpd_epi32
  q = (q + 1) & ~1;
  y = __int2double_rn(q);
  const long long q64 = q;
  const unsigned long long swap_sign = (unsigned long long)(q64 & 4) << 61;
  const bool poly_sin = (q64 & 2) == 0;
  double r = ax;
  r = __dadd_rn(r, __dmul_rn(y, kDp1D));
  r = __dadd_rn(r, __dmul_rn(y, kDp2D));
  r = __dadd_rn(r, __dmul_rn(y, kDp3D));
  const double z = __dmul_rn(r, r);
  double pc = kCosD[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) pc = __dadd_rn(__dmul_rn(pc, z), kCosD[i]);
  pc = __dmul_rn(__dmul_rn(pc, z), z);
  pc = __dsub_rn(pc, __dmul_rn(z, 0.5));
  pc = __dadd_rn(pc, 1.0);
  double ps = kSinD[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) ps = __dadd_rn(__dmul_rn(ps, z), kSinD[i]);
  ps = __dmul_rn(__dmul_rn(ps, z), r);
  ps = __dadd_rn(ps, r);
  const double ysin = poly_sin ? ps : pc;
  s = __longlong_as_double(__double_as_longlong(ysin) ^ sign_sin ^ swap_sign);
  const long long qc = q64 - 2;
  const unsigned long long cos_sign = (unsigned long long)(~qc & 4) << 61;
  const bool cos_poly_sin = (qc & 2) == 0;
  const double ycos = cos_poly_sin ? ps : pc;
  c = __longlong_as_double(__double_as_longlong(ycos) ^ cos_sign);
}


}  // namespace nsdf_b200
