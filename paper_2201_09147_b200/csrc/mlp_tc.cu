// tcgen05 fast path (FP16 operands, FP32 TMEM accumulators).  Round-1 placeholder: the
// fast mode is not enabled yet, so every launcher declines and the FFMA tiles run.
#include "mlp_tc.cuh"

namespace nsdf_b200 {

bool tc_supported(const DevNet&) { return false; }

bool tc_trace_iter(const LevelDesc&, float, float, int, const int*, const int*, int*, int*, int*, int*,
                   const RayState&, int, cudaStream_t) {
  return false;
}
bool tc_normals_shade(const DevField&, float, const int*, const int*, int, const RayState&, const ShadeParams&, bool,
                      int*, int*, float*, float*, uint8_t*, cudaStream_t) {
  return false;
}
bool tc_eval(const DevField&, const float*, int, int, float, float*, float*, cudaStream_t) { return false; }

}  // namespace nsdf_b200
