/*
 * nsdf_host.h — extern "C" entry points of libnsdf_b200.so, the drop-in C++ library that
 * re-implements the reference API (include/nsdf/*.hpp) over libnsdf_cuda.so.  These let a
 * C / ctypes caller drive the reference-shaped chain end to end:
 *   fields::load_manifest -> shading::render | tracer::trace_image | mlp::*_batch.
 * Return nsdf_status; nsdf_host_last_error() has the message.
 */
#ifndef NSDF_HOST_H_
#define NSDF_HOST_H_

#include "nsdf_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* nsdf_host_last_error(void);
int nsdf_host_render_manifest(const char* manifest, double time, const nsdf_camera* camera,
                              const nsdf_trace_config* trace, const nsdf_shade_config* shade,
                              int normal_source, int fine_index, float* rgb, float* depth,
                              uint8_t* mask);
int nsdf_host_trace_image_manifest(const char* manifest, double time, const nsdf_camera* camera,
                                   const nsdf_trace_config* trace, nsdf_hit_record* out);
int nsdf_host_forward_and_gradient(const char* sdfnet, const float* points, int k, float* dist,
                                   float* grad);

#ifdef __cplusplus
}
#endif

#endif /* NSDF_HOST_H_ */
