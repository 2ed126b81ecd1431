// nsdf-b200 extensions beyond the reference API (proj/include/nsdf has no multi-GPU calls):
// the engine's devices and frame-stream rendering across them.
#pragma once

#include <vector>

#include "nsdf/fields/nesting.hpp"
#include "nsdf/shading/shading.hpp"

namespace nsdf::b200 {

// Engine contexts of this process: NSDF_DEVICES ("0,1,2,3", "all"; a repeated device gets
// another context), else NSDF_DEVICE alone.
int context_count();

// The frames of an animation (nsdf_main.cpp:308-324: one slice per time, rendered in turn)
// sharded across the engine's contexts: frame f renders on context f % n, every context on
// its own device and thread concurrently (weights replicated device to device once per
// field); the images come back in frame order, each equal to shading::render of its slice.
std::vector<shading::ImageBuffer> render_frames(const fields::AnimatedSequence& anim, const std::vector<double>& times,
                                                const tracer::Camera& camera, const shading::RenderConfig& config);

}  // namespace nsdf::b200
