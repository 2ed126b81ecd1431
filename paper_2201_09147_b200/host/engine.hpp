// Process-wide access to the B200 engine for the drop-in C++ API: one nsdf_ctx per device
// (primary device NSDF_DEVICE, default 0; mode NSDF_MODE = fast | oracle | low, default fast;
// any other NSDF_MODE value is rejected with ErrorKind::config).
//
// Multi-GPU: NSDF_DEVICES = "0,1,2,3" or "all" makes shading::render split every frame's
// image tiles over those devices (nsdf_cuda_render_multi: weights replicated device to
// device once per field, every GPU stores its pixels into the primary GPU's framebuffer
// over NVLink).  The first listed device is the primary.  NSDF_TILE sets the tile edge
// (default 32 pixels).
#pragma once

#include <string>
#include <vector>

#include "nsdf/core.hpp"
#include "nsdf_cuda.h"

namespace nsdf::engine {

nsdf_ctx* context();                 // creates on first use; throws Error on failure
const std::vector<nsdf_ctx*>& contexts();  // [primary, others...] (NSDF_DEVICES); size >= 1
nsdf_field replica(size_t i, nsdf_field h);  // h (a primary-context field) in contexts()[i]
void forget(nsdf_field h);           // release h's replicas (field destructor)
int tile_size();                     // NSDF_TILE, default 32
void check(int status);              // nsdf_status -> nsdf::Error (device errors -> validation)
[[noreturn]] void unsupported(const std::string& what);

}  // namespace nsdf::engine
