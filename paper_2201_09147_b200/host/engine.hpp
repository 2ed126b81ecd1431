// Process-wide access to the B200 engine for the drop-in C++ API: one nsdf_ctx per process
// (device NSDF_DEVICE, default 0; mode NSDF_MODE = fast | oracle | low, default fast).
#pragma once

#include <string>

#include "nsdf/core.hpp"
#include "nsdf_cuda.h"

namespace nsdf::engine {

nsdf_ctx* context();                 // creates on first use; throws Error on failure
void check(int status);              // nsdf_status -> nsdf::Error (device errors -> validation)
[[noreturn]] void unsupported(const std::string& what);

}  // namespace nsdf::engine
