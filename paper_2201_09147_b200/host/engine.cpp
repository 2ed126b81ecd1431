#include "engine.hpp"

#include <cstdlib>
#include <cstring>
#include <mutex>

namespace nsdf::engine {

namespace {
std::once_flag g_once;
nsdf_ctx* g_ctx = nullptr;
int g_status = NSDF_OK;
std::string g_message;
}  // namespace

void check(int status) {
  if (status == NSDF_OK) return;
  const std::string msg = nsdf_cuda_last_error();
  switch (status) {
    case NSDF_ERR_CONTRACT: throw Error(ErrorKind::contract, msg);
    case NSDF_ERR_CONFIG: throw Error(ErrorKind::config, msg);
    case NSDF_ERR_PARSE: throw Error(ErrorKind::parse, msg);
    case NSDF_ERR_DIVERGENCE: throw Error(ErrorKind::divergence, msg);
    default: throw Error(ErrorKind::validation, msg);  // validation and device failures
  }
}

nsdf_ctx* context() {
  std::call_once(g_once, [] {
    int device = 0;
    if (const char* d = std::getenv("NSDF_DEVICE")) device = std::atoi(d);
    g_status = nsdf_cuda_create(device, &g_ctx);
    if (g_status != NSDF_OK) {
      g_message = nsdf_cuda_last_error();
      g_ctx = nullptr;
      return;
    }
    int mode = NSDF_MODE_FP16_FAST;
    if (const char* m = std::getenv("NSDF_MODE")) {
      if (!std::strcmp(m, "oracle") || !std::strcmp(m, "fp32")) mode = NSDF_MODE_FP32_ORACLE;
      else if (!std::strcmp(m, "low") || !std::strcmp(m, "fp16low")) mode = NSDF_MODE_FP16_LOW;
    }
    nsdf_cuda_set_mode(g_ctx, mode);
  });
  if (!g_ctx) throw Error(ErrorKind::validation, "nsdf B200 engine unavailable: " + g_message);
  return g_ctx;
}

void unsupported(const std::string& what) {
  throw Error(ErrorKind::config, what + " is not provided by the nsdf B200 engine (float render path only)");
}

}  // namespace nsdf::engine
