#include "engine.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

namespace nsdf::engine {

namespace {
std::once_flag g_once;
std::vector<nsdf_ctx*> g_ctxs;
int g_status = NSDF_OK;
std::string g_message;
std::mutex g_rep_mu;
std::map<std::pair<nsdf_field, size_t>, nsdf_field> g_replicas;  // (primary handle, context) -> handle

int parse_mode(const char* m) {
  if (!m || !*m || !std::strcmp(m, "fast") || !std::strcmp(m, "fp16")) return NSDF_MODE_FP16_FAST;
  if (!std::strcmp(m, "oracle") || !std::strcmp(m, "fp32")) return NSDF_MODE_FP32_ORACLE;
  if (!std::strcmp(m, "low") || !std::strcmp(m, "fp16low")) return NSDF_MODE_FP16_LOW;
  return -1;
}

std::vector<int> parse_devices(int primary) {
  std::vector<int> out{primary};
  const char* e = std::getenv("NSDF_DEVICES");
  if (!e || !*e) return out;
  if (!std::strcmp(e, "all")) {
    int n = 0;
    if (nsdf_cuda_device_count(&n) != NSDF_OK) return out;
    for (int d = 0; d < n; ++d)
      if (d != primary) out.push_back(d);
    return out;
  }
  out.clear();
  std::string s(e);
  size_t pos = 0;
  while (pos <= s.size()) {
    const size_t comma = std::min(s.find(',', pos), s.size());
    const std::string tok = s.substr(pos, comma - pos);
    if (!tok.empty()) {
      char* end = nullptr;
      const long d = std::strtol(tok.c_str(), &end, 10);
      if (!end || *end || d < 0) throw Error(ErrorKind::config, "NSDF_DEVICES: bad device '" + tok + "'");
      out.push_back(int(d));  // a repeated device gets another context (own stream + workspace)
    }
    pos = comma + 1;
  }
  if (out.empty()) throw Error(ErrorKind::config, "NSDF_DEVICES lists no device");
  return out;
}
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

const std::vector<nsdf_ctx*>& contexts() {
  std::call_once(g_once, [] {
    const char* m = std::getenv("NSDF_MODE");
    const int mode = parse_mode(m);
    if (mode < 0) {
      g_status = NSDF_ERR_CONFIG;
      g_message = std::string("NSDF_MODE='") + m + "' is not one of fast | fp16 | oracle | fp32 | low | fp16low";
      return;
    }
    int primary = 0;
    if (const char* d = std::getenv("NSDF_DEVICE")) primary = std::atoi(d);
    std::vector<int> devices;
    try {
      devices = parse_devices(primary);
    } catch (const Error& e) {
      g_status = NSDF_ERR_CONFIG;
      g_message = e.what();
      return;
    }
    for (int dev : devices) {
      nsdf_ctx* c = nullptr;
      g_status = nsdf_cuda_create(dev, &c);
      if (g_status == NSDF_OK) g_status = nsdf_cuda_set_mode(c, mode);
      if (g_status != NSDF_OK) {
        g_message = nsdf_cuda_last_error();
        for (nsdf_ctx* o : g_ctxs) nsdf_cuda_destroy(o);
        if (c) nsdf_cuda_destroy(c);
        g_ctxs.clear();
        return;
      }
      g_ctxs.push_back(c);
    }
  });
  if (g_ctxs.empty()) {
    if (g_status == NSDF_ERR_CONFIG) throw Error(ErrorKind::config, g_message);
    throw Error(ErrorKind::validation, "nsdf B200 engine unavailable: " + g_message);
  }
  return g_ctxs;
}

nsdf_ctx* context() { return contexts()[0]; }

nsdf_field replica(size_t i, nsdf_field h) {
  const auto& cs = contexts();
  if (i == 0) return h;
  std::lock_guard<std::mutex> lk(g_rep_mu);
  auto it = g_replicas.find({h, i});
  if (it != g_replicas.end()) return it->second;
  nsdf_field r = 0;
  check(nsdf_cuda_replicate_field(cs[0], h, cs[i], &r));
  g_replicas[{h, i}] = r;
  return r;
}

void forget(nsdf_field h) {
  if (g_ctxs.size() < 2) return;
  std::lock_guard<std::mutex> lk(g_rep_mu);
  for (size_t i = 1; i < g_ctxs.size(); ++i) {
    auto it = g_replicas.find({h, i});
    if (it == g_replicas.end()) continue;
    nsdf_cuda_release(g_ctxs[i], it->second);
    g_replicas.erase(it);
  }
}

int tile_size() {
  const char* e = std::getenv("NSDF_TILE");
  const int t = e ? std::atoi(e) : 32;
  return t > 0 ? t : 32;
}

void unsupported(const std::string& what) {
  throw Error(ErrorKind::config, what + " is not provided by the nsdf B200 engine (float render path only)");
}

}  // namespace nsdf::engine
