// Rng (xoshiro256++ with splitmix64 seeding, the published algorithms) and the host
// chunk runner kept for API compatibility (reference core.hpp:75-138).
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "nsdf/core.hpp"

namespace nsdf {

namespace {
inline uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
inline uint64_t splitmix64(uint64_t& state) {
  state += 0x9e3779b97f4a7c15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
}  // namespace

Rng::Rng(uint64_t seed) {
  uint64_t state = seed;
  for (auto& w : s_) w = splitmix64(state);
}

uint64_t Rng::next_u64() {
  const uint64_t out = rotl64(s_[0] + s_[3], 23) + s_[0];
  const uint64_t t = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= t;
  s_[3] = rotl64(s_[3], 45);
  return out;
}

double Rng::uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }

double Rng::normal(double mean, double sigma) {
  double u1 = uniform();
  const double u2 = uniform();
  while (u1 <= 1e-300) u1 = uniform();
  return mean + sigma * std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

Vec3 Rng::uniform_in_box(const Aabb& b) {
  const double x = uniform(b.lo.x, b.hi.x);
  const double y = uniform(b.lo.y, b.hi.y);
  const double z = uniform(b.lo.z, b.hi.z);
  return {x, y, z};
}

Rng Rng::fork(uint64_t stream_index) const {
  Rng r(0);
  r.s_ = s_;
  Rng mix(stream_index * 0x2545f4914f6cdd1dull + 0x9e3779b97f4a7c15ull);
  for (auto& w : r.s_) w ^= mix.next_u64();
  r.next_u64();
  return r;
}

int worker_thread_count() {
  static const int n = [] {
    if (const char* e = std::getenv("NSDF_THREADS")) {
      const int v = std::atoi(e);
      if (v > 0) return v;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? int(hw) : 1;
  }();
  return n;
}

void parallel_chunks(int chunk_count, const std::function<void(int)>& fn) {
  if (chunk_count <= 0) return;
  const int workers = std::min(worker_thread_count(), chunk_count);
  if (workers <= 1) {
    for (int i = 0; i < chunk_count; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  std::atomic<bool> stop{false};
  std::exception_ptr err;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&] {
      for (int i; !stop.load() && (i = next.fetch_add(1)) < chunk_count;) {
        try {
          fn(i);
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          if (!err) err = std::current_exception();
          stop = true;
        }
      }
    });
  for (auto& t : pool) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace nsdf
