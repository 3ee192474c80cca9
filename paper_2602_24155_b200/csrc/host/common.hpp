// drzg: B200-native controlled-reduction engine (arXiv 2602.24155).
// Shared integer types and the always-on contract check.  Mirrors the
// reference's convention (common.hpp:19-27): a violated precondition throws
// an exception carrying file:line; the C-ABI layer turns it into a status
// code plus a thread-local message.
#pragma once

#include <sched.h>
#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>
#include <mutex>
#include <functional>
#include <condition_variable>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace drzg {

using u8 = std::uint8_t;
using i8 = std::int8_t;
using u32 = std::uint32_t;
using i32 = std::int32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;
using u128 = unsigned __int128;
using i128 = __int128;

struct contract_error : std::logic_error {
  contract_error(const std::string& msg, const char* file, int line)
      : std::logic_error(std::string(file) + ":" + std::to_string(line) + ": " + msg) {}
};

// run_zeta's two non-contract failures (reference zeta.hpp:17-22)
struct singular_input : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct escalation_exhausted : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define DRZG_REQUIRE(cond, msg)                                            \
  do {                                                                     \
    if (!(cond)) throw ::drzg::contract_error((msg), __FILE__, __LINE__);  \
  } while (0)

constexpr int kMaxVars = 6;

// --- word arithmetic mod m (m < 2^63 unless noted) ---------------------------
inline u64 addm(u64 a, u64 b, u64 m) {
  u64 s = a + b;
  return s >= m ? s - m : s;
}
inline u64 subm(u64 a, u64 b, u64 m) { return a >= b ? a - b : a + m - b; }
inline u64 mulm(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
inline u64 powm(u64 a, u64 e, u64 m) {
  u64 r = 1 % m;
  a %= m;
  for (; e; e >>= 1) {
    if (e & 1) r = mulm(r, a, m);
    a = mulm(a, a, m);
  }
  return r;
}
// inverse of a unit mod m (m need not be prime)
inline u64 invm(u64 a, u64 m) {
  i64 t = 0, nt = 1, r = (i64)m, nr = (i64)(a % m);
  while (nr) {
    i64 q = r / nr;
    i64 tmp = t - q * nt;
    t = nt;
    nt = tmp;
    tmp = r - q * nr;
    r = nr;
    nr = tmp;
  }
  DRZG_REQUIRE(r == 1, "invm: not a unit");
  return (u64)(t < 0 ? t + (i64)m : t);
}
inline u64 ipow(u64 p, int e) {
  u64 r = 1;
  for (int i = 0; i < e; ++i) {
    DRZG_REQUIRE(r <= ~u64(0) / p, "ipow overflow");
    r *= p;
  }
  return r;
}

// 128-bit residues: values below 2^80 multiply exactly by splitting b
inline u128 mulm128(u128 a, u128 b, u128 m) {
  DRZG_REQUIRE((m >> 80) == 0, "mulm128: modulus above 2^80");
  a %= m;
  b %= m;
  u128 hi = b >> 40, lo = b & ((u128(1) << 40) - 1);
  u128 r = (a * hi) % m;
  r = ((r << 40) + a * lo) % m;
  return r;
}

// host threads this process may run on: the affinity mask (a container's
// cpuset), not every CPU of the node (std::thread::hardware_concurrency);
// oversubscribed host threads stall the launcher and leave the GPU idle
inline unsigned usable_cores() {
  static const unsigned n = [] {
    cpu_set_t set;
    CPU_ZERO(&set);
    if (sched_getaffinity(0, sizeof(set), &set) == 0) {
      const int c = CPU_COUNT(&set);
      if (c > 0) return (unsigned)c;
    }
    const unsigned h = std::thread::hardware_concurrency();
    return h ? h : 1u;
  }();
  return n;
}

// A fork-join pool kept for a whole run: run(parts, f) calls f(0..parts-1),
// part 0 on the calling thread, and returns when all are done (the p-chunk
// policy's per-sweep moves; spawning threads per sweep cost ~0.5 ms a sweep)
class ForkJoin {
 public:
  explicit ForkJoin(int threads) {
    for (int t = 1; t < threads; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  ~ForkJoin() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return (int)workers_.size() + 1; }
  void run(int parts, const std::function<void(int)>& f) {
    parts = std::max(1, std::min(parts, size()));
    {
      std::lock_guard<std::mutex> lk(mu_);
      f_ = &f;
      parts_ = parts;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    f_ = nullptr;
  }

 private:
  void loop(int t) {
    unsigned long long seen = 0;
    for (;;) {
      const std::function<void(int)>* f = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (t >= parts_) continue;
        f = f_;
      }
      (*f)(t);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* f_ = nullptr;
  int parts_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

// calls in flight in this process (frobenius_matrix on several host threads,
// e.g. a batch of hypersurfaces): their host thread pools share the cores
inline std::atomic<int>& active_calls() {
  static std::atomic<int> a{0};
  return a;
}
struct ActiveCall {
  ActiveCall() { active_calls().fetch_add(1); }
  ~ActiveCall() { active_calls().fetch_sub(1); }
};
// this call's share of the cores
inline unsigned call_cores() {
  const int a = std::max(1, active_calls().load());
  return std::max(1u, usable_cores() / (unsigned)a);
}

}  // namespace drzg
