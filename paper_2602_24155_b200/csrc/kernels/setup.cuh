// Setup-time eliminations on the device (see setup.cu).
#pragma once

#include <cstdlib>
#include <string>
#include <vector>

#include "../host/common.hpp"

namespace drzg {

// forward elimination over F_p with the first-nonzero pivot rule: pivot column
// of every row (or -1); m is rows x cols with entries in [0, p)
std::vector<int> pivot_scan_device(u64 p, int rows, int cols, const std::vector<u32>& m);

// inverse of an n x n matrix over Z/q (q = p^e < 256), entries in [0, q)
std::vector<u32> inverse_mod_q_device(u64 p, u64 q, int n, const std::vector<u32>& a);

// order at which the device versions are used (host below: launch latency wins)
constexpr int kDeviceSetupMin = 768;
// DRZG_SETUP=host|device overrides the size rule (tests compare both)
inline bool use_device_setup(int n) {
  const char* e = std::getenv("DRZG_SETUP");
  if (e && std::string(e) == "host") return false;
  if (e && std::string(e) == "device") return true;
  return n >= kDeviceSetupMin;
}

}  // namespace drzg
