// Brute-force point count on the device (see count.cu).
#pragma once

#include "../host/cohom.hpp"

namespace drzg {

// #X(F_{p^r}) for the hypersurface, same enumeration and budget rule as the
// reference count_points (oracle.hpp:190-245)
i64 count_points_device(const Hypersurface& X, int r, i64 budget);

// host enumeration below this many points (launch latency wins)
constexpr i64 kDeviceCountMin = 100000;

}  // namespace drzg
