// Exact division / balanced residues by the small digit base q on the device.
#pragma once

#include <stdint.h>

namespace drzg {

// exact floor division / balanced residue by a small q (q <= 255) for
// |x| < 2^30: u = x + q*2^30 >= 0, floor(u / q) = mulhi64(u, ceil(2^64/q))
// (exact because u < 2^39 and q < 2^8)
//
// Fast path (|x| < 2^23, q odd): t = rint(x * (1/q)) in fp32 is the nearest
// integer to x/q exactly — the relative error of the product is < 2^-24, so
// the absolute error is < 2^-1/q, below the 1/(2q) gap between x/q and any
// half-integer — and x - q*t is the balanced residue.
struct FastQ {
  int q = 0;
  unsigned long long magic = 0;
  long long off = 0;  // q * 2^30
  float inv = 0.f;    // 1/q rounded
  static FastQ make(int q) {
    FastQ f;
    f.q = q;
    f.magic = ~0ull / (unsigned long long)q + 1;
    f.off = (long long)q << 30;
    f.inv = 1.0f / (float)q;
    return f;
  }
#ifdef __CUDACC__
  // floor(x / q) and r = x - q*floor(x/q) in [0, q)
  __device__ __forceinline__ int divfloor(int x, int& r) const {
    unsigned long long u = (unsigned long long)((long long)x + off);
    unsigned long long d = __umul64hi(u, magic);
    r = (int)(u - d * (unsigned long long)q);
    return (int)((long long)d - (1ll << 30));
  }
  __device__ __forceinline__ int bal(int x) const {
    int r;
    divfloor(x, r);
    return r > (q >> 1) ? r - q : r;
  }
  // nearest quotient t and balanced residue x - q t, for |x| < 2^23
  __device__ __forceinline__ int balq(int x, int& t) const {
    float fx = (float)x;
    float ft = rintf(fx * inv);
    t = (int)ft;
    return x - q * t;
  }
  __device__ __forceinline__ int bal_fast(int x) const {
    int t;
    return balq(x, t);
  }
  // x / q for x divisible by q, |x| < 2^23
  __device__ __forceinline__ int div_exact_fast(int x) const { return (int)rintf((float)x * inv); }
#endif
};

}  // namespace drzg
