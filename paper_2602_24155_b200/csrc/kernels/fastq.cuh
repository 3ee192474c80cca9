// Exact division / balanced residues by the small digit base q on the device.
#pragma once

#include <stdint.h>

namespace drzg {

// exact floor division / balanced residue by a small q (q <= 255) for
// |x| < 2^30: u = x + q*2^30 >= 0, floor(u / q) = mulhi64(u, ceil(2^64/q))
// (exact because u < 2^39 and q < 2^8)
//
// Fast path (|x| < 2^22): x' = x + q*K with K = ceil(2^22/q) is in [0, 2^23),
// and for x' < 2^32/q (true for q < 512) floor(x'/q) = umulhi(x', ceil(2^32/q)):
// the magic's excess is < 1, so the product overshoots x'/q by < x'/2^32 <
// 1/q, which never crosses an integer.  All full-rate integer instructions.
struct FastQ {
  int q = 0;
  unsigned long long magic = 0;
  long long off = 0;  // q * 2^30
  unsigned m32 = 0;   // ceil(2^32 / q)
  int k22 = 0;        // ceil(2^22 / q)
  unsigned qinv = 0;  // q^{-1} mod 2^32 (q odd): exact division is one multiply
  static FastQ make(int q) {
    FastQ f;
    f.q = q;
    f.magic = ~0ull / (unsigned long long)q + 1;
    f.off = (long long)q << 30;
    f.m32 = (unsigned)(((1ull << 32) + (unsigned long long)q - 1) / (unsigned long long)q);
    f.k22 = (int)(((1 << 22) + q - 1) / q);
    unsigned inv = 1;  // Newton iteration for the inverse mod 2^32 (q odd)
    for (int i = 0; i < 5; ++i) inv *= 2u - (unsigned)q * inv;
    f.qinv = (q & 1) ? inv : 0u;
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
  // balanced residue x - q t and its quotient t, for |x| < 2^22
  __device__ __forceinline__ int balq(int x, int& t) const {
    unsigned xp = (unsigned)(x + q * k22);
    int tt = (int)__umulhi(xp, m32);
    int r = (int)xp - tt * q;
    tt -= k22;
    if (r > (q >> 1)) r -= q, ++tt;
    t = tt;
    return r;
  }
  __device__ __forceinline__ int bal_fast(int x) const {
    int t;
    return balq(x, t);
  }
  // x / q for x divisible by q (any int32 x, q odd): one multiply
  __device__ __forceinline__ int div_exact_inv(int x) const { return (int)((unsigned)x * qinv); }
  // balanced digit d = x - q t with |d| <= q/2 and its quotient t, for
  // |x| < 2^22, q odd: one add, a multiply-high and a multiply-add
  __device__ __forceinline__ int bal_split(int x, int& t) const {
    const int h = q >> 1;
    const unsigned xp = (unsigned)(x + h + q * k22);
    const int tq = (int)__umulhi(xp, m32);
    t = tq - k22;
    return (int)xp - tq * q - h;
  }
  // The packed variant of bal_split for |x| < 2^22 and odd q <= 255: with
  // the offset K = k22 rounded up to a multiple of 256 (x + h + qK stays below
  // 2^32 / q), tq = floor((x + h + qK) / q) has the quotient t in its low
  // byte (t = tq - K, K = 0 mod 256), and raw = x + h + qK - q tq in [0, q)
  // is the digit plus h: four raws are packed and h taken off bytewise
  // (unbias4), no per-element subtractions
  __device__ __forceinline__ unsigned hqk256() const {
    return (unsigned)((q >> 1) + q * (((k22 + 255) >> 8) << 8));
  }
  __device__ __forceinline__ int split_raw(int x, unsigned hqk, int& tq) const {
    const unsigned xp = (unsigned)x + hqk;
    tq = (int)__umulhi(xp, m32);
    return (int)xp - tq * q;
  }
  // bytes b in [0, q) -> b - h (two's complement), no carries between bytes:
  // b + 128 - h stays in [1, 255] for q <= 255
  __device__ __forceinline__ uint32_t unbias4(uint32_t packed) const {
    return (packed + 0x01010101u * (unsigned)(0x80 - (q >> 1))) ^ 0x80808080u;
  }
  // x / q for x divisible by q, |x| < 2^22
  __device__ __forceinline__ int div_exact_fast(int x) const {
    unsigned xp = (unsigned)(x + q * k22);
    return (int)__umulhi(xp, m32) - k22;
  }
#endif
};

}  // namespace drzg
