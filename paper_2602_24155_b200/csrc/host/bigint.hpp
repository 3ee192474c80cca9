// Arbitrary-precision integers for the host-side number theory (precision
// plan, kappa scales, unscaling, charpoly, coefficient recovery).  Thin RAII
// wrapper over the system libgmp.so.10 C entry points, declared here because
// the image ships the library without headers.  Nothing on the device path
// uses it.
#pragma once

#include <cstdlib>
#include <string>
#include <utility>

#include "common.hpp"

extern "C" {
struct drzg_mpz_struct {
  int alloc;
  int size;
  unsigned long* d;
};
void __gmpz_init(drzg_mpz_struct*);
void __gmpz_clear(drzg_mpz_struct*);
void __gmpz_set(drzg_mpz_struct*, const drzg_mpz_struct*);
void __gmpz_set_ui(drzg_mpz_struct*, unsigned long);
void __gmpz_set_si(drzg_mpz_struct*, long);
int __gmpz_set_str(drzg_mpz_struct*, const char*, int);
char* __gmpz_get_str(char*, int, const drzg_mpz_struct*);
unsigned long __gmpz_get_ui(const drzg_mpz_struct*);
long __gmpz_get_si(const drzg_mpz_struct*);
int __gmpz_fits_slong_p(const drzg_mpz_struct*);
void __gmpz_add(drzg_mpz_struct*, const drzg_mpz_struct*, const drzg_mpz_struct*);
void __gmpz_sub(drzg_mpz_struct*, const drzg_mpz_struct*, const drzg_mpz_struct*);
void __gmpz_mul(drzg_mpz_struct*, const drzg_mpz_struct*, const drzg_mpz_struct*);
void __gmpz_mul_si(drzg_mpz_struct*, const drzg_mpz_struct*, long);
void __gmpz_mul_2exp(drzg_mpz_struct*, const drzg_mpz_struct*, unsigned long);
void __gmpz_neg(drzg_mpz_struct*, const drzg_mpz_struct*);
int __gmpz_cmp(const drzg_mpz_struct*, const drzg_mpz_struct*);
int __gmpz_cmp_si(const drzg_mpz_struct*, long);
void __gmpz_tdiv_q(drzg_mpz_struct*, const drzg_mpz_struct*, const drzg_mpz_struct*);
void __gmpz_fdiv_r(drzg_mpz_struct*, const drzg_mpz_struct*, const drzg_mpz_struct*);
unsigned long __gmpz_fdiv_q_ui(drzg_mpz_struct*, const drzg_mpz_struct*, unsigned long);
void __gmpz_fdiv_q_2exp(drzg_mpz_struct*, const drzg_mpz_struct*, unsigned long);
int __gmpz_invert(drzg_mpz_struct*, const drzg_mpz_struct*, const drzg_mpz_struct*);
void __gmpz_ui_pow_ui(drzg_mpz_struct*, unsigned long, unsigned long);
void __gmpz_bin_uiui(drzg_mpz_struct*, unsigned long, unsigned long);
int __gmpz_divisible_p(const drzg_mpz_struct*, const drzg_mpz_struct*);
int __gmpz_divisible_ui_p(const drzg_mpz_struct*, unsigned long);
void __gmpz_divexact(drzg_mpz_struct*, const drzg_mpz_struct*, const drzg_mpz_struct*);
}

namespace drzg {

class Z {
 public:
  Z() { __gmpz_init(&z_); }
  Z(long v) { __gmpz_init(&z_); __gmpz_set_si(&z_, v); }  // NOLINT
  static Z from_u64(u64 v) { Z r; __gmpz_set_ui(&r.z_, (unsigned long)v); return r; }
  static Z from_u128(u128 v) {
    Z hi = from_u64((u64)(v >> 64)), lo = from_u64((u64)v), r;
    __gmpz_mul_2exp(&r.z_, &hi.z_, 64);
    __gmpz_add(&r.z_, &r.z_, &lo.z_);
    return r;
  }
  static Z from_str(const std::string& s) {
    Z r;
    DRZG_REQUIRE(__gmpz_set_str(&r.z_, s.c_str(), 10) == 0, "Z: bad integer literal");
    return r;
  }
  static Z pow(u64 b, u64 e) { Z r; __gmpz_ui_pow_ui(&r.z_, b, e); return r; }
  static Z binom(u64 n, u64 k) { Z r; __gmpz_bin_uiui(&r.z_, n, k); return r; }
  Z(const Z& o) { __gmpz_init(&z_); __gmpz_set(&z_, &o.z_); }
  Z(Z&& o) noexcept { __gmpz_init(&z_); std::swap(z_, o.z_); }
  ~Z() { __gmpz_clear(&z_); }
  Z& operator=(const Z& o) { if (this != &o) __gmpz_set(&z_, &o.z_); return *this; }
  Z& operator=(Z&& o) noexcept { std::swap(z_, o.z_); return *this; }

  std::string str() const {
    char* s = __gmpz_get_str(nullptr, 10, &z_);
    std::string out(s);
    std::free(s);
    return out;
  }
  bool fits_long() const { return __gmpz_fits_slong_p(&z_) != 0; }
  long to_long() const { return __gmpz_get_si(&z_); }
  u64 to_u64() const { DRZG_REQUIRE(sign() >= 0, "Z: negative to u64"); return __gmpz_get_ui(&z_); }
  u128 to_u128() const {
    DRZG_REQUIRE(sign() >= 0, "Z: negative to u128");
    Z hi;
    __gmpz_fdiv_q_2exp(&hi.z_, &z_, 64);
    Z lo = *this - (hi << 64);
    return ((u128)__gmpz_get_ui(&hi.z_) << 64) | __gmpz_get_ui(&lo.z_);
  }
  int sign() const { return z_.size < 0 ? -1 : (z_.size > 0 ? 1 : 0); }
  bool is_zero() const { return z_.size == 0; }

  friend Z operator+(const Z& a, const Z& b) { Z r; __gmpz_add(&r.z_, &a.z_, &b.z_); return r; }
  friend Z operator-(const Z& a, const Z& b) { Z r; __gmpz_sub(&r.z_, &a.z_, &b.z_); return r; }
  friend Z operator*(const Z& a, const Z& b) { Z r; __gmpz_mul(&r.z_, &a.z_, &b.z_); return r; }
  friend Z operator-(const Z& a) { Z r; __gmpz_neg(&r.z_, &a.z_); return r; }
  // truncating quotient (callers only divide exactly)
  friend Z operator/(const Z& a, const Z& b) { Z r; __gmpz_tdiv_q(&r.z_, &a.z_, &b.z_); return r; }
  friend Z operator<<(const Z& a, unsigned long s) { Z r; __gmpz_mul_2exp(&r.z_, &a.z_, s); return r; }
  Z& operator+=(const Z& o) { __gmpz_add(&z_, &z_, &o.z_); return *this; }
  Z& operator-=(const Z& o) { __gmpz_sub(&z_, &z_, &o.z_); return *this; }
  Z& operator*=(const Z& o) { __gmpz_mul(&z_, &z_, &o.z_); return *this; }
  friend bool operator==(const Z& a, const Z& b) { return __gmpz_cmp(&a.z_, &b.z_) == 0; }
  friend bool operator!=(const Z& a, const Z& b) { return __gmpz_cmp(&a.z_, &b.z_) != 0; }
  friend bool operator<(const Z& a, const Z& b) { return __gmpz_cmp(&a.z_, &b.z_) < 0; }
  friend bool operator>(const Z& a, const Z& b) { return __gmpz_cmp(&a.z_, &b.z_) > 0; }
  friend bool operator<=(const Z& a, const Z& b) { return __gmpz_cmp(&a.z_, &b.z_) <= 0; }
  friend bool operator>=(const Z& a, const Z& b) { return __gmpz_cmp(&a.z_, &b.z_) >= 0; }

  // floor remainder in [0, m)
  Z mod(const Z& m) const { Z r; __gmpz_fdiv_r(&r.z_, &z_, &m.z_); return r; }
  bool divisible_by(const Z& m) const { return __gmpz_divisible_p(&z_, &m.z_) != 0; }
  bool divisible_by(u64 m) const { return __gmpz_divisible_ui_p(&z_, m) != 0; }
  Z divexact(const Z& m) const { Z r; __gmpz_divexact(&r.z_, &z_, &m.z_); return r; }
  Z inverse_mod(const Z& m) const {
    Z r;
    DRZG_REQUIRE(__gmpz_invert(&r.z_, &z_, &m.z_) != 0, "Z: not invertible");
    return r;
  }
  // centered representative in (-m/2, m/2]
  Z centered(const Z& m) const {
    Z r = mod(m);
    if (r + r > m) r -= m;
    return r;
  }
  // v_p(x) capped at cap (x == 0 reports cap)
  int valuation(u64 p, int cap) const {
    if (is_zero()) return cap;
    Z t = *this;
    if (t.sign() < 0) t = -t;
    int v = 0;
    while (v < cap && t.divisible_by(p)) {
      Z q;
      __gmpz_fdiv_q_ui(&q.z_, &t.z_, p);
      t = q;
      ++v;
    }
    return v;
  }

 private:
  drzg_mpz_struct z_;
};

}  // namespace drzg
