// TEST INFRASTRUCTURE ONLY (oracle build).
//
// Minimal C++ value wrappers over the GMP C API (see gmp.h beside this file),
// covering the subset of gmpxx that the reference headers use: mpz_class and
// mpq_class with mixed integral arithmetic, comparisons, shifts and stream
// output.  No expression templates: every operation materialises its result,
// which only affects the speed of the reference's setup-time bignum code.
#pragma once

#include <gmp.h>

#include <cstdlib>
#include <ostream>
#include <string>
#include <type_traits>
#include <utility>

class mpz_class {
 public:
  mpz_class() { mpz_init(z_); }
  mpz_class(const mpz_class& o) { mpz_init_set(z_, o.z_); }
  mpz_class(mpz_class&& o) noexcept {
    mpz_init(z_);
    mpz_swap(z_, o.z_);
  }
  template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
  mpz_class(T v) {  // NOLINT: implicit on purpose, mirrors gmpxx
    if constexpr (std::is_signed_v<T>)
      mpz_init_set_si(z_, (long)v);
    else
      mpz_init_set_ui(z_, (unsigned long)v);
  }
  explicit mpz_class(const char* s, int base = 10) {
    mpz_init(z_);
    mpz_set_str(z_, s, base);
  }
  explicit mpz_class(const std::string& s, int base = 10) : mpz_class(s.c_str(), base) {}
  explicit mpz_class(mpz_srcptr p) { mpz_init_set(z_, p); }
  ~mpz_class() { mpz_clear(z_); }

  mpz_class& operator=(const mpz_class& o) {
    if (this != &o) mpz_set(z_, o.z_);
    return *this;
  }
  mpz_class& operator=(mpz_class&& o) noexcept {
    mpz_swap(z_, o.z_);
    return *this;
  }
  template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
  mpz_class& operator=(T v) {
    if constexpr (std::is_signed_v<T>)
      mpz_set_si(z_, (long)v);
    else
      mpz_set_ui(z_, (unsigned long)v);
    return *this;
  }

  mpz_ptr get_mpz_t() { return z_; }
  mpz_srcptr get_mpz_t() const { return z_; }
  std::string get_str(int base = 10) const {
    char* s = mpz_get_str(nullptr, base, z_);
    std::string out(s);
    std::free(s);
    return out;
  }
  long get_si() const { return mpz_get_si(z_); }
  unsigned long get_ui() const { return mpz_get_ui(z_); }
  bool fits_slong_p() const { return mpz_fits_slong_p(z_) != 0; }

  mpz_class& operator+=(const mpz_class& o) { mpz_add(z_, z_, o.z_); return *this; }
  mpz_class& operator-=(const mpz_class& o) { mpz_sub(z_, z_, o.z_); return *this; }
  mpz_class& operator*=(const mpz_class& o) { mpz_mul(z_, z_, o.z_); return *this; }
  mpz_class& operator/=(const mpz_class& o) { mpz_tdiv_q(z_, z_, o.z_); return *this; }
  mpz_class& operator%=(const mpz_class& o) { mpz_tdiv_r(z_, z_, o.z_); return *this; }
  mpz_class& operator<<=(unsigned long s) { mpz_mul_2exp(z_, z_, s); return *this; }
  mpz_class& operator>>=(unsigned long s) { mpz_fdiv_q_2exp(z_, z_, s); return *this; }

 private:
  mpz_t z_;
};

inline mpz_class operator+(const mpz_class& a, const mpz_class& b) {
  mpz_class r; mpz_add(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator-(const mpz_class& a, const mpz_class& b) {
  mpz_class r; mpz_sub(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator*(const mpz_class& a, const mpz_class& b) {
  mpz_class r; mpz_mul(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator/(const mpz_class& a, const mpz_class& b) {
  mpz_class r; mpz_tdiv_q(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator%(const mpz_class& a, const mpz_class& b) {
  mpz_class r; mpz_tdiv_r(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator&(const mpz_class& a, const mpz_class& b) {
  mpz_class r; mpz_and(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r;
}
inline mpz_class operator-(const mpz_class& a) {
  mpz_class r; mpz_neg(r.get_mpz_t(), a.get_mpz_t()); return r;
}
inline mpz_class operator<<(const mpz_class& a, unsigned long s) {
  mpz_class r; mpz_mul_2exp(r.get_mpz_t(), a.get_mpz_t(), s); return r;
}
inline mpz_class operator>>(const mpz_class& a, unsigned long s) {
  mpz_class r; mpz_fdiv_q_2exp(r.get_mpz_t(), a.get_mpz_t(), s); return r;
}
inline int cmp(const mpz_class& a, const mpz_class& b) { return mpz_cmp(a.get_mpz_t(), b.get_mpz_t()); }
inline bool operator==(const mpz_class& a, const mpz_class& b) { return cmp(a, b) == 0; }
inline bool operator!=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) != 0; }
inline bool operator<(const mpz_class& a, const mpz_class& b) { return cmp(a, b) < 0; }
inline bool operator<=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) <= 0; }
inline bool operator>(const mpz_class& a, const mpz_class& b) { return cmp(a, b) > 0; }
inline bool operator>=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) >= 0; }
inline std::ostream& operator<<(std::ostream& os, const mpz_class& a) { return os << a.get_str(); }

class mpq_class {
 public:
  mpq_class() { mpq_init(q_); }
  mpq_class(const mpq_class& o) { mpq_init(q_); mpq_set(q_, o.q_); }
  mpq_class(mpq_class&& o) noexcept { mpq_init(q_); mpq_swap(q_, o.q_); }
  mpq_class(const mpz_class& z) { mpq_init(q_); mpq_set_z(q_, z.get_mpz_t()); }  // NOLINT
  template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
  mpq_class(T v) {  // NOLINT
    mpq_init(q_);
    mpz_class z(v);
    mpq_set_z(q_, z.get_mpz_t());
  }
  mpq_class(const mpz_class& num, const mpz_class& den) {
    mpq_init(q_);
    mpz_set(mpq_numref(q_), num.get_mpz_t());
    mpz_set(mpq_denref(q_), den.get_mpz_t());
  }
  ~mpq_class() { mpq_clear(q_); }
  mpq_class& operator=(const mpq_class& o) {
    if (this != &o) mpq_set(q_, o.q_);
    return *this;
  }
  mpq_class& operator=(mpq_class&& o) noexcept { mpq_swap(q_, o.q_); return *this; }

  void canonicalize() { mpq_canonicalize(q_); }
  mpq_ptr get_mpq_t() { return q_; }
  mpq_srcptr get_mpq_t() const { return q_; }
  std::string get_str(int base = 10) const {
    char* s = mpq_get_str(nullptr, base, q_);
    std::string out(s);
    std::free(s);
    return out;
  }

 private:
  mpq_t q_;
};

inline mpq_class operator+(const mpq_class& a, const mpq_class& b) {
  mpq_class r; mpq_add(r.get_mpq_t(), a.get_mpq_t(), b.get_mpq_t()); return r;
}
inline mpq_class operator-(const mpq_class& a, const mpq_class& b) {
  mpq_class r; mpq_sub(r.get_mpq_t(), a.get_mpq_t(), b.get_mpq_t()); return r;
}
inline mpq_class operator*(const mpq_class& a, const mpq_class& b) {
  mpq_class r; mpq_mul(r.get_mpq_t(), a.get_mpq_t(), b.get_mpq_t()); return r;
}
inline mpq_class operator/(const mpq_class& a, const mpq_class& b) {
  mpq_class r; mpq_div(r.get_mpq_t(), a.get_mpq_t(), b.get_mpq_t()); return r;
}
inline mpq_class operator-(const mpq_class& a) {
  mpq_class r; mpq_neg(r.get_mpq_t(), a.get_mpq_t()); return r;
}
inline int cmp(const mpq_class& a, const mpq_class& b) { return mpq_cmp(a.get_mpq_t(), b.get_mpq_t()); }
inline bool operator==(const mpq_class& a, const mpq_class& b) { return cmp(a, b) == 0; }
inline bool operator!=(const mpq_class& a, const mpq_class& b) { return cmp(a, b) != 0; }
inline bool operator<(const mpq_class& a, const mpq_class& b) { return cmp(a, b) < 0; }
inline bool operator<=(const mpq_class& a, const mpq_class& b) { return cmp(a, b) <= 0; }
inline bool operator>(const mpq_class& a, const mpq_class& b) { return cmp(a, b) > 0; }
inline bool operator>=(const mpq_class& a, const mpq_class& b) { return cmp(a, b) >= 0; }
inline std::ostream& operator<<(std::ostream& os, const mpq_class& a) { return os << a.get_str(); }
