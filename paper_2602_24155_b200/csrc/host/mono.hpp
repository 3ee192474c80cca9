// Exponent vectors and grevlex monomial indexing.
//
// The reference orders every graded piece grevlex-descending
// (monomial.hpp:84-149, comparator :84-93) and that order defines the row and
// column order of every operator and state vector.  Descending grevlex is the
// lexicographic order on the reversed exponent tuple (e[nv-1], ..., e[1]), so
// a monomial's position has a closed form (hockey-stick sums of binomials)
// that the device kernels evaluate without any table:
//   rank(e) = sum_{j=nv-1..1} [ C(rem_j + j, j) - C(rem_j - e_j + j, j) ],
//   rem_j = deg - sum_{i>j} e_i.
#pragma once

#include <array>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.hpp"

#ifndef DRZG_HD
#ifdef __CUDACC__
#define DRZG_HD __host__ __device__ __forceinline__
#else
#define DRZG_HD inline
#endif
#endif

namespace drzg {

struct Expo {
  int e[kMaxVars] = {0, 0, 0, 0, 0, 0};
  int nv = 0;

  DRZG_HD Expo() {}
  DRZG_HD explicit Expo(int n) : nv(n) {}
  DRZG_HD int& operator[](int i) { return e[i]; }
  DRZG_HD int operator[](int i) const { return e[i]; }
  DRZG_HD int total() const {
    int s = 0;
    for (int i = 0; i < nv; ++i) s += e[i];
    return s;
  }
  DRZG_HD bool nonneg() const {
    for (int i = 0; i < nv; ++i)
      if (e[i] < 0) return false;
    return true;
  }
  DRZG_HD bool operator==(const Expo& o) const {
    if (nv != o.nv) return false;
    for (int i = 0; i < nv; ++i)
      if (e[i] != o.e[i]) return false;
    return true;
  }
  DRZG_HD Expo operator+(const Expo& o) const {
    Expo r = *this;
    for (int i = 0; i < nv; ++i) r.e[i] += o.e[i];
    return r;
  }
  DRZG_HD Expo operator-(const Expo& o) const {
    Expo r = *this;
    for (int i = 0; i < nv; ++i) r.e[i] -= o.e[i];
    return r;
  }
  DRZG_HD static Expo ones(int nv) {
    Expo r(nv);
    for (int i = 0; i < nv; ++i) r.e[i] = 1;
    return r;
  }
  DRZG_HD static Expo unit(int nv, int i) {
    Expo r(nv);
    r.e[i] = 1;
    return r;
  }
  // packed key with `bits` bits per entry (entries must be in [0, 2^bits))
  DRZG_HD u64 pack(int bits) const {
    u64 k = 0;
    for (int i = 0; i < nv; ++i) k = (k << bits) | (u64)(u32)e[i];
    return k;
  }
};

// binomials C(a, b) for a < kBinomRows, as a flat table usable on the device
constexpr int kBinomRows = 1200;
constexpr int kBinomCols = kMaxVars + 1;

struct Binom {
  // C(a, b), b <= kMaxVars
  std::vector<u64> tab;
  Binom() : tab((size_t)kBinomRows * kBinomCols, 0) {
    for (int a = 0; a < kBinomRows; ++a) {
      tab[(size_t)a * kBinomCols] = 1;
      for (int b = 1; b < kBinomCols; ++b)
        tab[(size_t)a * kBinomCols + b] =
            a == 0 ? 0 : tab[(size_t)(a - 1) * kBinomCols + b - 1] + tab[(size_t)(a - 1) * kBinomCols + b];
    }
  }
  static const Binom& get() {
    static Binom b;
    return b;
  }
};

DRZG_HD u64 binom_lookup(const u64* tab, int a, int b) {
  if (a < 0 || b < 0 || b > a) return 0;
  return tab[(size_t)a * kBinomCols + b];
}

// number of degree-deg monomials in nv variables
inline i64 mono_count(int nv, int deg) {
  if (deg < 0) return 0;
  i64 r = 1;
  for (int i = 1; i <= nv - 1; ++i) r = r * (deg + i) / i;
  return r;
}

// closed-form grevlex-descending rank of e among degree-|e| monomials
DRZG_HD i64 grevlex_rank(const u64* btab, const Expo& e) {
  int rem = e.total();
  i64 r = 0;
  for (int j = e.nv - 1; j >= 1; --j) {
    r += (i64)binom_lookup(btab, rem + j, j) - (i64)binom_lookup(btab, rem - e.e[j] + j, j);
    rem -= e.e[j];
  }
  return r;
}

inline i64 rank_of(const Expo& e) {
  DRZG_REQUIRE(e.nonneg(), "rank_of: negative exponent");
  DRZG_REQUIRE(e.total() + e.nv < kBinomRows, "rank_of: degree beyond binomial table");
  return grevlex_rank(Binom::get().tab.data(), e);
}

// all degree-deg monomials in nv variables, grevlex-descending, cached
struct MonoList {
  int nv = 0, deg = 0;
  std::vector<Expo> mons;
  int size() const { return (int)mons.size(); }
};

namespace detail {
inline void gen_rev(int nv, int pos, int left, Expo& cur, std::vector<Expo>& out) {
  // lexicographic ascending on (e[nv-1], ..., e[1]); e[0] takes the rest
  if (pos == 0) {
    cur.e[0] = left;
    out.push_back(cur);
    return;
  }
  for (int v = 0; v <= left; ++v) {
    cur.e[pos] = v;
    gen_rev(nv, pos - 1, left - v, cur, out);
  }
  cur.e[pos] = 0;
}
}  // namespace detail

inline const MonoList& monos(int nv, int deg) {
  static std::mutex mu;
  static std::unordered_map<u64, MonoList> cache;
  std::lock_guard<std::mutex> lk(mu);
  u64 key = ((u64)nv << 32) | (u32)deg;
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  DRZG_REQUIRE(nv >= 1 && nv <= kMaxVars, "monos: unsupported variable count");
  MonoList L;
  L.nv = nv;
  L.deg = deg;
  if (deg >= 0) {
    Expo cur(nv);
    L.mons.reserve((size_t)mono_count(nv, deg));
    detail::gen_rev(nv, nv - 1, deg, cur, L.mons);
  }
  return cache.emplace(key, std::move(L)).first->second;
}

}  // namespace drzg
