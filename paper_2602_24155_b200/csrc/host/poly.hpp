// Dense homogeneous polynomials over Z/m, indexed by grevlex position.
// Host-side setup only (Jacobian generators, power series f^j for the
// Frobenius expansion, reference homog.hpp:21-142).
#pragma once

#include <algorithm>
#include <thread>
#include <vector>

#include "mono.hpp"

namespace drzg {

struct HPoly {
  int nv = 0, deg = 0;
  std::vector<u128> c;  // parallel to monos(nv, deg).mons

  HPoly() = default;
  HPoly(int nvars, int degree) : nv(nvars), deg(degree), c((size_t)mono_count(nvars, degree), 0) {}
  const MonoList& table() const { return monos(nv, deg); }
  int size() const { return (int)c.size(); }
  bool is_zero() const {
    for (auto x : c)
      if (x) return false;
    return true;
  }
  struct Term {
    u128 c;
    Expo e;
  };
  std::vector<Term> terms() const {
    std::vector<Term> out;
    const auto& t = table();
    for (int i = 0; i < size(); ++i)
      if (c[i]) out.push_back({c[i], t.mons[i]});
    return out;
  }
};

// product reduced mod m (m < 2^100 and the second factor's coefficients
// small enough that one row of partial products fits 128 bits)
inline HPoly poly_mul_small(const HPoly& a, const HPoly& f, u128 m) {
  HPoly r(a.nv, a.deg + f.deg);
  auto ft = f.terms();
  const auto& ta = a.table();
  // accumulate per target without reduction: |f terms| * m * max|f coeff| < 2^128
  std::vector<u128> acc(r.c.size(), 0);
  for (int i = 0; i < a.size(); ++i) {
    if (!a.c[i]) continue;
    for (const auto& t : ft) acc[(size_t)rank_of(ta.mons[i] + t.e)] += a.c[i] * t.c;
  }
  for (size_t i = 0; i < acc.size(); ++i) r.c[i] = acc[i] % m;
  return r;
}

// the same product on `threads` host threads: each accumulates a range of a's
// terms into its own targets, then the ranges' sums are reduced per target
// (a target still receives at most |f terms| products in total, so the bound
// above holds for the sum)
// pool != nullptr: the parts run on its persistent threads (a power chain
// multiplies ~N times; spawning threads per product cost more than the
// product for the small early powers), and smaller operands split
inline HPoly poly_mul_small_par(const HPoly& a, const HPoly& f, u128 m, int threads, ForkJoin* pool = nullptr) {
  const int nth = std::max(1, std::min(pool ? std::min(threads, pool->size()) : threads,
                                       a.size() / (pool ? 1024 : 4096)));
  if (nth == 1) return poly_mul_small(a, f, m);
  HPoly r(a.nv, a.deg + f.deg);
  auto ft = f.terms();
  const auto& ta = a.table();
  const size_t nr = r.c.size();
  std::vector<std::vector<u128>> acc(nth);
  auto run = [&](int t) {
    acc[t].assign(nr, 0);
    const int i0 = (int)((i64)a.size() * t / nth), i1 = (int)((i64)a.size() * (t + 1) / nth);
    for (int i = i0; i < i1; ++i) {
      if (!a.c[i]) continue;
      for (const auto& tm : ft) acc[t][(size_t)rank_of(ta.mons[i] + tm.e)] += a.c[i] * tm.c;
    }
  };
  auto reduce = [&](int t) {
    const size_t k0 = nr * t / nth, k1 = nr * (t + 1) / nth;
    for (size_t k = k0; k < k1; ++k) {
      u128 v = 0;
      for (int u = 0; u < nth; ++u) v += acc[u][k];
      r.c[k] = v % m;
    }
  };
  auto parallel = [&](auto& phase) {
    if (pool) {
      pool->run(nth, [&](int t) { phase(t); });
      return;
    }
    std::vector<std::thread> ths;
    for (int t = 1; t < nth; ++t) ths.emplace_back([&, t] { phase(t); });
    phase(0);
    for (auto& th : ths) th.join();
  };
  parallel(run);
  parallel(reduce);
  return r;
}

inline HPoly poly_partial(const HPoly& f, int i) {
  DRZG_REQUIRE(f.deg >= 1, "partial: constant input");
  HPoly r(f.nv, f.deg - 1);
  const auto& tf = f.table();
  for (int k = 0; k < f.size(); ++k) {
    if (!f.c[k] || tf.mons[k][i] == 0) continue;
    Expo e = tf.mons[k];
    int ei = e[i];
    e[i] -= 1;
    r.c[(size_t)rank_of(e)] += (u128)ei * f.c[k];
  }
  return r;
}

inline HPoly poly_shift(const HPoly& f, const Expo& s) {
  HPoly r(f.nv, f.deg + s.total());
  const auto& tf = f.table();
  for (int k = 0; k < f.size(); ++k)
    if (f.c[k]) r.c[(size_t)rank_of(tf.mons[k] + s)] = f.c[k];
  return r;
}

}  // namespace drzg
