// Hypersurface data, Hodge numbers, smoothness, the monomial cohomology basis
// and the p-adic precision plan — the setup the reduction engine consumes.
// Restates, for the drop-in host side, reference cohomology.hpp:16-160 and
// frobenius.hpp:11-106 (same formulas, same tie-breaks, same outputs).
#pragma once

#include <set>
#include <vector>

#include "bigint.hpp"
#include "elim.hpp"
#include "poly.hpp"

namespace drzg {

struct Hypersurface {
  u64 p = 0;
  int n = 0, d = 0;
  HPoly f;  // integer coefficients (>= 0, as given)
  int nv() const { return n + 1; }

  // cohomology.hpp:24-32
  static Hypersurface make(u64 p, int n, int d, const std::vector<u64>& coeffs) {
    DRZG_REQUIRE(n >= 2 && n + 1 <= kMaxVars, "Hypersurface: unsupported n");
    DRZG_REQUIRE(d >= 2, "Hypersurface: degree too small");
    DRZG_REQUIRE(p > (u64)n, "Hypersurface: need p > n");
    DRZG_REQUIRE((u64)d % p != 0, "Hypersurface: p | d not supported");
    Hypersurface X;
    X.p = p;
    X.n = n;
    X.d = d;
    X.f = HPoly(n + 1, d);
    DRZG_REQUIRE((int)coeffs.size() == X.f.size(), "Hypersurface: coefficient count");
    for (int i = 0; i < X.f.size(); ++i) {
      DRZG_REQUIRE(coeffs[i] < (u64(1) << 20), "Hypersurface: coefficients must lie in [0, 2^20)");
      X.f.c[i] = coeffs[i];
    }
    return X;
  }
};

// cohomology.hpp:37-53: h_m = dim of degree dm-n-1 in the Artinian quotient
inline i64 artinian_dim(int n, int d, int k) {
  if (k < 0) return 0;
  Z acc(0);
  for (int j = 0; j * (d - 1) <= k && j <= n + 1; ++j) {
    Z t = Z::binom(n + 1, j) * Z::binom(k - j * (d - 1) + n, n);
    acc = (j & 1) ? acc - t : acc + t;
  }
  return acc.to_long();
}
inline std::vector<i64> hodge_numbers(int n, int d) {
  std::vector<i64> h(n + 1, 0);
  for (int m = 1; m <= n; ++m) h[m] = artinian_dim(n, d, d * m - n - 1);
  return h;
}
inline std::vector<i64> hodge_heights(int n, int d) {
  auto h = hodge_numbers(n, d);
  std::vector<i64> H{0};
  for (int m = 1; m <= n; ++m)
    for (i64 c = 0; c < h[m]; ++c) H.push_back(H.back() + (m - 1));
  return H;
}

// rows (i, mu) of the degree-k Jacobian map over F_p, columns monos(nv, k)
// (cohomology.hpp:75-98); weighted: x_i d_i f for i outside S
inline std::vector<u32> jacobian_rows_fp(const Hypersurface& X, int k, const std::set<int>& S, bool weighted,
                                         int* nrows) {
  int nv = X.nv();
  i64 ncols = mono_count(nv, k);
  std::vector<u32> out;
  int rows = 0;
  for (int i = 0; i < nv; ++i) {
    HPoly gen = poly_partial(X.f, i);
    if (weighted && !S.count(i)) gen = poly_shift(gen, Expo::unit(nv, i));
    int mu_deg = k - gen.deg;
    if (mu_deg < 0 || gen.is_zero()) continue;
    auto gt = gen.terms();
    for (const Expo& mu : monos(nv, mu_deg).mons) {
      size_t base = out.size();
      out.resize(base + ncols, 0);
      for (const auto& t : gt) out[base + rank_of(mu + t.e)] = (u32)(t.c % X.p);
      ++rows;
    }
  }
  *nrows = rows;
  return out;
}

// cohomology.hpp:102-111
inline bool check_smooth(const Hypersurface& X, const std::set<int>& S) {
  int k = (X.n + 1) * X.d - X.n - (int)S.size();
  int rows = 0;
  auto m = jacobian_rows_fp(X, k, S, true, &rows);
  i64 need = mono_count(X.nv(), k);
  if (rows < need) return false;
  return pivot_scan_fp(X.p, rows, (int)need, std::move(m)).rank >= need;
}

inline std::set<int> full_set(int nv) {
  std::set<int> S;
  for (int i = 0; i < nv; ++i) S.insert(i);
  return S;
}

// reduction.hpp:35-41
inline std::set<int> default_S(int n, int d) {
  std::set<int> S;
  int nv = n + 1;
  for (int i = (d >= nv ? 0 : nv - d); i < nv; ++i) S.insert(i);
  return S;
}

struct Basis {
  std::vector<Expo> mons;
  std::vector<int> pole_of;
  std::vector<i64> h;
  i64 b = 0;
  int slots_before(int m) const {
    i64 s = 0;
    for (int t = 1; t < m; ++t) s += h[t];
    return (int)s;
  }
};

// cohomology.hpp:134-160: per pole m, the non-pivot columns of the mod-p
// Jacobian row space in degree dm-n-1
inline Basis compute_basis(const Hypersurface& X) {
  Basis B;
  B.h.assign(X.n + 1, 0);
  for (int m = 1; m <= X.n; ++m) {
    int k = X.d * m - X.n - 1;
    const MonoList& tgt = monos(X.nv(), k);
    int rows = 0;
    auto mat = jacobian_rows_fp(X, k, {}, false, &rows);
    std::vector<char> is_pivot(tgt.size(), 0);
    if (rows > 0) {
      auto ps = pivot_scan_fp(X.p, rows, tgt.size(), std::move(mat));
      for (int pc : ps.pivot_col_of_row)
        if (pc >= 0) is_pivot[pc] = 1;
    }
    for (int c = 0; c < tgt.size(); ++c)
      if (!is_pivot[c]) {
        B.mons.push_back(tgt.mons[c]);
        B.pole_of.push_back(m);
        ++B.h[m];
      }
  }
  for (int m = 1; m <= X.n; ++m) B.b += B.h[m];
  auto expect = hodge_numbers(X.n, X.d);
  for (int m = 1; m <= X.n; ++m)
    DRZG_REQUIRE(B.h[m] == expect[m], "compute_basis: cokernel dimension off the Hodge number");
  return B;
}

// --- precision plan (frobenius.hpp:11-106) -----------------------------------
struct PrecisionPlan {
  u64 p = 0;
  int n = 0, d = 0;
  i64 b = 0;
  std::vector<i64> h, H;
  int A_sharp = 1, A = 1;
  std::vector<int> r_m, N_m, s_m;
  int M = 0;
  int escalations = 0;
  i64 max_pole(int m) const { return (i64)p * s_m[m]; }
};

struct PlanOverrides {
  std::vector<int> N_m;
  int r_uniform = 0;
};

inline i64 factorial_valuation(u64 n, u64 p) {
  i64 v = 0;
  while (n) {
    n /= p;
    v += (i64)n;
  }
  return v;
}

namespace detail {
inline int weil_digits(u64 p, i64 b, int n, i64 i) {
  Z bound = Z(4) * Z::binom(b, i) * Z::binom(b, i) * Z::pow(p, (u64)(i * (n - 1)));
  int w = 1;
  while (Z::pow(p, 2 * w) <= bound) ++w;
  return w;
}
inline void refresh_precision(PrecisionPlan& P) {
  P.s_m.assign(P.n + 1, 0);
  i64 M = 0;
  for (int m = 1; m <= P.n; ++m) {
    P.s_m[m] = P.N_m[m] + m - 1;
    i64 v = factorial_valuation((u64)P.p * P.s_m[m] - 1, P.p);
    M = std::max<i64>(M, P.r_m[m] + v - m + 1);
  }
  P.M = (int)M;
}
}  // namespace detail

inline PrecisionPlan choose_precision(u64 p, int n, int d, const PlanOverrides& ov = {}) {
  PrecisionPlan P;
  P.p = p;
  P.n = n;
  P.d = d;
  P.h = hodge_numbers(n, d);
  P.H = hodge_heights(n, d);
  for (int m = 1; m <= n; ++m) P.b += P.h[m];
  i64 half = (P.b + 1) / 2;
  int sharp = 1;
  for (i64 i = 1; i <= half; ++i) sharp = std::max(sharp, detail::weil_digits(p, P.b, n, i) - (int)P.H[i]);
  P.A_sharp = sharp;
  P.A = sharp + (int)P.H[half];
  P.r_m.assign(n + 1, 0);
  P.N_m.assign(n + 1, 0);
  for (int m = 1; m <= n; ++m) {
    P.r_m[m] = ov.r_uniform > 0 ? ov.r_uniform : P.A_sharp;
    if (!ov.N_m.empty()) {
      P.N_m[m] = ov.N_m.size() == 1 ? ov.N_m[0] : ov.N_m.at(m - 1);
      P.r_m[m] = std::max(1, P.N_m[m] - n);
    } else {
      P.N_m[m] = P.r_m[m] + n;
    }
    DRZG_REQUIRE(P.N_m[m] >= 1, "choose_precision: empty series");
  }
  if (ov.r_uniform > 0) {
    P.A_sharp = ov.r_uniform;
    P.A = ov.r_uniform + (int)P.H[half];
  }
  detail::refresh_precision(P);
  return P;
}

inline bool escalate_plan(PrecisionPlan& P) {
  if (P.escalations >= 3) return false;
  ++P.escalations;
  for (int m = 1; m <= P.n; ++m) {
    P.N_m[m] += 2;
    if (P.escalations >= 2) P.r_m[m] += 2;
  }
  if (P.escalations >= 2) {
    P.A_sharp += 2;
    P.A += 2;
  }
  detail::refresh_precision(P);
  return true;
}

}  // namespace drzg
