// Pole-order <= n classes onto the cohomology basis (reference FinalReducer,
// cohomology.hpp:166-257).  Per level m the reference unit-echelons the
// matrix [Jacobian generators | basis monomials] (rows Homog_{dm-n-1}) over
// Z/p^M and reads the solution off its pivot columns.  As for the reduction
// operator, every row is a pivot row, so the solution is Jp^{-1} g on the
// reference's pivot columns (first-unit rule, found over F_p) and zero
// elsewhere; it is computed here by the same base-q Dixon lifting.
#pragma once

#include <map>
#include <vector>

#include "frob.hpp"

namespace drzg {

// host Dixon solve of J x = b mod q^Ld for one right-hand side given as
// balanced digits (Ld x n); returns solution digits (Ld x n)
inline void dixon_solve_host(const DixonSystem& sys, const DigitPlan& dp, const std::vector<i8>& bdig,
                             std::vector<i8>& ydig) {
  const int n = sys.n, Ld = dp.Ld, q = dp.q;
  ydig.assign((size_t)Ld * n, 0);
  std::vector<i64> c(n, 0), in(n);
  auto balmod = [q](i64 x) {
    i64 r = x % q;
    if (r < 0) r += q;
    if (r > q / 2) r -= q;
    return r;
  };
  for (int k = 0; k < Ld; ++k) {
    for (int r = 0; r < n; ++r) in[r] = balmod(bdig[(size_t)k * n + r] + c[r]);
    i8* y = ydig.data() + (size_t)k * n;
    for (int r = 0; r < n; ++r) {
      i64 acc = 0;
      const i8* crow = sys.Cq.data() + (size_t)r * n;
      for (int j = 0; j < n; ++j) acc += (i64)crow[j] * in[j];
      y[r] = (i8)balmod(acc);
    }
    for (int r = 0; r < n; ++r) {
      i64 s = 0;
      for (int e = sys.rowptr[r]; e < sys.rowptr[r + 1]; ++e) s += (i64)sys.val[e] * y[sys.col[e]];
      i64 num = bdig[(size_t)k * n + r] + c[r] - s;
      DRZG_REQUIRE(num % q == 0, "dixon: inexact carry");
      c[r] = num / q;
    }
  }
}

class FinalReducer {
 public:
  FinalReducer(const Hypersurface& X, const Basis& B, const DigitPlan& dp, const HostMod& hm)
      : X_(&X), B_(&B), dp_(dp), hm_(hm) {}

  // build every level up front; afterwards reduce() only reads shared state
  // and may run concurrently on many columns
  void prepare() {
    for (int m = 1; m <= X_->n; ++m) level(m);
  }

  // test access: pivot columns and inverse of level m
  const std::vector<int>& level_pivots(int m) const { return levels_.at(m).pc; }
  const std::vector<i8>& level_inverse(int m) const { return levels_.at(m).sys.Cq; }

  // g over monos(nv, dm-n-1) as residues mod p^M; returns the b-vector
  std::vector<Z> reduce(std::vector<Z> g, int m) const {
    DRZG_REQUIRE(m >= 1 && m <= X_->n, "FinalReducer: pole order out of range");
    std::vector<Z> out((size_t)B_->b, Z(0));
    for (; m >= 1; --m) {
      const Level& L = levels_.at(m);
      DRZG_REQUIRE((int)g.size() == L.rows, "FinalReducer: bad coeff size");
      std::vector<Z> sol(L.ncols, Z(0));
      if (L.rows > 0) {
        std::vector<i8> bd((size_t)dp_.Ld * L.rows), yd;
        std::vector<i8> tmp(dp_.Ld);
        for (int r = 0; r < L.rows; ++r) {
          to_digits_z(g[r].mod(hm_.mz), dp_, tmp.data());
          for (int t = 0; t < dp_.Ld; ++t) bd[(size_t)t * L.rows + r] = tmp[t];
        }
        dixon_solve_host(L.sys, dp_, bd, yd);
        std::vector<i64> s(dp_.Ld);
        for (int r = 0; r < L.rows; ++r) {
          for (int t = 0; t < dp_.Ld; ++t) s[t] = yd[(size_t)t * L.rows + r];
          sol[L.pc[r]] = from_digit_sums(s.data(), dp_, hm_.mz);
        }
      }
      int base = B_->slots_before(m);
      for (int s2 = 0; s2 < (int)B_->h[m]; ++s2) out[(size_t)base + s2] = sol[L.gen_count + s2];
      if (m == 1) break;
      const int nv = X_->nv();
      int knext = X_->d * (m - 1) - X_->n - 1;
      std::vector<Z> g2((size_t)mono_count(nv, knext), Z(0));
      Z inv_m1 = Z(m - 1).inverse_mod(hm_.mz);
      for (int c = 0; c < L.gen_count; ++c) {
        if (sol[c].is_zero()) continue;
        int i = L.gen_i[c];
        const Expo& mu = L.gen_mu[c];
        if (mu[i] == 0) continue;
        g2[(size_t)rank_of(mu - Expo::unit(nv, i))] += sol[c] * Z((long)mu[i]);
      }
      for (auto& v : g2) v = (v * inv_m1).mod(hm_.mz);
      g = std::move(g2);
    }
    return out;
  }

 private:
  struct Level {
    int rows = 0, ncols = 0, gen_count = 0;
    std::vector<int> pc;
    std::vector<int> gen_i;
    std::vector<Expo> gen_mu;
    DixonSystem sys;
  };

  Level& level(int m) {
    auto it = levels_.find(m);
    if (it != levels_.end()) return it->second;
    Level L;
    const int nv = X_->nv();
    int k = X_->d * m - X_->n - 1;
    L.rows = (int)mono_count(nv, k);
    int mu_deg = k - (X_->d - 1);
    const auto& mus = monos(nv, mu_deg).mons;
    L.gen_count = mu_deg < 0 ? 0 : nv * (int)mus.size();
    L.ncols = L.gen_count + (int)B_->h[m];
    if (L.rows > 0) {
      std::vector<u32> data((size_t)L.rows * L.ncols, 0);
      int col = 0;
      for (int i = 0; i < nv && mu_deg >= 0; ++i) {
        auto dt = poly_partial(X_->f, i).terms();
        for (const Expo& mu : mus) {
          for (const auto& t : dt) data[(size_t)rank_of(mu + t.e) * L.ncols + col] = (u32)t.c;
          L.gen_i.push_back(i);
          L.gen_mu.push_back(mu);
          ++col;
        }
      }
      int base = B_->slots_before(m);
      for (int s = 0; s < (int)B_->h[m]; ++s) data[(size_t)rank_of(B_->mons[base + s]) * L.ncols + col + s] = 1;
      std::vector<u32> modp(data.size());
      for (size_t e = 0; e < data.size(); ++e) modp[e] = data[e] % (u32)X_->p;
      PivotScan ps;
      if (use_device_setup(L.rows)) {
        ps.pivot_col_of_row = pivot_scan_device(X_->p, L.rows, L.ncols, modp);
        for (int pc : ps.pivot_col_of_row) ps.rank += pc >= 0;
      } else {
        ps = pivot_scan_fp(X_->p, L.rows, L.ncols, std::move(modp));
      }
      DRZG_REQUIRE(ps.rank == L.rows, "FinalReducer: class outside Jacobian + basis span");
      L.pc = ps.pivot_col_of_row;
      L.sys = make_dixon(dp_, L.rows, L.ncols, data, L.pc);
    }
    return levels_.emplace(m, std::move(L)).first->second;
  }

  const Hypersurface* X_;
  const Basis* B_;
  DigitPlan dp_;
  HostMod hm_;
  std::map<int, Level> levels_;
};

}  // namespace drzg
