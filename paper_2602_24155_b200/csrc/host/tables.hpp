// Shared-operator tables for one (f, S, p^M) reduction context.
//
// Reference path being replaced: RuvContext (reduction.hpp:150-242) builds a
// unit echelon of the S-weighted Jacobian solve matrix J (rows Homog_L,
// columns the generators (i, mu)), build_ruv (:253-297) turns the solution of
// every unit right-hand side into the n+2 dense matrices of R_{x,v}, and
// eval_to_linear + linrec_eval (:300-339, linalg.hpp:337-410) apply them.
//
// Facts used (each checked against the reference in tests/):
//  * every row of J is a pivot row (S-smooth input), so the echelon's
//    transform is U = Jp^{-1} with Jp[:, r] = J[:, pc(r)], pc the pivot
//    column picked for row r by the reference's first-unit rule;
//  * build_ruv sends solution coordinate (i, mu) to the single side row
//    rank(mu + x^S - [i in S] e_i) with weight x_i + mu_i (the A_i and the
//    constant-matrix contributions land on the same row), hence
//      R_{x,v} w = T_x( Jp^{-1} P_v w ),   P_v w [r] = w[mon_r - v + x^S];
//  * Jp has small exact integer entries and few nonzeros per row, so
//    Jp^{-1} b mod p^M is computed by p-adic (Dixon) lifting in base
//    q = p^e <= 255: one dense int8 product with C = Jp^{-1} mod q per base-q
//    digit plus a sparse carry update with Jp.  No dense Z/p^M operator is
//    ever formed, and the pivot choice (which fixes the solution) is the
//    reference's, so results are bit-identical.
#pragma once

#include <set>
#include <vector>

#include "../kernels/setup.cuh"
#include "cohom.hpp"
#include "policy.hpp"

namespace drzg {

// digit system for residues mod p^M: balanced base q = p^e digits, int8
struct DigitPlan {
  u64 p = 0;
  int M = 0;
  int e = 1;      // q = p^e, the largest power with q <= 255
  int q = 0;
  int Ld = 0;     // digit planes, e * Ld >= M
  static DigitPlan make(u64 p, int M) {
    DigitPlan dp;
    dp.p = p;
    dp.M = M;
    u64 q = p;
    dp.e = 1;
    while (q * p <= 255) {
      q *= p;
      ++dp.e;
    }
    dp.q = (int)q;
    dp.Ld = (M + dp.e - 1) / dp.e;
    return dp;
  }
};

// a Dixon system: solve J x = b mod p^M for a square, invertible-mod-p
// integer matrix given sparsely (CSR) together with Cq = J^{-1} mod q
struct DixonSystem {
  int n = 0;                      // matrix order
  std::vector<i32> rowptr, col, val;  // CSR of J (exact small integers)
  std::vector<i8> Cq;             // n x n, balanced digits of J^{-1} mod q
};

// builds the Dixon system for the square submatrix of `dense` (rows x cols,
// exact small non-negative integers) on columns pc[0..rows)
inline DixonSystem make_dixon(const DigitPlan& dp, int rows, int cols, const std::vector<u32>& dense,
                              const std::vector<int>& pc) {
  DixonSystem sys;
  sys.n = rows;
  sys.rowptr.assign(rows + 1, 0);
  std::vector<u32> sq((size_t)rows * rows);
  for (int r = 0; r < rows; ++r) {
    for (int c = 0; c < rows; ++c) {
      u32 v = dense[(size_t)r * cols + pc[c]];
      sq[(size_t)r * rows + c] = v % (u32)dp.q;
      if (v) {
        sys.col.push_back(c);
        sys.val.push_back((i32)v);
      }
    }
    sys.rowptr[r + 1] = (i32)sys.col.size();
  }
  if (std::getenv("DRZG_DEBUG_NO_INVERSE")) return sys;  // structure-only debug dumps
  auto inv = use_device_setup(rows) ? inverse_mod_q_device(dp.p, (u64)dp.q, rows, sq)
                                    : inverse_mod_q(dp.p, (u64)dp.q, rows, std::move(sq));
  sys.Cq.resize(inv.size());
  for (size_t i = 0; i < inv.size(); ++i) {
    int v = (int)inv[i];
    if (v > dp.q / 2) v -= dp.q;
    sys.Cq[i] = (i8)v;
  }
  return sys;
}

struct RuvTables {
  u64 p = 0;
  int n = 0, d = 0, nv = 0;
  unsigned S = 0;   // bitmask
  Expo sexp;
  int D = 0;        // side degree dn - n
  int L = 0;        // solve degree d + D - |S|
  int side = 0;     // |Homog_D|
  int nL = 0;       // |Homog_L|
  DigitPlan dp;
  DixonSystem sys;  // Jp and Jp^{-1} mod q
  // per solution index r (= pivot row): generator (i, mu) of pc(r)
  std::vector<i32> sol_i, sol_mu, sol_row;
  // output side row g <- contributing solution indices (CSR)
  std::vector<i32> t_ptr, t_src;
  // per direction v (rank in Homog_d): gather table over Homog_L
  int ndir = 0;
  std::vector<i32> gidx;  // ndir x nL, rank in Homog_D or -1
  std::vector<i32> ginv;  // ndir x side: the L-row each side row feeds, or -1
};

inline RuvTables build_tables(const Hypersurface& X, int M, const std::set<int>& Sset) {
  RuvTables T;
  T.p = X.p;
  T.n = X.n;
  T.d = X.d;
  T.nv = X.nv();
  int nv = T.nv;
  for (int i : Sset) T.S |= 1u << i;
  T.sexp = Expo(nv);
  for (int i : Sset) T.sexp[i] = 1;
  T.D = X.d * X.n - X.n;
  int Ssz = (int)Sset.size();
  T.L = X.d + T.D - Ssz;
  T.side = (int)mono_count(nv, T.D);
  T.nL = (int)mono_count(nv, T.L);
  T.dp = DigitPlan::make(X.p, M);

  // generator columns, i ascending, mu grevlex (reduction.hpp:167-177)
  std::vector<int> mdeg(nv), goff(nv + 1);
  int cols = 0;
  for (int i = 0; i < nv; ++i) {
    mdeg[i] = T.D - Ssz + ((T.S >> i) & 1);
    goff[i] = cols;
    cols += (int)mono_count(nv, mdeg[i]);
  }
  goff[nv] = cols;
  // J (rows Homog_L) with exact small entries; reduction.hpp:224-238
  std::vector<u32> J((size_t)T.nL * cols, 0);
  for (int i = 0; i < nv; ++i) {
    HPoly gen = poly_partial(X.f, i);
    if (!((T.S >> i) & 1)) gen = poly_shift(gen, Expo::unit(nv, i));
    auto gt = gen.terms();
    const auto& mus = monos(nv, mdeg[i]).mons;
    for (int mi = 0; mi < (int)mus.size(); ++mi)
      for (const auto& t : gt) {
        DRZG_REQUIRE(t.c < (u128(1) << 24), "tables: generator coefficient too large");
        J[(size_t)rank_of(mus[mi] + t.e) * cols + goff[i] + mi] = (u32)t.c;
      }
  }
  std::vector<u32> Jp_mod_p(J.size());
  for (size_t k = 0; k < J.size(); ++k) Jp_mod_p[k] = (u32)(J[k] % X.p);
  PivotScan ps;
  if (use_device_setup(T.nL)) {
    ps.pivot_col_of_row = pivot_scan_device(X.p, T.nL, cols, Jp_mod_p);
    for (int pc : ps.pivot_col_of_row) ps.rank += pc >= 0;
  } else {
    ps = pivot_scan_fp(X.p, T.nL, cols, std::move(Jp_mod_p));
  }
  DRZG_REQUIRE(ps.rank == T.nL, "RuvContext: solve failed; input not S-smooth enough");
  T.sys = make_dixon(T.dp, T.nL, cols, J, ps.pivot_col_of_row);

  // decode each pivot column into (i, mu); reduction.hpp:264-285
  T.sol_i.resize(T.nL);
  T.sol_mu.resize(T.nL);
  T.sol_row.resize(T.nL);
  std::vector<std::vector<int>> by_row(T.side);
  for (int r = 0; r < T.nL; ++r) {
    int c = ps.pivot_col_of_row[r];
    int i = 0;
    while (c >= goff[i + 1]) ++i;
    const Expo& mu = monos(nv, mdeg[i]).mons[c - goff[i]];
    Expo sh = T.sexp;
    if ((T.S >> i) & 1) sh[i] -= 1;
    Expo tgt = mu + sh;
    T.sol_i[r] = i;
    T.sol_mu[r] = mu[i];
    T.sol_row[r] = (i32)rank_of(tgt);
    by_row[T.sol_row[r]].push_back(r);
  }
  T.t_ptr.assign(T.side + 1, 0);
  for (int g = 0; g < T.side; ++g) {
    for (int r : by_row[g]) T.t_src.push_back(r);
    T.t_ptr[g + 1] = (i32)T.t_src.size();
  }
  // gather tables: P_v w [r] = w[mon_r - v + x^S]
  const auto& dirs = monos(nv, X.d).mons;
  const auto& Lm = monos(nv, T.L).mons;
  T.ndir = (int)dirs.size();
  T.gidx.assign((size_t)T.ndir * T.nL, -1);
  for (int vi = 0; vi < T.ndir; ++vi)
    for (int r = 0; r < T.nL; ++r) {
      Expo g = Lm[r] - dirs[vi] + T.sexp;
      if (g.nonneg()) T.gidx[(size_t)vi * T.nL + r] = (i32)rank_of(g);
    }
  T.ginv.assign((size_t)T.ndir * T.side, -1);
  for (int vi = 0; vi < T.ndir; ++vi)
    for (int r = 0; r < T.nL; ++r) {
      i32 g = T.gidx[(size_t)vi * T.nL + r];
      if (g >= 0) T.ginv[(size_t)vi * T.side + g] = r;
    }
  return T;
}

}  // namespace drzg
