// Frobenius expansion of one basis column into compact seeds.
//
// Follows reference frobenius.hpp:121-144 (terms: exponent p(beta+alpha+1)-1,
// pole p(m+j), scalar D_{j,m} C_{j,alpha} mod p^{s_m}), zeta.hpp:56-69 (kappa_P
// prescale) and reduction.hpp:538-563 (seed: u = tweak(E+1, dn-n) made
// S-honest, one-hot vector at rank(E+1-u) carrying dc * kappa_P mod p^M).
// Seeds stay compact (exponent, one index, Ld digits) until the sweep that
// activates their pole materialises them on the device.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "tables.hpp"

namespace drzg {

// residue arithmetic mod p^M on the host: u128 while p^M < 2^80, else GMP
struct HostMod {
  u64 p = 0;
  int M = 0;
  bool wide = false;  // true -> GMP
  u128 m128 = 0;
  Z mz;
  static HostMod make(u64 p, int M) {
    HostMod h;
    h.p = p;
    h.M = M;
    h.mz = Z::pow(p, (u64)M);
    h.wide = h.mz >= (Z(1) << 80);
    if (!h.wide) h.m128 = h.mz.to_u128();
    return h;
  }
};

// balanced base-q digits of a residue (least significant first); the carry
// out of the top digit is a multiple of q^Ld, which p^M divides
inline void to_digits_u128(u128 v, const DigitPlan& dp, i8* out) {
  // v < 2^127 non-negative
  for (int t = 0; t < dp.Ld; ++t) {
    int r = (int)(v % (u128)dp.q);
    if (r > dp.q / 2) r -= dp.q;
    out[t] = (i8)r;
    v = (v - (u128)(i128)r) / (u128)dp.q;  // exact; r may be negative
  }
}
// the same for v < q^Ld when q^Ld <= 2^127: one 128-bit division splits v
// into base-q^c halves that fit 64 bits, then 64-bit digit extraction
// (the seed expansion converts millions of residues per column)
struct DigitSplitter {
  int q = 0, Ld = 0, c = 0;  // q^c < 2^63
  u64 qc = 1;
  static DigitSplitter make(const DigitPlan& dp) {
    DigitSplitter d;
    d.q = dp.q;
    d.Ld = dp.Ld;
    while (d.c < dp.Ld && d.qc <= (u64(1) << 62) / (u64)dp.q) d.qc *= (u64)dp.q, ++d.c;
    return d;
  }
  void digits(u128 v, i8* out) const {
    u64 lo, hi;
    if (c >= Ld) {
      lo = (u64)v;
      hi = 0;
    } else {
      lo = (u64)(v % qc);
      hi = (u64)(v / qc);  // < q^(Ld - c) < 2^64 when Ld - c <= c
    }
    int carry = 0;
    const int h = q / 2;
    for (int t = 0; t < Ld; ++t) {
      u64& src = t < c ? lo : hi;
      const int r0 = (int)(src % (u64)q);
      src /= (u64)q;
      int r = r0 + carry;
      carry = 0;
      if (r > h) r -= q, carry = 1;
      out[t] = (i8)r;
    }
  }
};

inline void to_digits_z(const Z& v0, const DigitPlan& dp, i8* out) {
  Z v = v0, q((long)dp.q);
  for (int t = 0; t < dp.Ld; ++t) {
    Z r = v.mod(q);
    long ri = r.to_long();
    if (ri > dp.q / 2) ri -= dp.q;
    out[t] = (i8)ri;
    v = (v - Z(ri)).divexact(q);
  }
}
// sum_t q^t s_t mod p^M for arbitrary (int64) digit sums
inline Z from_digit_sums(const i64* s, const DigitPlan& dp, const Z& mod) {
  Z acc(0), q((long)dp.q);
  for (int t = dp.Ld - 1; t >= 0; --t) acc = acc * q + Z((long)s[t]);
  return acc.mod(mod);
}

struct SeedBucket {
  std::vector<i32> u;     // nv per seed
  std::vector<i32> g;     // side index of the one-hot entry
  std::vector<i8> dig;    // Ld per seed
  size_t size() const { return g.size(); }
};

struct ColumnSeeds {
  int col = 0, m = 0;
  i64 Pmax = 0;
  i64 nterms = 0;
  std::map<int, SeedBucket> by_pole;  // pole -> seeds
};

// f^0..f^{N-1} mod p^s, cached per (N, s) for one hypersurface.  prime()
// computes the chain once at the largest (N, s) the run needs (the products
// split over threads); every other (N, s) is then that chain's prefix reduced
// mod p^s, one pass over the coefficients instead of a chain of products
struct PowerCache {
  std::mutex mu;
  std::map<std::pair<int, int>, std::vector<HPoly>> cache;
  std::pair<int, int> base{0, 0};
  static std::vector<HPoly> chain(const Hypersurface& X, int N, int s, int threads) {
    Z smod = Z::pow(X.p, (u64)s);
    DRZG_REQUIRE(smod < (Z(1) << 96), "power series modulus above 2^96");
    u128 m = smod.to_u128();
    std::vector<HPoly> out;
    HPoly one(X.nv(), 0);
    one.c[0] = 1;
    out.push_back(one);
    HPoly fr = X.f;
    for (auto& c : fr.c) c %= m;
    std::unique_ptr<ForkJoin> pool;
    if (threads > 1) pool = std::make_unique<ForkJoin>(threads);
    for (int j = 1; j < N; ++j) out.push_back(poly_mul_small_par(out.back(), fr, m, threads, pool.get()));
    return out;
  }
  void prime(const Hypersurface& X, int N, int s, int threads) {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(N, s);
    if (cache.find(key) == cache.end()) cache.emplace(key, chain(X, N, s, threads));
    base = key;
  }
  const std::vector<HPoly>& get(const Hypersurface& X, int N, int s, int threads = 1) {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(N, s);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (base.first >= N && base.second >= s) {
      // p^s divides p^{s_base}: reduce the primed chain's prefix
      const u128 m = Z::pow(X.p, (u64)s).to_u128();
      const auto& b = cache.at(base);
      std::vector<HPoly> out(b.begin(), b.begin() + N);
      for (auto& h : out)
        for (auto& c : h.c) c %= m;
      return cache.emplace(key, std::move(out)).first->second;
    }
    return cache.emplace(key, chain(X, N, s, threads)).first->second;
  }
};

// the seeds of column `col` from the powers f^j, j in [j0, j1) (a column's
// powers land in distinct poles p(m + j), so parts merge by moving buckets)
inline ColumnSeeds expand_column(const Hypersurface& X, const Basis& B, const PrecisionPlan& plan,
                                 const RuvTables& T, const HostMod& hm, PowerCache& pc, int col, int threads = 1,
                                 int j0 = 0, int j1 = 1 << 30) {
  ColumnSeeds out;
  out.col = col;
  int m = B.pole_of[col];
  out.m = m;
  const u64 p = X.p;
  const int nv = X.nv();
  int N = plan.N_m[m], s = plan.s_m[m];
  Z smodz = Z::pow(p, (u64)s);
  u128 smod = smodz.to_u128();
  out.Pmax = plan.max_pole(m);
  // D_{j,m} = (-1)^j sum_{i=j}^{N-1} C(m+i-1, i) C(i, j) mod p^s (modarith.hpp:143-182)
  std::vector<u128> Dj(N);
  for (int j = 0; j < N; ++j) {
    Z acc(0);
    for (int i = j; i < N; ++i) acc += Z::binom(m + i - 1, i) * Z::binom(i, j);
    if (j & 1) acc = -acc;
    Dj[j] = acc.mod(smodz).to_u128();
  }
  // kappa_P = prod_{t=P}^{Pmax-1} t mod p^M at poles P = p*k, k >= m (zeta.hpp:56-64)
  std::map<int, Z> kappa;
  kappa[(int)out.Pmax] = Z(1);
  {
    Z cur(1);
    for (i64 t = out.Pmax - 1; t >= (i64)p * m; --t) {
      cur = (cur * Z((long)t)).mod(hm.mz);
      if (t % (i64)p == 0 && t / (i64)p >= m) kappa[(int)t] = cur;
    }
  }
  const auto& powers = pc.get(X, N, s, threads);
  const Expo one = Expo::ones(nv);
  const Expo& beta = B.mons[col];
  const DigitPlan& dp = T.dp;
  const DigitSplitter split = DigitSplitter::make(dp);
  const bool small_s = (smod >> 63) == 0;  // D_j, C_{j,alpha} < p^s: their product fits 128 bits
  // v < p^M <= q^Ld; the 64-bit split covers q^Ld < 2^126 (Ld - c <= c)
  const bool fast_digits = !hm.wide && 2 * split.c >= dp.Ld;
  for (int j = 0; j < N; ++j) {
    if (Dj[j] == 0 || j < j0 || j >= j1) continue;
    int P = (int)p * (m + j);
    const Z& kap = kappa.at(P);
    u128 kap128 = hm.wide ? 0 : kap.to_u128();
    // wide moduli (p^M >= 2^80, e.g. the quintic surface's 7^49): kappa's
    // base-q digits once per pole; a seed's digits are then those of dc *
    // kappa mod q^Ld by one schoolbook pass (q^Ld is a multiple of p^M, so
    // this is the same residue mod p^M as the reference's dc * kappa mod p^M)
    std::vector<u64> kapd;
    if (hm.wide) {
      Z v = kap.mod(hm.mz), qz((long)dp.q);
      for (int t = 0; t < dp.Ld; ++t) {
        Z r = v.mod(qz);
        kapd.push_back((u64)r.to_long());
        v = (v - r).divexact(qz);
      }
    }
    SeedBucket& bk = out.by_pole[P];
    const HPoly& fj = powers[j];
    const auto& tab = fj.table();
    // seeds of monomials [a0, a1) of f^j, appended to `dst` in order
    auto expand = [&](int a0, int a1, SeedBucket& dst, i64& nterms) {
      for (int a = a0; a < a1; ++a) {
        if (!fj.c[a]) continue;
        u128 dc = small_s ? (Dj[j] * fj.c[a]) % smod : mulm128(Dj[j], fj.c[a], smod);
        if (dc == 0) continue;
        ++nterms;
        Expo full = beta + tab.mons[a] + one;
        for (int i = 0; i < nv; ++i) full[i] *= (int)p;  // E + 1
        Expo u;
        DRZG_REQUIRE(seed_u(full, T.D, T.S, &u), "seed: cannot honor the working set");
        Expo wm = full - u;
        DRZG_REQUIRE(wm.nonneg() && wm.total() == T.D, "seed: bad split");
        for (int i = 0; i < nv; ++i) dst.u.push_back(u[i]);
        dst.g.push_back((i32)rank_of(wm));
        size_t off = dst.dig.size();
        dst.dig.resize(off + dp.Ld);
        if (fast_digits) {
          // dc < p^s and kappa < p^M < 2^80: the product fits 128 bits when
          // s bits + 80 < 128, one reduction
          const u128 v = (dc >> 47) == 0 ? (dc * kap128) % hm.m128 : mulm128(dc, kap128, hm.m128);
          split.digits(v, dst.dig.data() + off);
        } else if (!hm.wide) {
          to_digits_u128(mulm128(dc, kap128, hm.m128), dp, dst.dig.data() + off);
        } else if ((dc >> 119) == 0) {
          // balanced digits of (sum_t kapd[t] q^t) * dc mod q^Ld (kapd[t] < 2^8,
          // dc < 2^119: every partial product and carry fits 128 bits)
          const u128 d64 = dc;
          u128 carry = 0;
          int bc = 0;  // balancing borrow into the next digit
          const int h = dp.q / 2;
          for (int t = 0; t < dp.Ld; ++t) {
            const u128 acc = (u128)kapd[t] * d64 + carry;  // < 2^127 + 2^120
            int r = (int)(acc % (u128)dp.q) + bc;
            carry = acc / (u128)dp.q;
            bc = 0;
            if (r > h) r -= dp.q, bc = 1;
            dst.dig[off + t] = (i8)r;
          }
        } else {
          to_digits_z((Z::from_u128(dc) * kap).mod(hm.mz), dp, dst.dig.data() + off);
        }
      }
    };
    const int na = fj.size();
    const int nth = std::max(1, std::min(threads, na / 8192));
    if (nth == 1) {
      expand(0, na, bk, out.nterms);
      continue;
    }
    // the column's monomials split over `threads` workers, concatenated in
    // order (the first columns of a run are on the device's critical path)
    std::vector<SeedBucket> part(nth);
    std::vector<i64> cnt(nth, 0);
    std::vector<std::exception_ptr> err(nth);
    std::vector<std::thread> pool;
    for (int t = 1; t < nth; ++t)
      pool.emplace_back([&, t] {
        try {
          expand((int)((i64)na * t / nth), (int)((i64)na * (t + 1) / nth), part[t], cnt[t]);
        } catch (...) {
          err[t] = std::current_exception();
        }
      });
    try {
      expand(0, (int)((i64)na / nth), part[0], cnt[0]);
    } catch (...) {
      err[0] = std::current_exception();
    }
    for (auto& th : pool) th.join();
    for (auto& e : err)
      if (e) std::rethrow_exception(e);
    for (int t = 0; t < nth; ++t) {
      out.nterms += cnt[t];
      bk.u.insert(bk.u.end(), part[t].u.begin(), part[t].u.end());
      bk.g.insert(bk.g.end(), part[t].g.begin(), part[t].g.end());
      bk.dig.insert(bk.dig.end(), part[t].dig.begin(), part[t].dig.end());
    }
  }
  return out;
}

}  // namespace drzg
