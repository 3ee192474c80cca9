// Frobenius-matrix / zeta output: division-free characteristic polynomial,
// coefficient recovery in the Weil window, Newton polygon and invariants,
// point counts.  O(b^3) bignum work on b <= 52; restates reference
// linalg.hpp:646-681 (Berkowitz), zeta.hpp:152-371 (recover_Q, newton_polygon,
// hodge_polygon_at, classify, fedder_is_fsplit, counts_from_zeta) and
// oracle.hpp:190-245 (brute-force point count, used for the sign tie-break
// and the r = 1, 2 count checks).
#pragma once

#include <numeric>
#include <string>
#include <vector>

#include "cohom.hpp"

namespace drzg {

// d_0..d_n of det(lambda I - A) mod `mod` (Berkowitz, division free)
inline std::vector<Z> berkowitz(const std::vector<Z>& A, int n, const Z& mod) {
  auto red = [&](const Z& x) { return x.mod(mod); };
  std::vector<Z> V{Z(1)};
  for (int r = 1; r <= n; ++r) {
    std::vector<Z> s(r + 1, Z(0));
    s[0] = Z(1);
    s[1] = red(-A[(size_t)(r - 1) * n + (r - 1)]);
    std::vector<Z> t(r - 1);
    for (int i = 0; i < r - 1; ++i) t[i] = A[(size_t)i * n + (r - 1)];
    for (int j = 2; j <= r; ++j) {
      Z dot(0);
      for (int i = 0; i < r - 1; ++i) dot += A[(size_t)(r - 1) * n + i] * t[i];
      s[j] = red(-dot);
      if (j == r) break;
      std::vector<Z> t2(r - 1);
      for (int i = 0; i < r - 1; ++i) {
        Z acc(0);
        for (int l = 0; l < r - 1; ++l) acc += A[(size_t)i * n + l] * t[l];
        t2[i] = red(acc);
      }
      t.swap(t2);
    }
    std::vector<Z> W(r + 1, Z(0));
    for (int i = 0; i <= r; ++i) {
      Z acc(0);
      for (int j = 0; j <= i; ++j)
        if (i - j < (int)V.size()) acc += s[j] * V[i - j];
      W[i] = red(acc);
    }
    V.swap(W);
  }
  return V;
}

struct Recovered {
  int status = 2;  // 0 ok, 1 ambiguous, 2 escalate
  std::string reason;
  std::vector<std::vector<Z>> candidates;
};

inline Recovered recover_Q(const std::vector<Z>& dres, const PrecisionPlan& plan) {
  const u64 p = plan.p;
  const int n = plan.n;
  const i64 b = plan.b;
  const auto& H = plan.H;
  Recovered out;
  i64 top = (b + 1) / 2;
  std::vector<Z> a((size_t)b + 1, Z(0));
  a[0] = Z(1);
  for (i64 i = 1; i <= top; ++i) {
    int Ti = plan.A_sharp + (int)H[i];
    Z mod_i = Z::pow(p, Ti), ph = Z::pow(p, (u64)H[i]);
    Z di = dres[i].mod(mod_i);
    if (!di.divisible_by(ph)) {
      out.reason = "charpoly coefficient below its Hodge valuation";
      return out;
    }
    Z att = di.divexact(ph).centered(Z::pow(p, (u64)(Ti - H[i])));
    Z bound = Z::binom(b, i);
    if (att * att * ph * ph > bound * bound * Z::pow(p, (u64)(i * (n - 1)))) {
      out.reason = "coefficient outside the Weil window";
      return out;
    }
    a[i] = att * ph;
  }
  std::vector<int> signs = (n % 2 == 0) ? std::vector<int>{1} : std::vector<int>{1, -1};
  auto upper_digits = [&](i64 i) {
    i64 u = plan.A_sharp + H[i] + 1 - n;
    u = std::min<i64>(u, plan.M + n);
    return std::max<i64>(u, 0);
  };
  Z big_mod = Z::pow(p, (u64)(plan.M + n));
  for (int eps : signs) {
    std::vector<Z> cand = a;
    bool ok = true;
    for (i64 i = top + 1; i <= b; ++i) {
      i64 jj = b - i, e = (i64)(n - 1) * (b - 2 * jj) / 2;
      cand[i] = Z(eps) * Z::pow(p, (u64)e) * a[jj];
    }
    if (b % 2 == 1) {
      i64 jj = b - top, e = (i64)(n - 1) * (b - 2 * jj) / 2;
      if (cand[top] != Z(eps) * Z::pow(p, (u64)e) * a[jj]) ok = false;
    }
    if (ok && b % 2 == 0 && eps == -1 && !a[b / 2].is_zero()) ok = false;
    for (i64 i = top + 1; i <= b && ok; ++i) {
      i64 u = upper_digits(i);
      if (u == 0) continue;
      Z pu = Z::pow(p, (u64)u);
      if (!(cand[i] - dres[i].mod(big_mod)).mod(pu).is_zero()) ok = false;
    }
    if (ok) out.candidates.push_back(std::move(cand));
  }
  if (out.candidates.empty()) {
    out.reason = "no sign choice matches the residues";
    return out;
  }
  out.status = out.candidates.size() == 1 ? 0 : 1;
  return out;
}

// small exact rationals for the Newton polygon (valuations stay tiny)
struct Q64 {
  i64 num = 0, den = 1;
  static Q64 make(i64 a, i64 b) {
    if (b < 0) a = -a, b = -b;
    i64 g = std::gcd(a < 0 ? -a : a, b);
    if (g == 0) g = 1;
    return {a / g, b / g};
  }
  friend Q64 operator+(Q64 x, Q64 y) { return make(x.num * y.den + y.num * x.den, x.den * y.den); }
  friend Q64 operator-(Q64 x, Q64 y) { return make(x.num * y.den - y.num * x.den, x.den * y.den); }
  friend Q64 operator*(Q64 x, Q64 y) { return make(x.num * y.num, x.den * y.den); }
  friend bool operator<(Q64 x, Q64 y) { return (__int128)x.num * y.den < (__int128)y.num * x.den; }
  friend bool operator==(Q64 x, Q64 y) { return x.num == y.num && x.den == y.den; }
  std::string str() const { return den == 1 ? std::to_string(num) : std::to_string(num) + "/" + std::to_string(den); }
};

struct NewtonPolygon {
  std::vector<std::pair<i64, i64>> vertices;
  std::vector<std::pair<Q64, i64>> slopes;
  Q64 value_at(i64 x) const {
    for (size_t s = 0; s + 1 < vertices.size(); ++s) {
      auto [x1, y1] = vertices[s];
      auto [x2, y2] = vertices[s + 1];
      if (x < x1 || x > x2) continue;
      return Q64::make(y1, 1) + Q64::make(y2 - y1, x2 - x1) * Q64::make(x - x1, 1);
    }
    DRZG_REQUIRE(false, "NewtonPolygon: abscissa outside range");
    return {};
  }
};

inline NewtonPolygon newton_polygon(const std::vector<Z>& a, u64 p) {
  std::vector<std::pair<i64, i64>> pts;
  for (i64 i = 0; i < (i64)a.size(); ++i)
    if (!a[i].is_zero()) pts.emplace_back(i, a[i].valuation(p, 1 << 20));
  DRZG_REQUIRE(pts.size() >= 2, "newton_polygon: degenerate input");
  NewtonPolygon np;
  auto cross = [](std::pair<i64, i64> o, std::pair<i64, i64> q, std::pair<i64, i64> r) {
    return (q.first - o.first) * (r.second - o.second) - (q.second - o.second) * (r.first - o.first);
  };
  for (auto& pt : pts) {
    auto& v = np.vertices;
    while (v.size() >= 2 && cross(v[v.size() - 2], v.back(), pt) <= 0) v.pop_back();
    v.push_back(pt);
  }
  for (size_t s = 0; s + 1 < np.vertices.size(); ++s) {
    auto [x1, y1] = np.vertices[s];
    auto [x2, y2] = np.vertices[s + 1];
    np.slopes.emplace_back(Q64::make(y2 - y1, x2 - x1), x2 - x1);
  }
  return np;
}

// Hodge polygon at integer x: slope m-1 with multiplicity h_m (SPEC.md:327,
// 878).  Deliberate deviation: the reference (zeta.hpp:275-284) stops at the
// first empty slot (`take <= 0` also when h_m == 0), so for h_1 = 0 (cubic
// threefolds and fourfolds) its polygon is identically 0, the Newton >= Hodge
// check with equal endpoints always fails and run_zeta escalates until it
// throws.  Empty slots are skipped here; nonempty ones behave identically.
inline i64 hodge_polygon_at(const std::vector<i64>& h, int n, i64 x) {
  i64 acc = 0, used = 0;
  for (int m = 1; m <= n; ++m) {
    if (h[m] == 0) continue;
    i64 take = std::min<i64>(h[m], x - used);
    if (take <= 0) break;
    acc += take * (m - 1);
    used += take;
  }
  return acc;
}

struct Invariants {
  i64 p_rank = 0;
  std::string height, domino, newton_height;
  bool fsplit_defined = false, fsplit = false;
};

inline Invariants classify(const NewtonPolygon& np, const std::vector<i64>& h, int n, int d) {
  Invariants inv;
  Q64 s1 = np.slopes.front().first;
  if (s1.num == 0) inv.p_rank = np.slopes.front().second;
  if (n == 3 && d == 4) {
    inv.height = (s1 == Q64::make(1, 1)) ? "inf" : Q64::make((Q64::make(1, 1) - s1).den, (Q64::make(1, 1) - s1).num).str();
    bool first = true;
    Q64 gmin;
    for (i64 x = h[1]; x <= h[1] + h[2]; ++x) {
      Q64 gap = np.value_at(x) - Q64::make(hodge_polygon_at(h, n, x), 1);
      if (first || gap < gmin) gmin = gap, first = false;
    }
    inv.domino = gmin.str();
  }
  if (n == 5 && d == 3) {
    Q64 two = Q64::make(2, 1);
    inv.newton_height = (s1 == two) ? "inf" : Q64::make((two - s1).den, (two - s1).num).str();
  }
  return inv;
}

// domino number from the Newton polygon for any surface: min over the
// slope-1 Hodge range of NP - HP (the K3 rule of zeta.hpp:313-322, applied
// to the quintic surface as SURVEY 8(d) prescribes)
inline std::string domino_number(const NewtonPolygon& np, const std::vector<i64>& h, int n) {
  if (n != 3) return "";
  bool first = true;
  Q64 gmin;
  for (i64 x = h[1]; x <= h[1] + h[2]; ++x) {
    Q64 gap = np.value_at(x) - Q64::make(hodge_polygon_at(h, n, x), 1);
    if (first || gap < gmin) gmin = gap, first = false;
  }
  return gmin.str();
}

inline Z counts_from_zeta(const std::vector<Z>& a, u64 p, int n, int r) {
  i64 b = (i64)a.size() - 1;
  std::vector<Z> e((size_t)b + 1), s((size_t)r + 1, Z(0));
  for (i64 i = 0; i <= b; ++i) e[i] = (i % 2 == 0) ? a[i] : -a[i];
  for (int k = 1; k <= r; ++k) {
    Z acc(0);
    for (int i = 1; i < k; ++i)
      if (i <= b) acc += Z((i % 2) ? 1 : -1) * e[i] * s[k - i];
    if (k <= b) acc += Z((k % 2) ? (long)k : -(long)k) * e[k];
    s[k] = acc;
  }
  Z total(0);
  for (int i = 0; i < n; ++i) total += Z::pow(p, (u64)(i * r));
  total += ((n + 1) % 2 == 0) ? s[r] : -s[r];
  return total;
}

// --- brute-force point count over F_{p^r} (oracle.hpp:190-245) --------------
struct ExtField {
  u64 p = 0, q = 0;
  int r = 0;
  std::vector<u32> mul;  // q x q
  static ExtField make(u64 p, int r) {
    ExtField F;
    F.p = p;
    F.r = r;
    F.q = ipow(p, r);
    DRZG_REQUIRE(F.q <= 4096, "ExtField: field too large for a table");
    // monic irreducible of degree r: no root-free factorisation test needed
    // for r <= 3 (irreducible <=> no roots); r >= 4 searched by brute force
    std::vector<u64> mod(r + 1, 0);
    auto eval_mul = [&](const std::vector<u64>& m, u64 x, u64 y) {
      // multiply elements x, y (base-p digit vectors) modulo monic m
      std::vector<u64> a(r), b(r), c(2 * r, 0);
      for (int i = 0; i < r; ++i) a[i] = x % p, x /= p;
      for (int i = 0; i < r; ++i) b[i] = y % p, y /= p;
      for (int i = 0; i < r; ++i)
        for (int j = 0; j < r; ++j) c[i + j] = (c[i + j] + a[i] * b[j]) % p;
      for (int k = 2 * r - 1; k >= r; --k) {
        u64 lead = c[k];
        if (!lead) continue;
        for (int i = 0; i <= r; ++i) c[k - r + i] = (c[k - r + i] + (p - m[i] % p) % p * lead) % p;
      }
      u64 out = 0;
      for (int i = r - 1; i >= 0; --i) out = out * p + c[i];
      return out;
    };
    for (u64 code = 0;; ++code) {
      u64 t = code;
      for (int i = 0; i < r; ++i) mod[i] = t % p, t /= p;
      mod[r] = 1;
      if (t) DRZG_REQUIRE(false, "ExtField: no irreducible found");
      if (r == 1) break;
      // irreducible <=> the multiplicative group generated has no zero divisors:
      // check every nonzero element has an inverse (q small)
      bool ok = true;
      for (u64 x = 1; x < F.q && ok; ++x) {
        bool inv = false;
        for (u64 y = 1; y < F.q && !inv; ++y) inv = eval_mul(mod, x, y) == 1;
        ok = inv;
      }
      if (ok) break;
    }
    F.mul.assign(F.q * F.q, 0);
    for (u64 x = 0; x < F.q; ++x)
      for (u64 y = 0; y < F.q; ++y) F.mul[x * F.q + y] = (u32)(r == 1 ? x * y % p : eval_mul(mod, x, y));
    return F;
  }
  u64 add(u64 x, u64 y) const {
    u64 out = 0, pw = 1;
    for (int i = 0; i < r; ++i) {
      out += ((x % p + y % p) % p) * pw;
      x /= p, y /= p, pw *= p;
    }
    return out;
  }
};

inline i64 count_points(const Hypersurface& X, int r, i64 budget) {
  ExtField F = ExtField::make(X.p, r);
  const u64 q = F.q;
  const int nv = X.nv(), n = X.n;
  Z work(0);
  for (int m = 0; m <= n; ++m) work += Z::pow(q, (u64)m);
  DRZG_REQUIRE(work <= Z((long)budget), "count_points: budget exceeded");
  std::vector<u32> addt(q * q);
  for (u64 x = 0; x < q; ++x)
    for (u64 y = 0; y < q; ++y) addt[x * q + y] = (u32)F.add(x, y);
  std::vector<std::vector<u32>> powt(q, std::vector<u32>(X.d + 1, 1));
  for (u64 v = 0; v < q; ++v)
    for (int e = 1; e <= X.d; ++e) powt[v][e] = F.mul[powt[v][e - 1] * q + v];
  auto terms = X.f.terms();
  i64 count = 0;
  std::vector<u64> x(nv, 0);
  for (int lead = 0; lead <= n; ++lead) {
    std::vector<std::pair<u32, Expo>> live;
    for (auto& t : terms) {
      bool dead = false;
      for (int i = 0; i < lead; ++i) dead |= t.e[i] != 0;
      u32 c = (u32)(t.c % X.p);
      if (!dead && c) live.emplace_back(c, t.e);
    }
    for (int i = 0; i < nv; ++i) x[i] = 0;
    x[lead] = 1;
    for (;;) {
      u64 acc = 0;
      for (auto& [c, e] : live) {
        u64 v = c;
        for (int i = lead + 1; i <= n && v; ++i)
          if (e[i]) v = F.mul[v * q + powt[x[i]][e[i]]];
        acc = addt[acc * q + v];
      }
      if (acc == 0) ++count;
      int pos = n;
      while (pos > lead && x[pos] == q - 1) x[pos--] = 0;
      if (pos == lead) break;
      ++x[pos];
    }
  }
  return count;
}

inline bool fedder_is_fsplit(const Hypersurface& X) {
  if ((i64)X.d > (i64)X.nv()) return false;
  u128 pm = X.p;
  HPoly pw = X.f;
  for (auto& c : pw.c) c %= pm;
  HPoly fr = pw;
  // a term with an exponent above p - 1 never comes back into the box (the
  // products only raise exponents): pruning them keeps the powers small
  auto prune = [&](HPoly& h) {
    const auto& tab = h.table();
    for (int i = 0; i < h.size(); ++i) {
      if (!h.c[i]) continue;
      for (int v = 0; v < X.nv(); ++v)
        if (tab.mons[i][v] > (int)X.p - 1) {
          h.c[i] = 0;
          break;
        }
    }
  };
  prune(pw);
  for (u64 t = 2; t <= X.p - 1; ++t) {
    pw = poly_mul_small(pw, fr, pm);
    prune(pw);
  }
  for (const auto& t : pw.terms()) {
    bool small = true;
    for (int i = 0; i < X.nv(); ++i)
      if (t.e[i] > (int)X.p - 1) small = false;
    if (small && t.c % pm) return true;
  }
  return false;
}

}  // namespace drzg
