// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include/drzeta/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libdrz_ref.so.  Used by tests/ (parity checks), by
// scripts/make_golden.py (fixtures under tests/golden/) and by bench.py's
// cpu_baseline / --impl reference leg.  Every function here only marshals
// plain arrays to and from the reference's own types and calls the
// reference's own functions:
//   linrec_eval            linalg.hpp:337-410
//   detail::sparse_steps   linalg.hpp:257-331  (SparseOp::build linalg.hpp:227)
//   StripePlan::make       linalg.hpp:35-58
//   reduce_chunk           reduction.hpp:394-423 (build_ruv :253-297)
//   frobenius_matrix       zeta.hpp:36-136
//   run_zeta               zeta.hpp:438-549
//   frobenius_terms / seed_reduction_input  frobenius.hpp:121-144, reduction.hpp:538-563
#include <drzeta/zeta.hpp>

#include <chrono>
#include <cstring>
#include <random>
#include <sstream>
#include <unordered_set>
#include <atomic>
#include <mutex>
#include <thread>

using namespace drz;

namespace {

char* dup_str(const std::string& s) {
  char* out = (char*)std::malloc(s.size() + 1);
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

std::string esc(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}

template <class F>
char* guarded(F&& f) {
  try {
    return dup_str(f());
  } catch (const std::exception& e) {
    return dup_str(std::string("{\"error\": \"") + esc(e.what()) + "\"}");
  }
}

Hypersurface make_x(u64 p, int n, int d, const u64* coeffs) {
  HomogPoly f(n + 1, d);
  for (int i = 0; i < f.size(); ++i) f.c[i] = (unsigned long)coeffs[i];
  return Hypersurface::make(p, n, d, f);
}

std::string zarr(const std::vector<mpz_class>& v) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << "\"" << v[i].get_str() << "\"";
  os << "]";
  return os.str();
}

template <class T>
std::string iarr(const std::vector<T>& v) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << v[i];
  os << "]";
  return os.str();
}

std::string expo_arr(const Expo& e) {
  std::ostringstream os;
  os << "[";
  for (int i = 0; i < e.nv; ++i) os << (i ? "," : "") << e[i];
  os << "]";
  return os.str();
}

std::string plan_json(const PrecisionPlan& P) {
  std::ostringstream os;
  os << "{\"M\":" << P.M << ",\"A\":" << P.A << ",\"A_sharp\":" << P.A_sharp
     << ",\"b\":" << P.b << ",\"escalations\":" << P.escalations
     << ",\"r_m\":" << iarr(P.r_m) << ",\"N_m\":" << iarr(P.N_m)
     << ",\"s_m\":" << iarr(P.s_m) << ",\"h\":" << iarr(P.h) << ",\"H\":" << iarr(P.H) << "}";
  return os.str();
}

PlanOverrides overrides(int r_uniform, int nm_override) {
  PlanOverrides ov;
  ov.r_uniform = r_uniform;
  if (nm_override > 0) ov.N_m = {nm_override};
  return ov;
}

ModMatrix mat_from(const StripePlan& pl, int side, const u64* planes) {
  ModMatrix A(pl, side, side);
  std::memcpy(A.d.data(), planes, sizeof(u64) * A.d.size());
  return A;
}

// trivial PepStoreBase over build_ruv, the same test double the reference's
// own suite uses (tests/test_reduction.cpp:33-50)
struct BuildStore : PepStoreBase {
  const RuvContext* C;
  PepStats st;
  explicit BuildStore(const RuvContext& c) : C(&c) {}
  std::shared_ptr<const PepEntry> get(const Expo& v) override {
    ++st.misses;
    return std::make_shared<const PepEntry>(build_ruv(*C, v));
  }
  PepStats stats() const override { return st; }
};

}  // namespace


// Value-free replay of frobenius_matrix's cost ledger (zeta.hpp:36-136 with
// run_policy p-chunk, reduction.hpp:464-533): the reference's move choice
// (choose_v_greedy, repair_v, k_max_legal, legal) is a function of (u, pole)
// alone, so the ledger of a hypersurface needs no matrices.  Seeds come from
// the reference's frobenius_terms; their exponent split restates
// seed_reduction_input (reduction.hpp:538-563) without materialising w (the
// random fourfold's seeds would be ~150 GB).  Bookkeeping per move is
// reduce_chunk's (reduction.hpp:419-422: matvecs += k, startups += 1), and
// states are merged by (u, pole) after every sweep (combine_states,
// reduction.hpp:426-451; the first sweep runs before any merge, as there).
// Used to pin the engine's ledger at plans the reference cannot run here.
namespace {
struct RKey {
  u64 u;
  int pole;
  bool operator==(const RKey& o) const { return u == o.u && pole == o.pole; }
};
struct RKeyHash {
  size_t operator()(const RKey& k) const { return std::hash<u64>()(k.u * 1315423911ull ^ (u64)k.pole); }
};
struct RState {
  Expo u;
  int pole;
};

CostLedger replay_column(const Hypersurface& X, const Basis& B, const PrecisionPlan& plan, const std::set<int>& S,
                         int j) {
  const int nv = X.nv(), n = X.n, d = X.d;
  const i64 p = (i64)X.p;
  const int D = d * n - n;
  CostLedger led;
  std::vector<RState> seeds;
  {
    auto terms = frobenius_terms(X, B.mons[j], B.pole_of[j], plan);
    seeds.reserve(terms.size());
    for (const auto& t : terms) {
      Expo full = t.exponent + Expo::ones(nv);
      Expo u = tweak(full, D);
      for (int i = 0; i < nv; ++i) {
        if (S.count(i) || u[i] >= 1) continue;
        int jj = -1;
        for (int c = 0; c < nv; ++c) {
          bool ok = S.count(c) ? u[c] >= 1 : u[c] >= 2;
          if (ok && (jj < 0 || u[c] > u[jj])) jj = c;
        }
        DRZ_REQUIRE(jj >= 0, "seed: cannot honor the working set");
        --u[jj];
        ++u[i];
      }
      Expo wmon = full - u;
      DRZ_REQUIRE(wmon.nonneg() && wmon.total() == D, "seed: bad split");
      seeds.push_back({u, t.pole});
    }
  }
  // active states bucketed by |u| (a sweep takes the top bucket), floor states apart
  std::map<int, std::vector<RState>, std::greater<int>> act;
  std::unordered_set<RKey, RKeyHash> floor;
  i64 total_states = (i64)seeds.size(), final_states = 0;
  auto move = [&](RState& st) {
    Expo v = choose_v_greedy(d, st.u, S);
    repair_v(st.u, v, S);
    i64 k = std::min(std::min(p, (i64)st.pole - n), k_max_legal(st.u, v, S));
    DRZ_REQUIRE(k >= 1, "p-chunk: no admissible move");
    DRZ_REQUIRE(legal(d, st.u, v, k, S), "reduce_chunk: illegal move");
    st.u = st.u - v.scaled((int)k);
    st.pole -= (int)k;
    led.matvecs += k;
    led.startups += 1;
  };
  auto place = [&](std::vector<RState>& moved) {
    for (auto& st : moved) {
      if (st.pole == n) {
        floor.insert({st.u.key(), st.pole});
        continue;
      }
      act[st.u.total()].push_back(st);
    }
  };
  // sweep 1: states at the top |u| move before any combine (duplicates move apart)
  {
    int top = -1;
    for (auto& s : seeds)
      if (s.pole > n) top = std::max(top, s.u.total());
    std::vector<RState> moved;
    for (auto& s : seeds) {
      if (s.pole > n && s.u.total() == top) move(s);
      moved.push_back(s);
    }
    seeds.clear();
    seeds.shrink_to_fit();
    place(moved);
  }
  // combine everything once (the first combine_states), then sweep by sweep
  for (auto& kv : act) {
    std::unordered_set<RKey, RKeyHash> seen;
    std::vector<RState> keep;
    for (auto& s : kv.second)
      if (seen.insert({s.u.key(), s.pole}).second) keep.push_back(s);
    kv.second.swap(keep);
  }
  while (!act.empty()) {
    auto it = act.begin();
    std::vector<RState> front = std::move(it->second);
    act.erase(it);
    // states landing on a bucket are merged against it at this sweep's combine
    std::map<int, std::unordered_set<RKey, RKeyHash>> seen;
    for (auto& s : front) move(s);
    for (auto& s : front) {
      if (s.pole == n) {
        floor.insert({s.u.key(), s.pole});
        continue;
      }
      auto& bucket = act[s.u.total()];
      auto& sn = seen[s.u.total()];
      if (sn.empty())
        for (auto& o : bucket) sn.insert({o.u.key(), o.pole});
      if (sn.insert({s.u.key(), s.pole}).second) bucket.push_back(s);
    }
  }
  for (auto& kv : act) final_states += (i64)kv.second.size();
  final_states += (i64)floor.size();
  led.combines = total_states - final_states;
  return led;
}
}  // namespace

extern "C" char* ref_replay_ledger(u64 p, int n, int d, const u64* coeffs, int r_uniform, int nm_override,
                                   int threads) {
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    Hypersurface X = make_x(p, n, d, coeffs);
    std::set<int> S = working_set_for(X, Policy::p_chunk);
    Basis B = compute_basis(X);
    PrecisionPlan plan = choose_precision(p, n, d, overrides(r_uniform, nm_override));
    std::vector<CostLedger> per(B.b);
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::mutex emu;
    for (int t = 0; t < std::max(1, threads); ++t)
      pool.emplace_back([&] {
        try {
          for (int j = next++; j < (int)B.b; j = next++) per[j] = replay_column(X, B, plan, S, j);
        } catch (...) {
          std::lock_guard<std::mutex> lk(emu);
          err = std::current_exception();
        }
      });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
    CostLedger tot;
    std::ostringstream cols;
    for (int j = 0; j < (int)B.b; ++j) {
      tot.matvecs += per[j].matvecs;
      tot.startups += per[j].startups;
      tot.combines += per[j].combines;
      cols << (j ? "," : "") << "[" << per[j].matvecs << "," << per[j].startups << "," << per[j].combines << "]";
    }
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::ostringstream os;
    os << "{\"matvecs\":" << tot.matvecs << ",\"startups\":" << tot.startups << ",\"combines\":" << tot.combines
       << ",\"columns\":[" << cols.str() << "],\"plan\":" << plan_json(plan) << ",\"seconds\":" << secs << "}";
    return os.str();
  });
}

extern "C" {

void ref_free(char* s) { std::free(s); }

int ref_stripe_plan(u64 p, int M, int* limbs, int* limb_exp, u64* beta, long* stripe) {
  try {
    StripePlan pl = StripePlan::make(p, M);
    *limbs = pl.limbs;
    *limb_exp = pl.limb_exp;
    *beta = pl.beta;
    *stripe = pl.stripe;
    return 0;
  } catch (...) {
    return 1;
  }
}

// w <- M(0)...M(tmax) w, A/B/w in the reference's plane-major base-beta layout
int ref_linrec_eval(u64 p, int M, int side, const u64* A, const u64* B, long tmax,
                    u64* w, long* matvecs) {
  try {
    StripePlan pl = StripePlan::make(p, M);
    ModMatrix a = mat_from(pl, side, A), b = mat_from(pl, side, B);
    ModVec v(pl, side);
    std::memcpy(v.d.data(), w, sizeof(u64) * v.d.size());
    i64 ctr = 0;
    linrec_eval(a, b, tmax, v, &ctr);
    std::memcpy(w, v.d.data(), sizeof(u64) * v.d.size());
    if (matvecs) *matvecs = ctr;
    return 0;
  } catch (...) {
    return 1;
  }
}

// the CSC path directly (bypasses linrec_eval's density dispatch)
int ref_sparse_steps(u64 p, int M, int side, const u64* A, const u64* B, long tmax,
                     u64* w, long* matvecs) {
  try {
    StripePlan pl = StripePlan::make(p, M);
    ModMatrix a = mat_from(pl, side, A), b = mat_from(pl, side, B);
    SparseOp sa = SparseOp::build(a), sb = SparseOp::build(b);
    ModVec v(pl, side);
    std::memcpy(v.d.data(), w, sizeof(u64) * v.d.size());
    i64 ctr = 0;
    detail::sparse_steps(pl, sa, sb, tmax, v, &ctr);
    std::memcpy(w, v.d.data(), sizeof(u64) * v.d.size());
    if (matvecs) *matvecs = ctr;
    return 0;
  } catch (...) {
    return 1;
  }
}

// y = A x mod p^M (linalg.hpp:144-192)
int ref_matvec(u64 p, int M, int side, const u64* A, const u64* x, u64* y) {
  try {
    StripePlan pl = StripePlan::make(p, M);
    ModMatrix a = mat_from(pl, side, A);
    ModVec v(pl, side);
    std::memcpy(v.d.data(), x, sizeof(u64) * v.d.size());
    ModVec out = matvec(a, v);
    std::memcpy(y, out.d.data(), sizeof(u64) * out.d.size());
    return 0;
  } catch (...) {
    return 1;
  }
}

// grevlex-descending monomial table (monomial.hpp:129-149), flattened
char* ref_mono_table(int nv, int deg) {
  return guarded([&] {
    const MonoTable& t = mono_table(nv, deg);
    std::ostringstream os;
    os << "{\"mons\":[";
    for (int i = 0; i < t.size(); ++i) os << (i ? "," : "") << expo_arr(t.mons[i]);
    os << "]}";
    return os.str();
  });
}

// random smooth hypersurface by the reference CLI's generator rule
// (drzeta_main.cpp:112-122): mt19937_64(seed), coefficient rng() % p per
// grevlex monomial, redrawn until smooth for the full set and for the
// policy's working set (run_zeta's own two checks, zeta.hpp:440-445).
// mode "fermat" returns sum x_i^d.
char* ref_hypersurface(u64 p, int n, int d, u64 seed, const char* mode, const char* policy) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::string md(mode);
    int nv = n + 1;
    const MonoTable& tab = mono_table(nv, d);
    int tries = 0;
    for (;;) {
      ++tries;
      HomogPoly f(nv, d);
      if (md == "fermat") {
        for (int i = 0; i < nv; ++i) {
          Expo e(nv);
          e[i] = d;
          f.coeff(e) = 1;
        }
      } else {
        for (int i = 0; i < tab.size(); ++i) f.c[i] = (unsigned long)(rng() % p);
      }
      if (f.is_zero()) continue;
      Hypersurface X = Hypersurface::make(p, n, d, f);
      Policy pol = policy_from_name(policy);
      if (!check_smooth(X, full_set(nv))) {
        if (md == "fermat") throw std::runtime_error("fermat not smooth");
        continue;
      }
      if (!check_smooth(X, working_set_for(X, pol))) {
        if (md == "fermat") throw std::runtime_error("fermat not S-smooth");
        continue;
      }
      std::ostringstream os;
      os << "{\"tries\":" << tries << ",\"coeffs\":[";
      for (int i = 0; i < f.size(); ++i) os << (i ? "," : "") << f.c[i].get_str();
      os << "]}";
      return os.str();
    }
  });
}

char* ref_plan(u64 p, int n, int d, int r_uniform, int nm_override) {
  return guarded([&] { return plan_json(choose_precision(p, n, d, overrides(r_uniform, nm_override))); });
}

char* ref_basis(u64 p, int n, int d, const u64* coeffs) {
  return guarded([&] {
    Hypersurface X = make_x(p, n, d, coeffs);
    Basis B = compute_basis(X);
    std::ostringstream os;
    os << "{\"b\":" << B.b << ",\"pole_of\":" << iarr(B.pole_of) << ",\"mons\":[";
    for (size_t i = 0; i < B.mons.size(); ++i) os << (i ? "," : "") << expo_arr(B.mons[i]);
    os << "]}";
    return os.str();
  });
}

// one column's expansion terms and seeds (frobenius.hpp:121-144,
// zeta.hpp:56-69, reduction.hpp:538-563)
char* ref_seeds(u64 p, int n, int d, const u64* coeffs, int r_uniform, int nm_override, int col) {
  return guarded([&] {
    Hypersurface X = make_x(p, n, d, coeffs);
    Basis B = compute_basis(X);
    PrecisionPlan plan = choose_precision(p, n, d, overrides(r_uniform, nm_override));
    StripePlan kp = StripePlan::make(p, plan.M);
    std::set<int> S = default_S(n, d);
    RuvContext C(X, kp, S);
    ModulusContext mctx = ModulusContext::make(p, plan.M);
    int m = B.pole_of[col];
    i64 Pmax = plan.max_pole(m);
    auto terms = frobenius_terms(X, B.mons[col], m, plan);
    std::map<int, mpz_class> kappa;
    kappa[(int)Pmax] = 1;
    mpz_class cur = 1;
    for (i64 t = Pmax - 1; t >= (i64)p * m; --t) {
      cur = mod_reduce(cur * t, mctx.modulus);
      if (t % (i64)p == 0 && t / (i64)p >= m) kappa[(int)t] = cur;
    }
    std::ostringstream os;
    os << "{\"m\":" << m << ",\"Pmax\":" << Pmax << ",\"terms\":[";
    for (size_t i = 0; i < terms.size(); ++i) {
      const auto& t = terms[i];
      GameState st = seed_reduction_input(C, t, kappa.at(t.pole));
      int idx = -1;
      mpz_class val = 0;
      for (int g = 0; g < C.side; ++g)
        if (st.w.get(g) != 0) {
          idx = g;
          val = st.w.get(g);
        }
      os << (i ? "," : "") << "{\"E\":" << expo_arr(t.exponent) << ",\"P\":" << t.pole
         << ",\"dc\":\"" << t.dc.get_str() << "\",\"u\":" << expo_arr(st.u) << ",\"g\":" << idx
         << ",\"val\":\"" << val.get_str() << "\"}";
    }
    os << "]}";
    return os.str();
  });
}

// one chunk of k pole drops along v from state (u, pole) with vector w (plane
// layout of the plan's StripePlan); writes w_out, returns ledger + plan
char* ref_chunk(u64 p, int n, int d, const u64* coeffs, int M, const int* u, int pole,
                const int* v, long k, const u64* w_in, u64* w_out) {
  return guarded([&] {
    Hypersurface X = make_x(p, n, d, coeffs);
    StripePlan kp = StripePlan::make(p, M);
    std::set<int> S = default_S(n, d);
    RuvContext C(X, kp, S);
    BuildStore store(C);
    GameState st;
    st.u = Expo(n + 1);
    Expo vv(n + 1);
    for (int i = 0; i <= n; ++i) {
      st.u[i] = u[i];
      vv[i] = v[i];
    }
    st.pole = pole;
    st.w = ModVec(kp, C.side);
    std::memcpy(st.w.d.data(), w_in, sizeof(u64) * st.w.d.size());
    CostLedger led;
    reduce_chunk(C, store, st, vv, k, led);
    std::memcpy(w_out, st.w.d.data(), sizeof(u64) * st.w.d.size());
    std::ostringstream os;
    os << "{\"side\":" << C.side << ",\"limbs\":" << kp.limbs << ",\"u\":" << expo_arr(st.u)
       << ",\"pole\":" << st.pole << ",\"matvecs\":" << led.matvecs << ",\"startups\":" << led.startups
       << "}";
    return os.str();
  });
}

// Frobenius matrix (zeta.hpp:36-136) plus the charpoly residues the driver
// derives from it (zeta.hpp:456-458)
char* ref_frobenius(u64 p, int n, int d, const u64* coeffs, const char* policy, const char* pep,
                    int threads, int r_uniform, int nm_override, int only_pole) {
  return guarded([&] {
    Hypersurface X = make_x(p, n, d, coeffs);
    Policy pol = policy_from_name(policy);
    std::set<int> S = working_set_for(X, pol);
    Basis B = compute_basis(X);
    PrecisionPlan plan = choose_precision(p, n, d, overrides(r_uniform, nm_override));
    auto t0 = std::chrono::steady_clock::now();
    FrobeniusOutput fo = frobenius_matrix(X, B, plan, pol, pep, S, only_pole, threads);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<mpz_class> dres;
    if (!only_pole)
      dres = berkowitz_charpoly(fo.F, (int)fo.b, mpz_pow_ui(p, (unsigned long)(plan.M + n)));
    std::ostringstream os;
    os << "{\"b\":" << fo.b << ",\"plan\":" << plan_json(plan) << ",\"F\":" << zarr(fo.F)
       << ",\"charpoly\":" << zarr(dres) << ",\"matvecs\":" << fo.cost.matvecs
       << ",\"startups\":" << fo.cost.startups << ",\"combines\":" << fo.cost.combines
       << ",\"pep_misses\":" << fo.pep.misses << ",\"seconds\":" << secs << "}";
    return os.str();
  });
}

// Fedder's F-splitting criterion of run_zeta's invariants (zeta.hpp:336-350,
// 536-539): 1 / 0, or -1 where run_zeta leaves it undefined (d > n + 1)
int ref_fsplit(u64 p, int n, int d, const u64* coeffs) {
  Hypersurface X = make_x(p, n, d, coeffs);
  if (d > X.nv()) return -1;
  return fedder_is_fsplit(X) ? 1 : 0;
}

// full driver (zeta.hpp:438-549)
char* ref_zeta(u64 p, int n, int d, const u64* coeffs, const char* policy, const char* pep,
               int threads, int r_uniform, int nm_override, int verify_counts) {
  return guarded([&] {
    Hypersurface X = make_x(p, n, d, coeffs);
    ZetaOptions o;
    o.policy = policy_from_name(policy);
    o.pep = pep;
    o.threads = threads;
    o.overrides = overrides(r_uniform, nm_override);
    o.verify_counts = verify_counts != 0;
    ZetaResult r = run_zeta(X, o);
    std::ostringstream os;
    os << "{\"Q\":" << zarr(r.Q) << ",\"ambiguous\":" << (r.ambiguous ? "true" : "false")
       << ",\"plan\":" << plan_json(r.plan) << ",\"matvecs\":" << r.cost.matvecs
       << ",\"startups\":" << r.cost.startups << ",\"combines\":" << r.cost.combines
       << ",\"pep_misses\":" << r.pep.misses << ",\"p_rank\":" << r.inv.p_rank << ",\"height\":\""
       << r.inv.height << "\",\"domino\":\"" << r.inv.domino << "\",\"newton_height\":\""
       << r.inv.newton_height << "\",\"slopes\":[";
    for (size_t i = 0; i < r.np.slopes.size(); ++i)
      os << (i ? "," : "") << "[\"" << mpq_str(r.np.slopes[i].first) << "\"," << r.np.slopes[i].second << "]";
    os << "],\"counts\":[";
    for (size_t i = 0; i < r.counts.size(); ++i)
      os << (i ? "," : "") << "[" << r.counts[i].r << ",\"" << r.counts[i].from_zeta.get_str() << "\","
         << (r.counts[i].ok ? "true" : "false") << "]";
    os << "],\"seconds\":" << r.wall_seconds << "}";
    return os.str();
  });
}

// Bounded sample of the reference's own hot path for CPU-baseline timing:
// the exact setup of frobenius_matrix (zeta.hpp:41-69: RuvContext, lazy PEP
// store, frobenius_terms, kappa prescale, seeds) for column `col`, then the
// reference run_policy (p-chunk) on `threads` disjoint groups of that
// column's top-pole seeds (at most max_seeds per group), one std::thread per
// group sharing the store exactly as the column workers do (zeta.hpp:109-133).
// Reports wall seconds and the ledger of the sampled work.
char* ref_policy_sample(u64 p, int n, int d, const u64* coeffs, int r_uniform, int nm_override, int col,
                        int max_seeds, int threads) {
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    Hypersurface X = make_x(p, n, d, coeffs);
    Basis B = compute_basis(X);
    PrecisionPlan plan = choose_precision(p, n, d, overrides(r_uniform, nm_override));
    StripePlan kp = StripePlan::make(p, plan.M);
    std::set<int> S = default_S(n, d);
    RuvContext C(X, kp, S);
    auto store = make_pep_store("lazy", C);
    ModulusContext mctx = ModulusContext::make(p, plan.M);
    int m = B.pole_of[col];
    i64 Pmax = plan.max_pole(m);
    auto terms = frobenius_terms(X, B.mons[col], m, plan);
    std::map<int, mpz_class> kappa;
    kappa[(int)Pmax] = 1;
    mpz_class cur = 1;
    for (i64 t = Pmax - 1; t >= (i64)p * m; --t) {
      cur = mod_reduce(cur * t, mctx.modulus);
      if (t % (i64)p == 0 && t / (i64)p >= m) kappa[(int)t] = cur;
    }
    std::vector<std::vector<GameState>> groups(threads);
    int g = 0;
    for (const auto& t : terms) {
      if (t.pole != (int)Pmax) continue;
      if ((int)groups[g].size() < max_seeds) groups[g].push_back(seed_reduction_input(C, t, kappa.at(t.pole)));
      g = (g + 1) % threads;
    }
    double setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<CostLedger> leds(threads);
    auto t1 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i)
      pool.emplace_back([&, i] { run_policy(C, *store, std::move(groups[i]), Policy::p_chunk, leds[i]); });
    for (auto& th : pool) th.join();
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    CostLedger tot;
    for (auto& l : leds) {
      tot.matvecs += l.matvecs;
      tot.startups += l.startups;
      tot.combines += l.combines;
    }
    std::ostringstream os;
    os << "{\"seconds\":" << secs << ",\"setup_seconds\":" << setup << ",\"matvecs\":" << tot.matvecs
       << ",\"startups\":" << tot.startups << ",\"combines\":" << tot.combines << ",\"threads\":" << threads
       << ",\"Pmax\":" << Pmax << "}";
    return os.str();
  });
}

// Berkowitz charpoly + recover_Q on a given F (zeta.hpp:456-470)
char* ref_charpoly(u64 p, int n, int d, int r_uniform, int nm_override, int b, const char* const* F) {
  return guarded([&] {
    PrecisionPlan plan = choose_precision(p, n, d, overrides(r_uniform, nm_override));
    std::vector<mpz_class> f((size_t)b * b);
    for (size_t i = 0; i < f.size(); ++i) f[i] = mpz_class(F[i]);
    auto dres = berkowitz_charpoly(f, b, mpz_pow_ui(p, (unsigned long)(plan.M + n)));
    RecoverOutcome rec = recover_Q(dres, plan);
    std::ostringstream os;
    os << "{\"charpoly\":" << zarr(dres) << ",\"status\":" << (int)rec.status << ",\"candidates\":[";
    for (size_t i = 0; i < rec.candidates.size(); ++i) os << (i ? "," : "") << zarr(rec.candidates[i]);
    os << "]}";
    return os.str();
  });
}


// A reusable RuvContext + build_ruv store for many chunks at one (f, M): the
// random cubic fourfold's context (a 3003 x 6237 unit echelon, MpzEchelon
// at 2 limbs) takes hours to build, so the fixture script builds it once.
struct RefCtx {
  Hypersurface X;
  StripePlan kp;
  std::set<int> S;
  RuvContext C;
  BuildStore store;
  RefCtx(const Hypersurface& x, const StripePlan& p, const std::set<int>& s)
      : X(x), kp(p), S(s), C(x, p, s), store(C) {}
};

void* ref_ctx_new(u64 p, int n, int d, const u64* coeffs, int M) {
  try {
    Hypersurface X = make_x(p, n, d, coeffs);
    return new RefCtx(X, StripePlan::make(p, M), default_S(n, d));
  } catch (...) {
    return nullptr;
  }
}

void ref_ctx_free(void* h) { delete (RefCtx*)h; }

// reduce_chunk (reduction.hpp:394-423) on the shared context
char* ref_ctx_chunk(void* h, const int* u, int pole, const int* v, long k, const u64* w_in, u64* w_out) {
  return guarded([&] {
    RefCtx& R = *(RefCtx*)h;
    int nv = R.X.nv();
    GameState st;
    st.u = Expo(nv);
    Expo vv(nv);
    for (int i = 0; i < nv; ++i) {
      st.u[i] = u[i];
      vv[i] = v[i];
    }
    st.pole = pole;
    st.w = ModVec(R.kp, R.C.side);
    std::memcpy(st.w.d.data(), w_in, sizeof(u64) * st.w.d.size());
    CostLedger led;
    auto t0 = std::chrono::steady_clock::now();
    reduce_chunk(R.C, R.store, st, vv, k, led);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(w_out, st.w.d.data(), sizeof(u64) * st.w.d.size());
    std::ostringstream os;
    os << "{\"side\":" << R.C.side << ",\"limbs\":" << R.kp.limbs << ",\"u\":" << expo_arr(st.u)
       << ",\"pole\":" << st.pole << ",\"matvecs\":" << led.matvecs << ",\"startups\":" << led.startups
       << ",\"seconds\":" << secs << "}";
    return os.str();
  });
}


// reference run_policy (reduction.hpp:464-533) on caller-given GameStates
// (u, pole, w in ModVec layout), then floor_to_numerator (reduction.hpp:
// 566-581) of every floor state: the oracle of the device states API
char* ref_run_policy_states(u64 p, int n, int d, const u64* coeffs, int M, const char* policy, int count,
                            const int* u, const int* pole, const u64* w) {
  return guarded([&] {
    Hypersurface X = make_x(p, n, d, coeffs);
    Policy pol = policy_from_name(policy);
    StripePlan kp = StripePlan::make(p, M);
    RuvContext C(X, kp, working_set_for(X, pol));
    auto store = make_pep_store("lazy", C);
    const int nv = n + 1;
    std::vector<GameState> sts;
    for (int i = 0; i < count; ++i) {
      GameState st;
      st.u = Expo(nv);
      for (int j = 0; j < nv; ++j) st.u[j] = u[(size_t)i * nv + j];
      st.pole = pole[i];
      st.w = ModVec(kp, C.side);
      std::memcpy(st.w.d.data(), w + (size_t)i * st.w.d.size(), sizeof(u64) * st.w.d.size());
      sts.push_back(std::move(st));
    }
    CostLedger led;
    std::vector<GameState> fl = run_policy(C, *store, std::move(sts), pol, led);
    std::vector<mpz_class> g;
    for (const auto& st : fl) floor_to_numerator(C, st, g);
    std::ostringstream os;
    os << "{\"matvecs\":" << led.matvecs << ",\"startups\":" << led.startups << ",\"combines\":" << led.combines
       << ",\"g\":" << zarr(g) << ",\"states\":[";
    for (size_t i = 0; i < fl.size(); ++i) {
      os << (i ? "," : "") << "{\"u\":" << expo_arr(fl[i].u) << ",\"pole\":" << fl[i].pole << ",\"w\":[";
      for (size_t j = 0; j < fl[i].w.d.size(); ++j) os << (j ? "," : "") << "\"" << fl[i].w.d[j] << "\"";
      os << "]}";
    }
    os << "]}";
    return os.str();
  });
}


// build_ruv(C, v) (reduction.hpp:253-297): the n+2 matrices in ModMatrix plane
// layout, (n+2) x limbs x side x side, plus PepEntry::nnz
int ref_build_ruv(u64 p, int n, int d, const u64* coeffs, int M, const char* policy, const int* v, u64* out,
                  long* nnz) {
  try {
    Hypersurface X = make_x(p, n, d, coeffs);
    StripePlan kp = StripePlan::make(p, M);
    RuvContext C(X, kp, working_set_for(X, policy_from_name(policy)));
    Expo vv(n + 1);
    for (int i = 0; i <= n; ++i) vv[i] = v[i];
    PepEntry E = build_ruv(C, vv);
    size_t off = 0;
    for (const auto& m : E.mats) {
      std::memcpy(out + off, m.d.data(), sizeof(u64) * m.d.size());
      off += m.d.size();
    }
    *nnz = E.nnz;
    return 0;
  } catch (...) {
    return 1;
  }
}

}  // extern "C"
