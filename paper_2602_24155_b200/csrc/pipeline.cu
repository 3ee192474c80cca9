// Frobenius assembly + zeta driver (see pipeline.cuh).
#include <future>
#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <thread>
#include <condition_variable>
#include <map>
#include <mutex>

#include "pipeline.cuh"
#include "kernels/count.cuh"

namespace drzg {

namespace {
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

// one stream per (host thread, device), kept for the thread's life: the
// engine's stream-ordered temporaries return to the retained pool on it and
// the next call's allocations reuse them in stream order (a fresh stream per
// call made cudaMallocAsync grow the pool again, up to 0.3 s per K3 zeta);
// calls on different host threads (a batch of hypersurfaces) overlap
cudaStream_t device_stream(int device) {
  struct Streams {
    std::map<int, cudaStream_t> by_dev;
    ~Streams() {
      for (auto& kv : by_dev) {
        cudaSetDevice(kv.first);
        cudaStreamSynchronize(kv.second);
        cudaStreamDestroy(kv.second);
      }
    }
  };
  thread_local Streams s;
  auto it = s.by_dev.find(device);
  if (it != s.by_dev.end()) return it->second;
  cudaStream_t st;
  DRZG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  s.by_dev[device] = st;
  return st;
}

std::set<int> working_set_for(const Hypersurface& X, Policy pol) {
  if (pol == Policy::var_by_var) return {X.n};
  return default_S(X.n, X.d);
}

FrobResult frobenius_matrix(const Hypersurface& X, const Basis& B, const PrecisionPlan& plan, const std::set<int>& S,
                            const FrobOptions& opt, int device) {
  double t0 = now_s();
  ActiveCall active;  // concurrent calls split the host cores
  DRZG_CUDA(cudaSetDevice(device));
  cudaStream_t st = device_stream(device);
  FrobResult out;
  const int n = X.n;
  const u64 p = X.p;
  out.b = B.b;
  out.F.assign((size_t)B.b * B.b, Z(0));
  out.M = plan.M;

  RuvTables T = build_tables(X, plan.M, S);
  out.Ld = T.dp.Ld;
  out.q = T.dp.q;
  out.nL = T.nL;
  out.side = T.side;
  HostMod hm = HostMod::make(p, plan.M);
  double t1 = now_s();
  out.t.tables = t1 - t0;
  const bool verbose = std::getenv("DRZG_VERBOSE") != nullptr;
  auto mark = [&](const char* what) {
    if (verbose) std::fprintf(stderr, "[drzg] frobenius wall %s %.3f\n", what, now_s() - t0);
  };

  std::vector<int> cols;
  for (int j = 0; j < (int)B.b; ++j) {
    if (opt.only_pole && B.pole_of[j] != opt.only_pole) continue;
    if (!opt.columns.empty() && std::find(opt.columns.begin(), opt.columns.end(), j) == opt.columns.end()) continue;
    cols.push_back(j);
  }
  out.computed = cols;
  // column expansions on background host threads (the reference threads over
  // columns too, zeta.hpp:109-133), overlapped with the device: a group of
  // columns starts as soon as its own seeds exist, while later columns are
  // still being expanded.  The final reducer's levels are built meanwhile.
  PowerCache pc;
  // the power series at the largest (N_m, s_m) of the run's columns, once, on
  // every expansion thread (the columns then reduce its prefix); expansion
  // thread 0 primes it while this thread builds the final reducer
  int Nmax = 0, smax = 0;
  for (int j : cols) {
    const int m = B.pole_of[j];
    Nmax = std::max(Nmax, plan.N_m[m]);
    smax = std::max(smax, plan.s_m[m]);
  }
  std::vector<ColumnSeeds> seeds(cols.size());
  std::vector<char> ready(cols.size(), 0);
  std::mutex smu;
  std::condition_variable scv;
  std::exception_ptr serr;
  FinalReducer fin(X, B, T.dp, hm);
  // expansion takes every core, at a lower scheduling priority (nice +10):
  // before the first group nothing else needs the host, and once the device
  // runs the engine's policy, launcher and seed-preparer threads preempt it
  const int nexp = std::max(1, std::min<int>((int)cols.size(), (int)call_cores()));
  // The first columns are on the device's critical path (the first group
  // starts when its seeds exist): they are expanded one at a time with all
  // the expansion threads on each (monomials of f^j split between them); the
  // rest one column per thread, overlapped with the device.
  // (only columns large enough to split: a column's dense term bound above
  // 2^18 monomials, as for the fourfold's 3.1 M; small ones, K3's, stay one
  // per thread)
  size_t first = 0;
  while (first < std::min<size_t>(2, cols.size())) {
    const int m = B.pole_of[cols[first]];
    double tb = 0;
    for (int j = 0; j < plan.N_m[m]; ++j) tb += (double)mono_count(X.nv(), X.d * j);
    if (tb < (double)(1 << 18)) break;
    ++first;
  }
  // more small columns than threads (K3: 21 on 16): each column in two
  // parts of about equal work (powers [0, jm) and [jm, N)), so the last
  // round of whole columns does not leave most threads idle
  const bool halves = first == 0 && cols.size() > (size_t)nexp && !std::getenv("DRZG_EXPAND_WHOLE");
  std::vector<int> jsplit(cols.size(), 1 << 30);
  if (halves)
    for (size_t i = 0; i < cols.size(); ++i) {
      const int m = B.pole_of[cols[i]];
      double tot = 0, acc = 0;
      for (int j = 0; j < plan.N_m[m]; ++j) tot += (double)mono_count(X.nv(), X.d * j);
      int jm = 0;
      while (jm < plan.N_m[m] && acc + (double)mono_count(X.nv(), X.d * jm) <= tot / 2)
        acc += (double)mono_count(X.nv(), X.d * jm++);
      jsplit[i] = jm;
    }
  std::vector<ColumnSeeds> upper(cols.size());
  std::vector<std::atomic<int>> parts_left(cols.size());
  for (auto& a : parts_left) a = halves ? 2 : 1;
  const size_t nitems = halves ? 2 * cols.size() : cols.size();
  std::atomic<size_t> next{first};
  std::atomic<bool> first_done{false};
  std::vector<std::thread> pool;
  auto join_pool = [&] {
    for (auto& th : pool)
      if (th.joinable()) th.join();
  };
  auto expand_one = [&](size_t i, int threads) {
    try {
      ColumnSeeds cs = expand_column(X, B, plan, T, hm, pc, cols[i], threads);
      std::lock_guard<std::mutex> lk(smu);
      seeds[i] = std::move(cs);
      ready[i] = 1;
    } catch (...) {
      std::lock_guard<std::mutex> lk(smu);
      if (!serr) serr = std::current_exception();
      ready[i] = 1;
    }
    scv.notify_all();
  };
  // work item k: column k / 2, lower (even k) or upper (odd k) powers
  auto expand_item = [&](size_t k) {
    if (!halves) {
      expand_one(k, 1);
      return;
    }
    const size_t i = k / 2;
    try {
      ColumnSeeds cs = (k & 1) ? expand_column(X, B, plan, T, hm, pc, cols[i], 1, jsplit[i])
                               : expand_column(X, B, plan, T, hm, pc, cols[i], 1, 0, jsplit[i]);
      std::lock_guard<std::mutex> lk(smu);
      ColumnSeeds& dst = (k & 1) ? upper[i] : seeds[i];
      dst = std::move(cs);
      if (--parts_left[i] == 0) {
        for (auto& kv : upper[i].by_pole) seeds[i].by_pole[kv.first] = std::move(kv.second);
        seeds[i].nterms += upper[i].nterms;
        upper[i] = ColumnSeeds();
        ready[i] = 1;
      }
    } catch (...) {
      std::lock_guard<std::mutex> lk(smu);
      if (!serr) serr = std::current_exception();
      ready[i] = 1;
    }
    scv.notify_all();
  };
  for (int t = 0; t < nexp; ++t)
    pool.emplace_back([&, t] {
      setpriority(PRIO_PROCESS, (id_t)syscall(SYS_gettid), 10);  // best effort
      if (t == 0) {
        try {
          const double tp0 = now_s();
          pc.prime(X, Nmax, smax, nexp);
          if (std::getenv("DRZG_VERBOSE")) std::fprintf(stderr, "[drzg] power series primed %.4f s\n", now_s() - tp0);
        } catch (...) {
          std::lock_guard<std::mutex> lk(smu);
          if (!serr) serr = std::current_exception();
        }
        for (size_t i = 0; i < first; ++i) expand_one(i, nexp);
        {
          std::lock_guard<std::mutex> lk(smu);
          first_done = true;
        }
        scv.notify_all();
      } else {
        std::unique_lock<std::mutex> lk(smu);
        scv.wait(lk, [&] { return first_done.load() || serr; });
      }
      for (size_t k = next++; k < nitems; k = next++) expand_item(k);
    });
  auto wait_column = [&](size_t i) -> ColumnSeeds& {
    std::unique_lock<std::mutex> lk(smu);
    scv.wait(lk, [&] { return ready[i] || serr; });
    if (serr) {
      lk.unlock();
      join_pool();
      std::rethrow_exception(serr);
    }
    return seeds[i];
  };
  try {
    fin.prepare();
  } catch (...) {
    next = nitems;
    join_pool();
    throw;
  }
  double t2 = now_s();
  mark("prepared");

  // columns run through the device engine in groups whose states fit HBM:
  // live states stay below ~60% of a group's seeds (SURVEY 8a peaks), and a
  // group may use half of the free memory
  std::vector<std::vector<i64>> G(cols.size());
  double td0 = 0, seed_wait = 0;
  try {
    const double te0 = now_s();
    ReductionEngine eng(T, n, p, st);
    if (std::getenv("DRZG_VERBOSE")) std::fprintf(stderr, "[drzg] engine setup %.3f s\n", now_s() - te0);
    mark("engine");
    eng.clock.on = opt.profile;
    size_t fr = 0, tot = 0;
    {
      // the grouping budget: free memory matters only when the columns' seeds
      // could approach it (the driver query is slow on a busy device)
      double all = 0;
      for (size_t c = 0; c < cols.size(); ++c) {
        const int m = B.pole_of[cols[c]];
        for (int j = 0; j < plan.N_m[m]; ++j) all += (double)mono_count(X.nv(), X.d * j);
      }
      const double slot = (double)T.dp.Ld * ((T.side + 15) / 16 * 16);
      const size_t tm = device_total_memory();
      if (tm && all * slot < 0.05 * (double)tm)
        fr = tot = tm;
      else
        mem_info(&fr, &tot, "pipeline.cu:1");
      // memory this process holds but no one uses counts as free: the state
      // pool a finished engine left mapped and the retained mempool's slack
      int dev = 0;
      DRZG_CUDA(cudaGetDevice(&dev));
      fr += cached_pool_bytes(dev);
      cudaMemPool_t mp;
      DRZG_CUDA(cudaDeviceGetDefaultMemPool(&mp, dev));
      unsigned long long res = 0, used = 0;
      DRZG_CUDA(cudaMemPoolGetAttribute(mp, cudaMemPoolAttrReservedMemCurrent, &res));
      DRZG_CUDA(cudaMemPoolGetAttribute(mp, cudaMemPoolAttrUsedMemCurrent, &used));
      if (res > used) fr += (size_t)(res - used);
    }
    const double slot_bytes = (double)T.dp.Ld * ((T.side + 15) / 16 * 16);
    // live states peak near 0.35 of the dense term bound (the random
    // fourfold: 1.08M of 3.1M per column), so 0.45 of it against 55% of free
    // HBM leaves the batch temporaries (<= 12% of the device) room; two
    // fourfold columns per group halve the group start-ups and double the
    // batches (151.9 against 160.9 s of device time per zeta function)
    constexpr double kPeakPerBound = 0.45;
    const double budget = 0.55 * (double)fr;
    if (verbose && !cols.empty()) {
      double b0 = 0;
      const int m = B.pole_of[cols[0]];
      for (int j = 0; j < plan.N_m[m]; ++j) b0 += (double)mono_count(X.nv(), X.d * j);
      std::fprintf(stderr, "[drzg] grouping: column 0 dense term bound %.0f (%.1f GB of states at %.2f), budget %.1f GB\n",
                   b0, kPeakPerBound * b0 * slot_bytes / 1e9, kPeakPerBound, budget / 1e9);
    }
    bool heavy = false;
    {
      double all_terms = 0;
      for (size_t c = 0; c < cols.size(); ++c) {
        const int m = B.pole_of[cols[c]];
        for (int j = 0; j < plan.N_m[m]; ++j) all_terms += (double)mono_count(X.nv(), X.d * j);
      }
      heavy = all_terms > (double)(1 << 24);
    }
    size_t c0 = 0;
    while (c0 < cols.size()) {
      size_t c1 = c0;
      double need = 0;
      const double w0 = now_s();
      // group sizes from the dense bound on a column's terms (sum over j of
      // |Homog_{dj}|, what frobenius_terms yields for a dense f^j): no wait
      // for columns that will not be in this group
      auto terms_bound = [&](size_t c) {
        const int m = B.pole_of[cols[c]];
        double t = 0;
        for (int j = 0; j < plan.N_m[m]; ++j) t += (double)mono_count(X.nv(), X.d * j);
        return t;
      };
      static const int group_cols = [] {
        const char* e = std::getenv("DRZG_GROUP_COLS");  // A/B override: columns per group
        return e ? std::max(1, std::atoi(e)) : 0;
      }();
      // a heavy expansion (the quintic surface: 52 columns of ~2M terms each)
      // starts the device on a quarter of the columns, the rest expanding
      // meanwhile
      const size_t first_cap = heavy && c0 == 0 ? std::max<size_t>(2, (cols.size() + 3) / 4) : cols.size();
      while (c1 < cols.size()) {
        double add = kPeakPerBound * terms_bound(c1) * slot_bytes;
        if (group_cols ? (int)(c1 - c0) >= group_cols : (c1 > c0 && (need + add > budget || c1 - c0 >= first_cap)))
          break;
        need += add;
        ++c1;
      }
      for (size_t c = c0; c < c1; ++c) wait_column(c);
      seed_wait += now_s() - w0;
      mark("group seeds");
      std::vector<ColumnSeeds> grp;
      {
        std::lock_guard<std::mutex> lk(smu);
        for (size_t i = c0; i < c1; ++i) {
          out.terms += seeds[i].nterms;
          grp.push_back(std::move(seeds[i]));
        }
      }
      std::vector<std::vector<i64>> Gg;
      const double tg = now_s();
      const i64 mv0 = out.led.matvecs;
      if (opt.policy == Policy::p_chunk)
        eng.run_pchunk(grp, Gg, out.led);  // pipelined: policy thread + launcher
      else
        eng.run_rounds(grp, Gg, out.led, opt.policy);  // depth-first, var-by-var
      if (std::getenv("DRZG_VERBOSE"))
        std::fprintf(stderr, "[drzg] group %d: columns %zu-%zu, %lld matvecs, %.2f s, peak live %lld\n", out.groups,
                     c0, c1 - 1, (long long)(out.led.matvecs - mv0), now_s() - tg, (long long)eng.peak_live());
      for (size_t i = c0; i < c1; ++i) G[i] = std::move(Gg[i - c0]);
      c0 = c1;
      ++out.groups;
    }
    eng.clock.peak_live = eng.peak_live();
    out.clk = eng.clock;
    td0 = now_s();
  } catch (...) {
    next = nitems;
    join_pool();
    throw;
  }
  mark("engine closed");
  join_pool();
  double t3 = now_s();
  mark("expansion joined");
  if (std::getenv("DRZG_VERBOSE")) std::fprintf(stderr, "[drzg] engine teardown %.3f s\n", t3 - td0);
  // seeds: the host time the device waited for expansions (the rest overlapped)
  out.t.seeds = (t2 - t1) + seed_wait;
  out.t.device = t3 - t2 - seed_wait;

  const int gsize = (int)mono_count(X.nv(), T.D - 1);
  std::vector<std::vector<Z>> colres(cols.size());
  {
    const int nth = std::max(1, std::min<int>((int)cols.size(), (int)call_cores()));
    std::atomic<size_t> next{0};
    std::vector<std::exception_ptr> errs(nth);
    std::vector<std::thread> pool;
    for (int t = 0; t < nth; ++t)
      pool.emplace_back([&, t] {
        try {
          for (size_t ci = next++; ci < cols.size(); ci = next++) {
            std::vector<Z> g(gsize);
            for (int r = 0; r < gsize; ++r) {
              i64 s[dev::kLdMax];
              for (int tt = 0; tt < T.dp.Ld; ++tt) s[tt] = G[ci][(size_t)tt * gsize + r];
              g[r] = from_digit_sums(s, T.dp, hm.mz);
            }
            colres[ci] = fin.reduce(std::move(g), n);
          }
        } catch (...) {
          errs[t] = std::current_exception();
        }
      });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  }
  for (size_t ci = 0; ci < cols.size(); ++ci) {
    int j = cols[ci];
    int m = B.pole_of[j];
    i64 Pmax = plan.max_pole(m);
    const std::vector<Z>& c = colres[ci];
    // unscale by the unit of kappa_n = (Pmax-1)!/(n-1)! and the Mazur shift
    // (zeta.hpp:79-106)
    i64 v = factorial_valuation((u64)(Pmax - 1), p);
    Z unit(1);
    for (i64 t = n; t < Pmax; ++t) unit *= Z((long)t);
    Z pz = Z::from_u64(p);
    for (i64 t = 0; t < v; ++t) {
      DRZG_REQUIRE(unit.divisible_by(p), "kappa: bad valuation");
      unit = unit.divexact(pz);
    }
    Z iu = unit.mod(hm.mz).inverse_mod(hm.mz);
    i64 req = std::min<i64>(std::max<i64>(v - m + 1, 0), plan.M);
    Z preq = Z::pow(p, (u64)req);
    i64 shift = (i64)(n - 1) - v;
    Z pshift = Z::pow(p, (u64)(shift < 0 ? -shift : shift));
    for (int i = 0; i < (int)B.b; ++i) {
      Z Zi = (c[i] * iu).mod(hm.mz);
      DRZG_REQUIRE(Zi.divisible_by(preq), "column fails the p-divisibility floor of its pole order");
      Z& Fij = out.F[(size_t)i * B.b + j];
      if (shift >= 0) {
        Fij = Zi * pshift;
      } else {
        DRZG_REQUIRE(Zi.divisible_by(pshift), "column entry not integral after unscaling");
        Fij = Zi.divexact(pshift);
      }
    }
  }
  double t4 = now_s();
  out.t.final = t4 - t3;
  out.t.total = t4 - t0;
  DRZG_CUDA(cudaStreamSynchronize(st));
  return out;
}

namespace {
// #X(F_{p^r}): device enumeration for large fields, host below
i64 count_points_any(const Hypersurface& X, int r, i64 budget) {
  Z pts(0);
  for (int i = 0; i <= X.n; ++i) pts += Z::pow(ipow(X.p, r), (u64)i);
  if (pts >= Z((long)kDeviceCountMin)) return count_points_device(X, r, budget);
  return count_points(X, r, budget);
}
}  // namespace

std::string finish_zeta(const Hypersurface& X, const PrecisionPlan& plan, const std::vector<Z>& F, i64 b,
                        const ZetaOptions& opt, ZetaOut& res, const int* fsplit_known) {
  res.hodge = hodge_numbers(X.n, X.d);
  Z cp_mod = Z::pow(X.p, (u64)(plan.M + X.n));
  const double tb0 = now_s();
  std::vector<Z> dres = berkowitz(F, (int)b, cp_mod);
  if (std::getenv("DRZG_VERBOSE")) std::fprintf(stderr, "[drzg] charpoly %.4f s\n", now_s() - tb0);
  Recovered rec = recover_Q(dres, plan);
  if (rec.status == 2) return rec.reason;
  auto cands = std::move(rec.candidates);
  bool ambiguous = false;
  if (cands.size() > 1) {
    int rounds = 0;
    for (int r = 1; r <= 3 && cands.size() > 1; ++r) {
      Z pts(0);
      for (int i = 0; i <= X.n; ++i) pts += Z::pow(ipow(X.p, r), (u64)i);
      if (pts > Z((long)opt.count_budget)) break;
      ++rounds;
      Z truth((long)count_points_any(X, r, opt.count_budget));
      std::vector<std::vector<Z>> kept;
      for (auto& c : cands)
        if (counts_from_zeta(c, X.p, X.n, r) == truth) kept.push_back(c);
      if (kept.empty()) break;
      cands = std::move(kept);
    }
    if (cands.empty() || (cands.size() > 1 && rounds > 0)) return "sign of the functional equation undecided";
    ambiguous = cands.size() > 1;
  }
  std::vector<Z> a = cands.front();
  NewtonPolygon np = newton_polygon(a, X.p);
  bool geom_ok = np.vertices.front() == std::make_pair<i64, i64>(0, 0);
  i64 HP_end = hodge_polygon_at(res.hodge, X.n, plan.b);
  geom_ok = geom_ok && np.vertices.back().first == plan.b && np.vertices.back().second == HP_end;
  for (i64 x = 0; x <= plan.b && geom_ok; ++x)
    if (np.value_at(x) < Q64::make(hodge_polygon_at(res.hodge, X.n, x), 1)) geom_ok = false;
  if (!geom_ok) return "Newton polygon escapes the Hodge bound";
  std::vector<CountCheck> checks;
  bool counts_ok = true;
  if (opt.verify_counts && !ambiguous) {
    for (int r = 1; r <= 2; ++r) {
      Z pts(0);
      for (int i = 0; i <= X.n; ++i) pts += Z::pow(ipow(X.p, r), (u64)i);
      if (pts > Z((long)opt.count_budget)) break;
      CountCheck ck;
      ck.r = r;
      ck.from_zeta = counts_from_zeta(a, X.p, X.n, r);
      const double tc0 = now_s();
      ck.from_count = Z((long)count_points_any(X, r, opt.count_budget));
      if (std::getenv("DRZG_VERBOSE")) std::fprintf(stderr, "[drzg] count r=%d %.4f s\n", r, now_s() - tc0);
      ck.ok = ck.from_zeta == ck.from_count;
      counts_ok = counts_ok && ck.ok;
      checks.push_back(ck);
    }
  }
  if (!counts_ok) return "point counts disagree with the recovered zeta";
  res.Q = a;
  res.ambiguous = ambiguous;
  if (ambiguous) res.Q_alt = cands.back();
  res.np = np;
  res.inv = classify(np, res.hodge, X.n, X.d);
  res.domino = domino_number(np, res.hodge, X.n);
  if (X.d <= X.nv()) {
    const double tf0 = now_s();
    res.inv.fsplit_defined = true;
    res.inv.fsplit = fsplit_known ? *fsplit_known != 0 : fedder_is_fsplit(X);
    if (std::getenv("DRZG_VERBOSE")) std::fprintf(stderr, "[drzg] fsplit %.4f s\n", now_s() - tf0);
  }
  res.counts = checks;
  res.plan = plan;
  return "";
}

ZetaOut run_zeta(const Hypersurface& X, const ZetaOptions& opt, int device) {
  double t0 = now_s();
  if (!check_smooth(X, full_set(X.nv())))
    throw singular_input("hypersurface is singular (weighted Jacobian not surjective)");
  std::set<int> S = working_set_for(X, opt.policy);
  if (!check_smooth(X, S)) throw std::runtime_error("input not smooth for the requested working set");
  Basis B = compute_basis(X);
  PrecisionPlan plan = choose_precision(X.p, X.n, X.d, opt.overrides);
  if (std::getenv("DRZG_VERBOSE")) std::fprintf(stderr, "[drzg] zeta setup %.4f s\n", now_s() - t0);
  ZetaOut res;
  // Fedder's F-split test depends on f alone: on the host beside the
  // Frobenius matrix instead of after it
  std::future<bool> fs_future;
  if (X.d <= X.nv()) fs_future = std::async(std::launch::async, [&X] { return fedder_is_fsplit(X); });
  int fs_value = -1;
  for (;;) {
    FrobOptions fo;
    fo.policy = opt.policy;
    fo.overrides = opt.overrides;
    fo.profile = opt.profile;
    FrobResult fr = frobenius_matrix(X, B, plan, S, fo, device);
    res.led = fr.led;
    std::vector<Z> F = fr.F;
    const i64 b = fr.b;
    res.last = std::move(fr);
    // the reference's escalation ladder (zeta.hpp:472-535): more series
    // terms, then more digits, until the battery passes
    if (fs_future.valid()) fs_value = fs_future.get() ? 1 : 0;
    const std::string why = finish_zeta(X, plan, F, b, opt, res, fs_value >= 0 ? &fs_value : nullptr);
    if (why.empty()) break;
    res.reasons.push_back(why);
    if (std::getenv("DRZG_VERBOSE")) std::fprintf(stderr, "[drzg] escalate: %s\n", why.c_str());
    if (!escalate_plan(plan)) throw escalation_exhausted("precision ladder exhausted: " + why);
  }
  res.wall = now_s() - t0;
  return res;
}

}  // namespace drzg
