// The C ABI (include/drzg.h): marshalling between the reference's plain
// layouts and the engine, exceptions -> status codes + thread-local message.
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>
#include <string>

#include "../../include/drzg.h"
#include "kernels/count.cuh"
#include "kernels/linrec.cuh"
#include "kernels/tc_gemm.cuh"
#include "pipeline.cuh"

using namespace drzg;

namespace {

thread_local std::string g_err;

template <class F>
int guard_int(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}

template <class F>
char* guard_str(F&& f) {
  try {
    std::string s = f();
    char* out = (char*)std::malloc(s.size() + 1);
    std::memcpy(out, s.c_str(), s.size() + 1);
    g_err.clear();
    return out;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  } catch (...) {
    g_err = "unknown error";
    return nullptr;
  }
}

// StripePlan::make (linalg.hpp:35-58): smallest limb count with beta =
// p^ceil(M/limbs) <= 2^62 and limbs (beta-1)^2 <= 2^126
drzg_stripe_plan stripe_plan(u64 p, int M) {
  DRZG_REQUIRE(p >= 2 && M >= 1, "StripePlan: bad modulus");
  for (int limbs = 1; limbs <= 64; ++limbs) {
    int e = (M + limbs - 1) / limbs;
    Z pe = Z::pow(p, (u64)e);
    if (pe > Z::from_u64(u64(1) << 62)) continue;
    u64 beta = pe.to_u64();
    u128 prod = (u128)(beta - 1) * (beta - 1);
    u128 cap = u128(1) << 126;
    if (prod > cap / (u128)limbs) continue;
    drzg_stripe_plan pl{};
    pl.p = p;
    pl.M = M;
    pl.limbs = limbs;
    pl.limb_exp = e;
    pl.beta = beta;
    u128 s = cap / (prod * (u128)limbs);
    pl.stripe = s > (u128)((i64)1 << 40) ? ((i64)1 << 40) : (i64)s;
    return pl;
  }
  DRZG_REQUIRE(false, "StripePlan: no viable limb split");
  return {};
}

LinrecPlan linrec_plan(const drzg_stripe_plan* sp) {
  LinrecPlan lp;
  lp.p = sp->p;
  lp.M = sp->M;
  lp.limbs = sp->limbs;
  lp.limb_exp = sp->limb_exp;
  lp.beta = sp->beta;
  lp.top_mod = ipow(sp->p, sp->M - sp->limb_exp * (sp->limbs - 1));
  return lp;
}

std::string zjson(const std::vector<Z>& v) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << "\"" << v[i].str() << "\"";
  os << "]";
  return os.str();
}
template <class T>
std::string ijson(const std::vector<T>& v) {
  std::ostringstream os;
  os << "[";
  for (size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << v[i];
  os << "]";
  return os.str();
}
std::string plan_json(const PrecisionPlan& P) {
  std::ostringstream os;
  os << "{\"M\":" << P.M << ",\"A\":" << P.A << ",\"A_sharp\":" << P.A_sharp << ",\"b\":" << P.b
     << ",\"escalations\":" << P.escalations << ",\"r_m\":" << ijson(P.r_m) << ",\"N_m\":" << ijson(P.N_m)
     << ",\"s_m\":" << ijson(P.s_m) << "}";
  return os.str();
}
std::string frob_json_body(const FrobResult& fr) {
  std::ostringstream os;
  os.precision(9);
  os << "\"b\":" << fr.b << ",\"M\":" << fr.M << ",\"digits\":{\"q\":" << fr.q << ",\"Ld\":" << fr.Ld
     << "},\"nL\":" << fr.nL << ",\"side\":" << fr.side << ",\"terms\":" << fr.terms << ",\"groups\":" << fr.groups
     << ",\"matvecs\":" << fr.led.matvecs << ",\"startups\":" << fr.led.startups
     << ",\"combines\":" << fr.led.combines << ",\"computed\":" << ijson(fr.computed)
     << ",\"times\":{\"tables\":" << fr.t.tables << ",\"seeds\":" << fr.t.seeds << ",\"device\":" << fr.t.device
     << ",\"final\":" << fr.t.final << ",\"total\":" << fr.t.total << "}"
     << ",\"kernels\":{\"gemm_ms\":" << fr.clk.gemm_ms << ",\"carry_ms\":" << fr.clk.carry_ms
     << ",\"gather_ms\":" << fr.clk.gather_ms << ",\"epilogue_ms\":" << fr.clk.epi_ms << ",\"flush_ms\":" << fr.clk.flush_ms
     << ",\"other_ms\":" << fr.clk.other_ms << ",\"gemm_launches\":" << fr.clk.gemm_launches
     << ",\"gemm_macs\":" << fr.clk.gemm_macs << ",\"carry_launches\":" << fr.clk.carry_launches
     << ",\"carry_macs\":" << fr.clk.carry_macs << ",\"device_ms\":" << fr.clk.device_ms << ",\"peak_live_states\":" << fr.clk.peak_live << "}"
     << ",\"traffic\":{\"h2d_bytes\":" << g_traffic.h2d.load() << ",\"d2h_bytes\":" << g_traffic.d2h.load()
     << ",\"launches\":" << g_traffic.launches.load() << "}";
  return os.str();
}
std::string zeta_json_body(const ZetaOut& r) {
  std::ostringstream os;
  os.precision(9);
  os << "\"Q\":" << zjson(r.Q) << ",\"Q_alt\":" << zjson(r.Q_alt)
     << ",\"ambiguous\":" << (r.ambiguous ? "true" : "false") << ",\"plan\":" << plan_json(r.plan)
     << ",\"p_rank\":" << r.inv.p_rank << ",\"height\":\"" << r.inv.height << "\",\"domino\":\"" << r.inv.domino
     << "\",\"domino_any\":\"" << r.domino << "\",\"newton_height\":\"" << r.inv.newton_height
     << "\",\"fsplit\":" << (r.inv.fsplit_defined ? (r.inv.fsplit ? "true" : "false") : "null") << ",\"slopes\":[";
  for (size_t i = 0; i < r.np.slopes.size(); ++i)
    os << (i ? "," : "") << "[\"" << r.np.slopes[i].first.str() << "\"," << r.np.slopes[i].second << "]";
  os << "],\"counts\":[";
  for (size_t i = 0; i < r.counts.size(); ++i)
    os << (i ? "," : "") << "[" << r.counts[i].r << ",\"" << r.counts[i].from_zeta.str() << "\","
       << (r.counts[i].ok ? "true" : "false") << "]";
  os << "],\"escalations\":[";
  for (size_t i = 0; i < r.reasons.size(); ++i) os << (i ? "," : "") << "\"" << r.reasons[i] << "\"";
  os << "]";
  return os.str();
}
Policy policy_of(int p) {
  DRZG_REQUIRE(p >= 0 && p <= 2, "unknown policy");
  return (Policy)p;
}
PlanOverrides overrides(int r_uniform, int nm) {
  PlanOverrides ov;
  ov.r_uniform = r_uniform;
  if (nm > 0) ov.N_m = {nm};
  return ov;
}
std::vector<u64> coeff_vec(int n, int d, const uint64_t* coeffs) {
  size_t cnt = (size_t)mono_count(n + 1, d);
  return std::vector<u64>(coeffs, coeffs + cnt);
}

}  // namespace

namespace drzg {
void set_last_error(const std::string& s) { g_err = s; }
}  // namespace drzg

extern "C" {

const char* drzg_last_error(void) { return g_err.c_str(); }
void drzg_free(char* s) { std::free(s); }

int drzg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int drzg_stripe_plan_make(uint64_t p, int32_t M, drzg_stripe_plan* out) {
  return guard_int([&] { *out = stripe_plan(p, M); });
}

int drzg_linrec_eval_device(const drzg_stripe_plan* plan, int32_t side, const uint64_t* dA, const uint64_t* dB,
                            int64_t tmax, uint64_t* dw, int64_t* matvecs, void* stream, float* kernel_ms) {
  return guard_int([&] {
    linrec_device(linrec_plan(plan), side, dA, dB, tmax, dw, (cudaStream_t)stream, kernel_ms, nullptr);
    if (matvecs) *matvecs += tmax + 1;
  });
}

int drzg_linrec_eval(const drzg_stripe_plan* plan, int32_t side, const uint64_t* A, const uint64_t* B, int64_t tmax,
                     uint64_t* w, int64_t* matvecs) {
  return guard_int([&] {
    size_t nn = (size_t)plan->limbs * side * side, nv = (size_t)plan->limbs * side;
    DevBuf<uint64_t> dA, dB, dw;
    dA.alloc(nn);
    dB.alloc(nn);
    dw.alloc(nv);
    DRZG_CUDA(cudaMemcpy(dA.p, A, nn * 8, cudaMemcpyHostToDevice));
    DRZG_CUDA(cudaMemcpy(dB.p, B, nn * 8, cudaMemcpyHostToDevice));
    DRZG_CUDA(cudaMemcpy(dw.p, w, nv * 8, cudaMemcpyHostToDevice));
    linrec_device(linrec_plan(plan), side, dA.p, dB.p, tmax, dw.p, 0, nullptr, nullptr);
    DRZG_CUDA(cudaMemcpy(w, dw.p, nv * 8, cudaMemcpyDeviceToHost));
    if (matvecs) *matvecs += tmax + 1;
  });
}

int drzg_sparse_steps(const drzg_stripe_plan* plan, int32_t side, const int64_t* a_col_ptr, const int32_t* a_row_idx,
                      const uint64_t* a_digs, const int64_t* b_col_ptr, const int32_t* b_row_idx,
                      const uint64_t* b_digs, int64_t tmax, uint64_t* w, int64_t* matvecs) {
  return guard_int([&] {
    const int L = plan->limbs;
    // CSC (SparseOp) -> CSR on the host, once per call
    auto to_csr = [&](const int64_t* cp, const int32_t* ri, const uint64_t* dg, std::vector<int>& ptr,
                      std::vector<int>& col, std::vector<uint64_t>& val) {
      i64 nnz = cp[side];
      ptr.assign(side + 1, 0);
      for (i64 e = 0; e < nnz; ++e) ptr[ri[e] + 1]++;
      for (int i = 0; i < side; ++i) ptr[i + 1] += ptr[i];
      col.assign(nnz, 0);
      val.assign((size_t)nnz * L, 0);
      std::vector<int> fill(ptr.begin(), ptr.end() - 1);
      for (int j = 0; j < side; ++j)
        for (i64 e = cp[j]; e < cp[j + 1]; ++e) {
          int pos = fill[ri[e]]++;
          col[pos] = j;
          for (int t = 0; t < L; ++t) val[(size_t)pos * L + t] = dg[(size_t)e * L + t];
        }
    };
    std::vector<int> ap, ac, bp, bc;
    std::vector<uint64_t> av, bv;
    to_csr(a_col_ptr, a_row_idx, a_digs, ap, ac, av);
    to_csr(b_col_ptr, b_row_idx, b_digs, bp, bc, bv);
    DevBuf<int> dap, dac, dbp, dbc;
    DevBuf<uint64_t> dav, dbv, dw;
    dap.upload(ap, 0);
    dac.upload(ac, 0);
    dbp.upload(bp, 0);
    dbc.upload(bc, 0);
    dav.upload(av, 0);
    dbv.upload(bv, 0);
    std::vector<uint64_t> hw(w, w + (size_t)L * side);
    dw.upload(hw, 0);
    CsrPair csr{dap.p, dac.p, dav.p, dbp.p, dbc.p, dbv.p};
    linrec_device(linrec_plan(plan), side, nullptr, nullptr, tmax, dw.p, 0, nullptr, &csr);
    DRZG_CUDA(cudaMemcpy(w, dw.p, hw.size() * 8, cudaMemcpyDeviceToHost));
    if (matvecs) *matvecs += tmax + 1;
  });
}

char* drzg_reduce_chunk(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t M, int32_t* u,
                        int32_t pole, const int32_t* v, int64_t k, uint64_t* w, int32_t device) {
  return guard_str([&]() -> std::string {
    DRZG_CUDA(cudaSetDevice(device));
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    RuvTables T = build_tables(X, M, default_S(n, d));
    DRZG_REQUIRE(pole - k >= n, "reduce_chunk: chunk passes the floor");
    drzg_stripe_plan sp = stripe_plan(p, M);
    HostMod hm = HostMod::make(p, M);
    const int nv = n + 1, Ld = T.dp.Ld;
    // ModVec digits -> residues -> balanced base-q digit planes
    std::vector<i8> dig((size_t)Ld * T.side);
    std::vector<i8> tmp(Ld);
    Z beta = Z::from_u64(sp.beta);
    for (int g = 0; g < T.side; ++g) {
      Z val(0);
      for (int t = sp.limbs - 1; t >= 0; --t) val = val * beta + Z::from_u64(w[(size_t)t * T.side + g]);
      to_digits_z(val.mod(hm.mz), T.dp, tmp.data());
      for (int t = 0; t < Ld; ++t) dig[(size_t)t * T.side + g] = tmp[t];
    }
    Expo ue(nv), ve(nv);
    for (int i = 0; i < nv; ++i) ue[i] = u[i], ve[i] = v[i];
    cudaStream_t st;
    DRZG_CUDA(cudaStreamCreate(&st));
    Ledger led;
    {
      ReductionEngine eng(T, n, p, st);
      eng.chunk_batch({ue}, {(int)rank_of(ve)}, {k}, dig, led);
    }
    DRZG_CUDA(cudaStreamDestroy(st));
    std::vector<i64> s(Ld);
    for (int g = 0; g < T.side; ++g) {
      for (int t = 0; t < Ld; ++t) s[t] = dig[(size_t)t * T.side + g];
      Z val = from_digit_sums(s.data(), T.dp, hm.mz);
      for (int t = 0; t < sp.limbs; ++t) {
        Z q = Z::from_u64(sp.beta);
        Z r = val.mod(q);
        w[(size_t)t * T.side + g] = r.to_u64();
        val = (val - r).divexact(q);
      }
    }
    for (int i = 0; i < nv; ++i) u[i] -= (int)(k * v[i]);
    std::ostringstream os;
    os << "{\"side\":" << T.side << ",\"nL\":" << T.nL << ",\"pole\":" << pole - k << ",\"matvecs\":" << led.matvecs
       << ",\"startups\":" << led.startups << "}";
    return os.str();
  });
}

char* drzg_frobenius(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t policy, int32_t r_uniform,
                     int32_t nm_override, int32_t only_pole, const int32_t* columns, int32_t ncolumns,
                     int32_t device, int32_t profile) {
  return guard_str([&]() -> std::string {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    Policy pol = policy_of(policy);
    std::set<int> S = working_set_for(X, pol);
    Basis B = compute_basis(X);
    PrecisionPlan plan = choose_precision(p, n, d, overrides(r_uniform, nm_override));
    FrobOptions fo;
    fo.policy = pol;
    fo.overrides = overrides(r_uniform, nm_override);
    fo.only_pole = only_pole;
    fo.profile = profile != 0;
    if (columns)
      for (int i = 0; i < ncolumns; ++i) fo.columns.push_back(columns[i]);
    g_traffic.reset();
    FrobResult fr = frobenius_matrix(X, B, plan, S, fo, device);
    std::vector<Z> dres;
    if (!only_pole && fo.columns.empty())
      dres = berkowitz(fr.F, (int)fr.b, Z::pow(p, (u64)(plan.M + n)));
    std::ostringstream os;
    os << "{" << frob_json_body(fr) << ",\"plan\":" << plan_json(plan) << ",\"F\":" << zjson(fr.F)
       << ",\"charpoly\":" << zjson(dres) << "}";
    return os.str();
  });
}

char* drzg_zeta(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t policy, int32_t r_uniform,
                int32_t nm_override, int32_t verify_counts, int64_t count_budget, int32_t device, int32_t profile) {
  return guard_str([&]() -> std::string {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    ZetaOptions zo;
    zo.policy = policy_of(policy);
    zo.overrides = overrides(r_uniform, nm_override);
    zo.verify_counts = verify_counts != 0;
    if (count_budget > 0) zo.count_budget = count_budget;
    zo.profile = profile != 0;
    g_traffic.reset();
    ZetaOut r = run_zeta(X, zo, device);
    return "{" + zeta_json_body(r) + ",\"seconds\":" + std::to_string(r.wall) + ",\"frobenius\":{" +
           frob_json_body(r.last) + "}}";
  });
}

char* drzg_zeta_from_F(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t r_uniform,
                       int32_t nm_override, int32_t escalations, int32_t b, const char* const* F,
                       int32_t verify_counts, int64_t count_budget) {
  return guard_str([&]() -> std::string {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    ZetaOptions zo;
    zo.overrides = overrides(r_uniform, nm_override);
    zo.verify_counts = verify_counts != 0;
    if (count_budget > 0) zo.count_budget = count_budget;
    PrecisionPlan plan = choose_precision(p, n, d, zo.overrides);
    for (int e = 0; e < escalations; ++e) DRZG_REQUIRE(escalate_plan(plan), "zeta_from_F: no such escalation step");
    DRZG_REQUIRE(b == (int)plan.b, "zeta_from_F: F is not b x b for this plan");
    std::vector<Z> f((size_t)b * b);
    for (size_t i = 0; i < f.size(); ++i) f[i] = Z::from_str(F[i]);
    ZetaOut r;
    const std::string why = finish_zeta(X, plan, f, b, zo, r);
    if (!why.empty()) return "{\"status\":\"escalate\",\"reason\":\"" + why + "\",\"plan\":" + plan_json(plan) + "}";
    return "{\"status\":\"ok\"," + zeta_json_body(r) + "}";
  });
}

int drzg_random_hypersurface(uint64_t p, int32_t n, int32_t d, uint64_t seed, int32_t policy, int32_t fermat,
                              uint64_t* coeffs_out, int32_t* tries_out) {
  return guard_int([&] {
    const MonoList& tab = monos(n + 1, d);
    std::mt19937_64 rng(seed);
    int tries = 0;
    for (;;) {
      ++tries;
      DRZG_REQUIRE(tries < 100000, "random_hypersurface: no smooth draw");
      std::vector<u64> c(tab.size(), 0);
      if (fermat) {
        for (int i = 0; i <= n; ++i) {
          Expo e(n + 1);
          e[i] = d;
          c[(size_t)rank_of(e)] = 1;
        }
      } else {
        for (auto& x : c) x = rng() % p;
      }
      bool zero = true;
      for (auto x : c) zero = zero && x == 0;
      if (zero) continue;
      Hypersurface X = Hypersurface::make(p, n, d, c);
      bool ok = check_smooth(X, full_set(n + 1)) && check_smooth(X, working_set_for(X, policy_of(policy)));
      DRZG_REQUIRE(ok || !fermat, "random_hypersurface: Fermat hypersurface not smooth");
      if (!ok) continue;
      std::copy(c.begin(), c.end(), coeffs_out);
      if (tries_out) *tries_out = tries;
      return;
    }
  });
}

// brute-force #X(F_{p^r}) (reference count_points, oracle.hpp:190-245)
int drzg_count_points(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t r, int64_t budget,
                      int64_t* out) {
  return guard_int([&] {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    *out = count_points(X, r, budget);
  });
}

// the device enumeration (kernels/count.cu)
int drzg_count_points_device(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t r, int64_t budget,
                             int64_t* out) {
  return guard_int([&] {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    *out = count_points_device(X, r, budget);
  });
}

char* drzg_charpoly(uint64_t p, int32_t n, int32_t d, int32_t r_uniform, int32_t nm_override, int32_t b,
                    const char* const* F) {
  return guard_str([&]() -> std::string {
    PrecisionPlan plan = choose_precision(p, n, d, overrides(r_uniform, nm_override));
    std::vector<Z> f((size_t)b * b);
    for (size_t i = 0; i < f.size(); ++i) f[i] = Z::from_str(F[i]);
    auto dres = berkowitz(f, b, Z::pow(p, (u64)(plan.M + n)));
    Recovered rec = recover_Q(dres, plan);
    std::ostringstream os;
    os << "{\"charpoly\":" << zjson(dres) << ",\"status\":" << rec.status << ",\"candidates\":[";
    for (size_t i = 0; i < rec.candidates.size(); ++i) os << (i ? "," : "") << zjson(rec.candidates[i]);
    os << "]}";
    return os.str();
  });
}

}  // extern "C"

// test hook: raw int32 D = A . B^T through the tcgen05 kernel (host buffers)
extern "C" int drzg_test_tc_gemm(int32_t M, int32_t N, int32_t K, const int8_t* A, const int8_t* B, int32_t* D,
                                 int32_t a_unsigned) {
  return guard_int([&] {
    int ld = (K + 15) / 16 * 16;
    DevBuf<int8_t> dA, dB;
    DevBuf<int32_t> dD;
    std::vector<int8_t> ha((size_t)M * ld, 0), hb((size_t)N * ld, 0);
    for (int i = 0; i < M; ++i)
      for (int k = 0; k < K; ++k) ha[(size_t)i * ld + k] = A[(size_t)i * K + k];
    for (int i = 0; i < N; ++i)
      for (int k = 0; k < K; ++k) hb[(size_t)i * ld + k] = B[(size_t)i * K + k];
    dA.upload(ha, 0);
    dB.upload(hb, 0);
    dD.alloc((size_t)M * N);
    TcEpiArgs e;
    e.mode = (int)TcEpilogue::raw;
    e.a_unsigned = a_unsigned;
    e.M = M;
    e.N = N;
    e.out = dD.p;
    tc_gemm_i8(dA.p, M, ld, dB.p, N, ld, ld, e, 0);
    DRZG_CUDA(cudaDeviceSynchronize());
    DRZG_CUDA(cudaMemcpy(D, dD.p, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  });
}

// micro-benchmark hook: one Dixon digit (mode 1) or carry (mode 2) GEMM of
// nL x nL against `states` synthetic states with the engine's layouts;
// returns the mean CUDA-event milliseconds per launch
extern "C" int drzg_bench_tc_gemm(int32_t nL, int32_t states, int32_t mode, int32_t iters, float* ms_out) {
  return guard_int([&] {
    const int nLp = (nL + 63) / 64 * 64, Ld = 12;
    DevBuf<int8_t> A, IN, Y, Bg;
    DevBuf<int8_t> H;
    A.alloc((size_t)nLp * nLp);
    IN.alloc((size_t)states * nLp);
    Y.alloc((size_t)states * Ld * nLp);
    Bg.alloc((size_t)states * Ld * nLp);
    // state-contiguous layouts, pitch = states (multiple of 64)
    H.alloc((size_t)states * nLp);
    DRZG_CUDA(cudaMemset(A.p, 1, A.n));
    DRZG_CUDA(cudaMemset(IN.p, 1, IN.n));
    DRZG_CUDA(cudaMemset(Y.p, 0, Y.n));
    DRZG_CUDA(cudaMemset(Bg.p, 0, Bg.n));
    DRZG_CUDA(cudaMemset(H.p, 0, H.n));
    TcEpiArgs e;
    e.mode = mode;
    e.M = nL;
    e.N = states;
    e.q = 49;
    e.fq = FastQ::make(49);
    e.Ld = Ld;
    e.k = 3;
    e.nLp = nLp;
    e.nL = nL;
    e.Y = Y.p;
    e.Bg = Bg.p;
    e.H = H.p;
    e.IN = IN.p;
    e.a_unsigned = mode == 2;
    e.b_mn = 1;
    e.P = states;
    auto run = [&] {
      if (mode == 2)
        tc_gemm_i8(A.p, nLp, nLp, Y.p + (size_t)3 * nLp * states, states, states, nLp, e, 0);
      else
        tc_gemm_i8(A.p, nLp, nLp, IN.p, states, states, nLp, e, 0);
    };
    run();
    cudaEvent_t e0, e1;
    DRZG_CUDA(cudaEventCreate(&e0));
    DRZG_CUDA(cudaEventCreate(&e1));
    DRZG_CUDA(cudaEventRecord(e0, 0));
    for (int i = 0; i < iters; ++i) run();
    DRZG_CUDA(cudaEventRecord(e1, 0));
    DRZG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    DRZG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

// test hook, MN-major B: D = A . B^T with B stored K x Npad (states contiguous)
extern "C" int drzg_test_tc_gemm_mn(int32_t M, int32_t N, int32_t K, const int8_t* A, const int8_t* B, int32_t* D,
                                    int32_t a_unsigned) {
  return guard_int([&] {
    int ld = (K + 15) / 16 * 16;
    int P = (N + 63) / 64 * 64;
    DevBuf<int8_t> dA, dB;
    DevBuf<int32_t> dD;
    std::vector<int8_t> ha((size_t)M * ld, 0), hb((size_t)K * P, 0);
    for (int i = 0; i < M; ++i)
      for (int k = 0; k < K; ++k) ha[(size_t)i * ld + k] = A[(size_t)i * K + k];
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) hb[(size_t)k * P + n] = B[(size_t)n * K + k];
    dA.upload(ha, 0);
    dB.upload(hb, 0);
    dD.alloc((size_t)M * N);
    TcEpiArgs e;
    e.mode = (int)TcEpilogue::raw;
    e.a_unsigned = a_unsigned;
    e.b_mn = 1;
    e.P = P;
    e.M = M;
    e.N = N;
    e.out = dD.p;
    tc_gemm_i8(dA.p, M, ld, dB.p, N, P, K, e, 0);
    DRZG_CUDA(cudaDeviceSynchronize());
    DRZG_CUDA(cudaMemcpy(D, dD.p, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  });
}

// test hook: host vs device pivot scan (rows x cols over F_p) and inverse mod
// q (n x n, made invertible by construction); *mismatches = differing entries
extern "C" int drzg_test_setup(uint64_t p, uint64_t q, int32_t n, int32_t cols, uint64_t seed, int64_t* mismatches) {
  return guard_int([&] {
    std::mt19937_64 rng(seed);
    std::vector<u32> m((size_t)n * cols);
    for (auto& x : m) x = (u32)(rng() % p);
    auto host = pivot_scan_fp(p, n, cols, m);
    auto devp = pivot_scan_device(p, n, cols, m);
    i64 bad = 0;
    for (int r = 0; r < n; ++r) bad += host.pivot_col_of_row[r] != devp[r];
    // unit lower x unit upper (mod q) is invertible
    std::vector<u32> a((size_t)n * n, 0);
    {
      std::vector<u64> Lm((size_t)n * n, 0), Um((size_t)n * n, 0);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          if (j < i) Lm[(size_t)i * n + j] = rng() % q;
          if (j > i) Um[(size_t)i * n + j] = rng() % q;
        }
      for (int i = 0; i < n; ++i) Lm[(size_t)i * n + i] = Um[(size_t)i * n + i] = 1 + rng() % (p - 1);
      for (int i = 0; i < n; ++i)
        for (int k = 0; k <= i; ++k) {
          u64 l = Lm[(size_t)i * n + k];
          if (!l) continue;
          for (int j = k; j < n; ++j) a[(size_t)i * n + j] = (u32)((a[(size_t)i * n + j] + l * Um[(size_t)k * n + j]) % q);
        }
    }
    auto hi = inverse_mod_q(p, q, n, a);
    auto di = inverse_mod_q_device(p, q, n, a);
    for (size_t i = 0; i < hi.size(); ++i) bad += hi[i] != di[i];
    *mismatches = bad;
  });
}

// test hook: build the reduction tables with the host and the device setup
// and count differing pivot choices / inverse entries
extern "C" int drzg_test_tables(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t M, int64_t* diff) {
  return guard_int([&] {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    setenv("DRZG_SETUP", "host", 1);
    RuvTables A = build_tables(X, M, default_S(n, d));
    setenv("DRZG_SETUP", "device", 1);
    RuvTables B = build_tables(X, M, default_S(n, d));
    unsetenv("DRZG_SETUP");
    i64 bad = 0;
    for (size_t i = 0; i < A.sol_row.size(); ++i) bad += A.sol_row[i] != B.sol_row[i] || A.sol_i[i] != B.sol_i[i];
    for (size_t i = 0; i < A.sys.Cq.size(); ++i) bad += A.sys.Cq[i] != B.sys.Cq[i];
    bad += A.sys.col != B.sys.col || A.sys.val != B.sys.val;
    *diff = bad;
  });
}

extern "C" int drzg_test_final_levels(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t M, int64_t* diff) {
  return guard_int([&] {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    Basis B = compute_basis(X);
    DigitPlan dp = DigitPlan::make(p, M);
    HostMod hm = HostMod::make(p, M);
    setenv("DRZG_SETUP", "host", 1);
    FinalReducer fa(X, B, dp, hm);
    fa.prepare();
    setenv("DRZG_SETUP", "device", 1);
    FinalReducer fb(X, B, dp, hm);
    fb.prepare();
    unsetenv("DRZG_SETUP");
    i64 bad = 0;
    for (int m = 1; m <= n; ++m) {
      bad += fa.level_pivots(m) != fb.level_pivots(m) ? 1000000 : 0;
      const auto& a = fa.level_inverse(m);
      const auto& b = fb.level_inverse(m);
      if (a.size() != b.size()) bad += 1000;
      else
        for (size_t i = 0; i < a.size(); ++i) bad += a[i] != b[i];
    }
    *diff = bad;
  });
}

namespace drzg {
std::pair<long long, long long> debug_order_blocks(const RuvTables& T);
}
// Fedder's F-splitting criterion as run_zeta's invariants report it (host
// only): 1 / 0, or -1 where it is undefined (d > n + 1); reference
// zeta.hpp:336-350
extern "C" int drzg_fsplit(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t* out) {
  return guard_int([&] {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    *out = d > X.nv() ? -1 : (fedder_is_fsplit(X) ? 1 : 0);
  });
}

// debug hook: nonzero 128 x 128 Jp blocks of the carry order, without (out[0])
// and with (out[1]) the T_x grouping of solution indices
extern "C" int drzg_debug_order(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t M, int64_t* out) {
  return guard_int([&] {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    setenv("DRZG_SETUP", "host", 1);
    setenv("DRZG_DEBUG_NO_INVERSE", "1", 1);
    RuvTables T = build_tables(X, M, default_S(n, d));
    unsetenv("DRZG_SETUP");
    unsetenv("DRZG_DEBUG_NO_INVERSE");
    auto b = debug_order_blocks(T);
    out[0] = b.first;
    out[1] = b.second;
  });
}

// debug hook: the Dixon system's structure (Jp CSR, rows Homog_L in grevlex
// rank, columns = solution indices) and the generator of every solution
// index, written as int32 arrays to `path`:
//   nL, nnz, rowptr[nL+1], col[nnz], val[nnz], sol_i[nL], sol_row[nL], sol_mu[nL]
extern "C" int drzg_debug_system(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t M,
                                 const char* path) {
  return guard_int([&] {
    Hypersurface X = Hypersurface::make(p, n, d, coeff_vec(n, d, coeffs));
    setenv("DRZG_SETUP", "host", 1);
    setenv("DRZG_DEBUG_NO_INVERSE", "1", 1);
    RuvTables T = build_tables(X, M, default_S(n, d));
    unsetenv("DRZG_SETUP");
    unsetenv("DRZG_DEBUG_NO_INVERSE");
    FILE* f = std::fopen(path, "wb");
    DRZG_REQUIRE(f != nullptr, "debug_system: cannot open output");
    int32_t hdr[2] = {T.nL, (int32_t)T.sys.col.size()};
    std::fwrite(hdr, 4, 2, f);
    std::fwrite(T.sys.rowptr.data(), 4, T.sys.rowptr.size(), f);
    std::fwrite(T.sys.col.data(), 4, T.sys.col.size(), f);
    std::fwrite(T.sys.val.data(), 4, T.sys.val.size(), f);
    std::fwrite(T.sol_i.data(), 4, T.sol_i.size(), f);
    std::fwrite(T.sol_row.data(), 4, T.sol_row.size(), f);
    std::fwrite(T.sol_mu.data(), 4, T.sol_mu.size(), f);
    std::fclose(f);
  });
}
