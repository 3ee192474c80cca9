// The states-level C ABI (include/drzg.h, "reduction-policy interface"):
// a device context standing in for the reference's (RuvContext, PepStoreBase)
// pair, GameStates resident in its HBM slot pool, and the reference's
// reduce_chunk / combine_states / run_policy / floor_to_numerator on them.
// Residues cross the boundary in the reference's ModVec layout (limbs planes
// of base-beta digits, linalg.hpp:94-117); on the device they are balanced
// base-q digit planes.
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>

#include "../../include/drzg.h"
#include "pipeline.cuh"

#include "states_ctx.hpp"

using namespace drzg;

namespace drzg {
void set_last_error(const std::string& s);  // capi.cu: the message drzg_last_error() returns
}

namespace {
template <class F>
int sguard(F&& f) {
  try {
    f();
    set_last_error("");
    return 0;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 1;
  } catch (...) {
    set_last_error("unknown error");
    return 1;
  }
}

drzg_stripe_plan plan_of(u64 p, int M) {
  drzg_stripe_plan sp{};
  DRZG_REQUIRE(drzg_stripe_plan_make(p, M, &sp) == 0, "StripePlan: no viable limb split");
  return sp;
}

// ModVec (limbs planes, base beta) of length len -> residues -> Ld x len balanced digits
std::vector<i8> modvec_to_digits(const StatesCtx& C, const uint64_t* w, int len) {
  const DigitPlan& dp = C.T.dp;
  std::vector<i8> out((size_t)dp.Ld * len), tmp(dp.Ld);
  const Z beta = Z::from_u64(C.sp.beta);
  for (int g = 0; g < len; ++g) {
    Z val(0);
    for (int t = C.sp.limbs - 1; t >= 0; --t) val = val * beta + Z::from_u64(w[(size_t)t * len + g]);
    to_digits_z(val.mod(C.hm.mz), dp, tmp.data());
    for (int t = 0; t < dp.Ld; ++t) out[(size_t)t * len + g] = tmp[t];
  }
  return out;
}

void residue_to_modvec(const StatesCtx& C, Z val, uint64_t* w, int len, int g) {
  const Z beta = Z::from_u64(C.sp.beta);
  for (int t = 0; t < C.sp.limbs; ++t) {
    Z r = val.mod(beta);
    w[(size_t)t * len + g] = r.to_u64();
    val = (val - r).divexact(beta);
  }
}

StatesCtx& ctx_of(void* h) {
  DRZG_REQUIRE(h != nullptr, "drzg: null context");
  return *static_cast<StatesCtx*>(h);
}

ReductionEngine::Live& state_of(StatesCtx& C, int id) {
  DRZG_REQUIRE(id >= 0 && id < (int)C.states.size() && C.alive[id], "drzg: unknown or freed state id");
  return C.states[id];
}

int new_id(StatesCtx& C, const ReductionEngine::Live& s) {
  C.states.push_back(s);
  C.alive.push_back(1);
  return (int)C.states.size() - 1;
}
}  // namespace

extern "C" {

drzg_ctx* drzg_ctx_create(uint64_t p, int32_t n, int32_t d, const uint64_t* coeffs, int32_t M, int32_t policy,
                          int32_t device) {
  StatesCtx* out = nullptr;
  int rc = sguard([&] {
    DRZG_REQUIRE(policy >= 0 && policy <= 2, "unknown policy");
    auto C = std::make_unique<StatesCtx>();
    const size_t cnt = (size_t)mono_count(n + 1, d);
    C->X = Hypersurface::make(p, n, d, std::vector<u64>(coeffs, coeffs + cnt));
    C->M = M;
    C->policy = (Policy)policy;
    C->device = device;
    std::set<int> S = working_set_for(C->X, C->policy);
    DRZG_REQUIRE(check_smooth(C->X, S), "RuvContext: input not smooth for the working set");
    C->T = build_tables(C->X, M, S);
    C->sp = plan_of(p, M);
    C->hm = HostMod::make(p, M);
    DRZG_CUDA(cudaSetDevice(device));
    DRZG_CUDA(cudaStreamCreateWithFlags(&C->st, cudaStreamNonBlocking));
    C->eng = std::make_unique<ReductionEngine>(C->T, n, p, C->st);
    out = C.release();
  });
  if (rc) return nullptr;
  return reinterpret_cast<drzg_ctx*>(out);
}

void drzg_ctx_free(drzg_ctx* h) { delete reinterpret_cast<StatesCtx*>(h); }

int drzg_ctx_info(drzg_ctx* h, int32_t* side, int32_t* floor_len, drzg_stripe_plan* plan, int32_t* digit_base,
                  int32_t* digit_planes) {
  return sguard([&] {
    StatesCtx& C = ctx_of(h);
    if (side) *side = C.T.side;
    if (floor_len) *floor_len = C.eng->floor_size();
    if (plan) *plan = C.sp;
    if (digit_base) *digit_base = C.T.dp.q;
    if (digit_planes) *digit_planes = C.T.dp.Ld;
  });
}

int drzg_states_seed(drzg_ctx* h, int32_t count, const int32_t* u, const int32_t* pole, const uint64_t* w,
                     int32_t* ids_out) {
  return sguard([&] {
    StatesCtx& C = ctx_of(h);
    std::lock_guard<std::mutex> lk(C.mu);
    DRZG_CUDA(cudaSetDevice(C.device));
    const int nv = C.T.nv, side = C.T.side, Ld = C.T.dp.Ld;
    const size_t wlen = (size_t)C.sp.limbs * side;
    std::vector<int> eptr{0}, eg;
    std::vector<i8> ed;
    for (int i = 0; i < count; ++i) {
      std::vector<i8> dig = modvec_to_digits(C, w + (size_t)i * wlen, side);
      for (int g = 0; g < side; ++g) {
        bool nz = false;
        for (int t = 0; t < Ld; ++t) nz |= dig[(size_t)t * side + g] != 0;
        if (!nz) continue;
        eg.push_back(g);
        for (int t = 0; t < Ld; ++t) ed.push_back(dig[(size_t)t * side + g]);
      }
      eptr.push_back((int)eg.size());
    }
    std::vector<int> slots = C.eng->seed_states(eptr, eg, ed);
    for (int i = 0; i < count; ++i) {
      ReductionEngine::Live s;
      s.u = Expo(nv);
      for (int j = 0; j < nv; ++j) s.u[j] = u[(size_t)i * nv + j];
      s.pole = pole[i];
      s.slot = slots[i];
      ids_out[i] = new_id(C, s);
    }
  });
}

int drzg_states_read(drzg_ctx* h, int32_t count, const int32_t* ids, int32_t* u_out, int32_t* pole_out,
                     uint64_t* w_out) {
  return sguard([&] {
    StatesCtx& C = ctx_of(h);
    std::lock_guard<std::mutex> lk(C.mu);
    DRZG_CUDA(cudaSetDevice(C.device));
    const int nv = C.T.nv, side = C.T.side, Ld = C.T.dp.Ld;
    std::vector<int> slots;
    for (int i = 0; i < count; ++i) {
      const auto& s = state_of(C, ids[i]);
      slots.push_back(s.slot);
      if (u_out)
        for (int j = 0; j < nv; ++j) u_out[(size_t)i * nv + j] = s.u[j];
      if (pole_out) pole_out[i] = s.pole;
    }
    if (!w_out) return;
    std::vector<i8> dig = C.eng->read_states(slots);
    const size_t wlen = (size_t)C.sp.limbs * side;
    std::vector<i64> sums(Ld);
    for (int i = 0; i < count; ++i)
      for (int g = 0; g < side; ++g) {
        for (int t = 0; t < Ld; ++t) sums[t] = dig[((size_t)i * Ld + t) * side + g];
        residue_to_modvec(C, from_digit_sums(sums.data(), C.T.dp, C.hm.mz), w_out + (size_t)i * wlen, side, g);
      }
  });
}

int drzg_states_free(drzg_ctx* h, int32_t count, const int32_t* ids) {
  return sguard([&] {
    StatesCtx& C = ctx_of(h);
    std::lock_guard<std::mutex> lk(C.mu);
    std::vector<int> slots;
    for (int i = 0; i < count; ++i) {
      slots.push_back(state_of(C, ids[i]).slot);
      C.alive[ids[i]] = 0;
    }
    C.eng->release_slots(slots);
  });
}

int drzg_step_batch(drzg_ctx* h, int32_t count, const int32_t* ids, const int32_t* v, const int64_t* k,
                    int64_t* ledger) {
  return sguard([&] {
    StatesCtx& C = ctx_of(h);
    std::lock_guard<std::mutex> lk(C.mu);
    DRZG_CUDA(cudaSetDevice(C.device));
    const int nv = C.T.nv;
    std::vector<ReductionEngine::Live*> sts;
    std::vector<int> vd;
    std::vector<i64> kk;
    for (int i = 0; i < count; ++i) {
      sts.push_back(&state_of(C, ids[i]));
      Expo ve(nv);
      for (int j = 0; j < nv; ++j) ve[j] = v[(size_t)i * nv + j];
      DRZG_REQUIRE(ve.nonneg() && ve.total() == C.T.d, "reduce_chunk: illegal move");
      vd.push_back((int)rank_of(ve));
      kk.push_back(k[i]);
    }
    Ledger led;
    C.eng->step_states(sts, vd, kk, led);
    if (ledger) ledger[0] += led.matvecs, ledger[1] += led.startups, ledger[2] += led.combines;
  });
}

int drzg_states_combine(drzg_ctx* h, int32_t count, const int32_t* ids, int32_t* ids_out, int32_t* count_out,
                        int64_t* ledger) {
  return sguard([&] {
    StatesCtx& C = ctx_of(h);
    std::lock_guard<std::mutex> lk(C.mu);
    DRZG_CUDA(cudaSetDevice(C.device));
    std::vector<ReductionEngine::Live> sts;
    std::vector<int> id_of_slot_order;
    for (int i = 0; i < count; ++i) {
      sts.push_back(state_of(C, ids[i]));
      sts.back().col = 0;
    }
    std::map<int, int> id_by_slot;
    for (int i = 0; i < count; ++i) id_by_slot[C.states[ids[i]].slot] = ids[i];
    Ledger led;
    C.eng->combine_live(sts, led);
    std::set<int> kept;
    int m = 0;
    for (auto& s : sts) {
      const int id = id_by_slot.at(s.slot);
      kept.insert(id);
      ids_out[m++] = id;
    }
    for (int i = 0; i < count; ++i)
      if (!kept.count(ids[i])) C.alive[ids[i]] = 0;  // merged into an earlier state (its slot is freed)
    *count_out = m;
    if (ledger) ledger[0] += led.matvecs, ledger[1] += led.startups, ledger[2] += led.combines;
  });
}

int drzg_run_policy(drzg_ctx* h, int32_t count, const int32_t* ids, int32_t policy, int32_t* ids_out,
                    int32_t* count_out, int64_t* ledger) {
  return sguard([&] {
    StatesCtx& C = ctx_of(h);
    std::lock_guard<std::mutex> lk(C.mu);
    DRZG_CUDA(cudaSetDevice(C.device));
    DRZG_REQUIRE(policy >= 0 && policy <= 2, "unknown policy");
    std::vector<ReductionEngine::Live> sts;
    std::map<int, int> id_by_slot;
    for (int i = 0; i < count; ++i) {
      sts.push_back(state_of(C, ids[i]));
      sts.back().col = 0;
      id_by_slot[sts.back().slot] = ids[i];
    }
    Ledger led;
    C.eng->run_policy_live(sts, (Policy)policy, led);
    std::set<int> kept;
    int m = 0;
    for (auto& s : sts) {
      const int id = id_by_slot.at(s.slot);
      C.states[id].u = s.u;
      C.states[id].pole = s.pole;
      kept.insert(id);
      ids_out[m++] = id;
    }
    for (int i = 0; i < count; ++i)
      if (!kept.count(ids[i])) C.alive[ids[i]] = 0;
    *count_out = m;
    if (ledger) ledger[0] += led.matvecs, ledger[1] += led.startups, ledger[2] += led.combines;
  });
}

int drzg_floor_accumulate(drzg_ctx* h, int32_t count, const int32_t* ids, uint64_t* g) {
  return sguard([&] {
    StatesCtx& C = ctx_of(h);
    std::lock_guard<std::mutex> lk(C.mu);
    DRZG_CUDA(cudaSetDevice(C.device));
    const int Ld = C.T.dp.Ld, gs = C.eng->floor_size();
    std::vector<ReductionEngine::Live> sts;
    for (int i = 0; i < count; ++i) {
      sts.push_back(state_of(C, ids[i]));
      sts.back().col = 0;
    }
    DevBuf<long long> dG;
    dG.alloc((size_t)Ld * gs, C.st);
    DRZG_CUDA(cudaMemsetAsync(dG.p, 0, dG.n * sizeof(long long), C.st));
    C.eng->floor_accumulate(sts, dG.p, 1);
    std::vector<long long> hG(dG.n);
    DRZG_CUDA(cudaMemcpyAsync(hG.data(), dG.p, dG.n * sizeof(long long), cudaMemcpyDeviceToHost, C.st));
    DRZG_CUDA(cudaStreamSynchronize(C.st));
    const Z beta = Z::from_u64(C.sp.beta);
    std::vector<i64> sums(Ld);
    for (int r = 0; r < gs; ++r) {
      for (int t = 0; t < Ld; ++t) sums[t] = hG[(size_t)t * gs + r];
      Z add = from_digit_sums(sums.data(), C.T.dp, C.hm.mz);
      Z cur(0);
      for (int t = C.sp.limbs - 1; t >= 0; --t) cur = cur * beta + Z::from_u64(g[(size_t)t * gs + r]);
      residue_to_modvec(C, (cur + add).mod(C.hm.mz), g, gs, r);
    }
  });
}

}  // extern "C"
