// The PEP (precomputed operator family) store behind the C ABI: the
// reference's PepStoreBase::get / stats (reduction.hpp:143-147) with the
// eager / lazy / lru:N / lfuda:N backings of make_pep_store (pep.hpp:15-209).
//
// An entry is the reference's PepEntry for one move vector v (reduction.hpp:
// 121-137): the n+2 matrices A_0..A_n, A_{n+1} with R_{x,v} = sum_i x_i A_i +
// A_{n+1}, in ModMatrix plane layout.  The engine never needs them (its step is
// T_x(Jp^-1 P_v w)), so they are built on demand for callers that
// keep the reference's PEP + eval_to_linear + linrec_eval route: column g of
// every matrix comes from y = Jp^-1 e_j with j = rank(v + g - x^S), solved for
// all g at once on the device (ReductionEngine::solve_units), then scattered
// exactly as build_ruv does (reduction.hpp:253-297).
#include <condition_variable>
#include <cstring>
#include <functional>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/drzg.h"
#include "pipeline.cuh"
#include "states_ctx.hpp"

namespace drzg {
void set_last_error(const std::string& s);

struct PepEntryHost {
  int nmat = 0, limbs = 0, side = 0;
  std::vector<uint64_t> planes;  // nmat x limbs x side x side, row-major
  i64 nnz = 0;
  Expo v;
};
using PepPtr = std::shared_ptr<const PepEntryHost>;

// build_ruv(C, v) from the device solves
PepPtr build_entry(StatesCtx& C, const Expo& v) {
  const RuvTables& T = C.T;
  const int nv = T.nv, side = T.side, Ld = T.dp.Ld, nmat = nv + 1, limbs = C.sp.limbs;
  DRZG_REQUIRE(v.nv == nv && v.nonneg() && v.total() == T.d, "pep: bad move vector");
  const auto& sm = monos(nv, T.D).mons;
  std::vector<int> jrow(side, -1), rows;
  std::unordered_map<int, int> col_of;
  for (int g = 0; g < side; ++g) {
    Expo rhs = v + sm[g] - T.sexp;
    if (!rhs.nonneg()) continue;  // x^S does not divide x^v g: zero column
    const int j = (int)rank_of(rhs);
    auto it = col_of.find(j);
    if (it == col_of.end()) {
      it = col_of.emplace(j, (int)rows.size()).first;
      rows.push_back(j);
    }
    jrow[g] = it->second;
  }
  std::vector<i8> Y;
  {
    std::lock_guard<std::mutex> lk(C.mu);
    DRZG_CUDA(cudaSetDevice(C.device));
    Y = C.eng->solve_units(rows);
  }
  auto E = std::make_shared<PepEntryHost>();
  E->nmat = nmat;
  E->limbs = limbs;
  E->side = side;
  E->v = v;
  E->planes.assign((size_t)nmat * limbs * side * side, 0);
  const HostMod& hm = C.hm;
  const u64 beta = C.sp.beta;
  const int q = T.dp.q;
  // residue of a solution coordinate from its balanced digits
  auto residue128 = [&](const i8* dig) {
    i128 acc = 0;
    for (int k = Ld - 1; k >= 0; --k) acc = acc * q + dig[k];
    i128 m = (i128)hm.m128;
    acc %= m;
    if (acc < 0) acc += m;
    return (u128)acc;
  };
  auto put = [&](int t, int row, int g, const Z& val) {
    Z x = val;
    for (int l = 0; l < limbs; ++l) {
      Z r = x.mod(Z::from_u64(beta));
      E->planes[(((size_t)t * limbs + l) * side + row) * side + g] = r.to_u64();
      x = (x - r).divexact(Z::from_u64(beta));
    }
  };
  // per column g: A_i[row(r)] += y_r, A_{n+1}[row(r)] += mu_i y_r (both at
  // sol_row[r]: reduction.hpp:264-285 puts them on the same side row)
  std::vector<std::vector<std::pair<int, int>>> by_row(side);  // row -> (r, i)
  for (int r = 0; r < T.nL; ++r) by_row[T.sol_row[r]].push_back({r, T.sol_i[r]});
  std::vector<i8> dig(Ld);
  for (int g = 0; g < side; ++g) {
    if (jrow[g] < 0) continue;
    const i8* yc = Y.data() + (size_t)jrow[g] * Ld * T.nL;
    for (int row = 0; row < side; ++row) {
      if (by_row[row].empty()) continue;
      if (!hm.wide) {
        std::vector<u128> acc(nmat, 0);
        std::vector<char> hit(nmat, 0);
        for (auto [r, i] : by_row[row]) {
          for (int k = 0; k < Ld; ++k) dig[k] = yc[(size_t)k * T.nL + r];
          const u128 y = residue128(dig.data());
          if (!y) continue;
          acc[i] = (acc[i] + y) % hm.m128;
          hit[i] = 1;
          if (T.sol_mu[r] > 0) {
            acc[nv] = (acc[nv] + mulm128(y, (u128)T.sol_mu[r], hm.m128)) % hm.m128;
            hit[nv] = 1;
          }
        }
        for (int t = 0; t < nmat; ++t)
          if (hit[t] && acc[t]) {
            ++E->nnz;
            u128 x = acc[t];
            for (int l = 0; l < limbs; ++l) {
              E->planes[(((size_t)t * limbs + l) * side + row) * side + g] = (uint64_t)(x % beta);
              x /= beta;
            }
          }
      } else {
        std::vector<Z> acc(nmat, Z(0));
        std::vector<char> hit(nmat, 0);
        for (auto [r, i] : by_row[row]) {
          std::vector<i64> s(Ld);
          for (int k = 0; k < Ld; ++k) s[k] = yc[(size_t)k * T.nL + r];
          const Z y = from_digit_sums(s.data(), T.dp, hm.mz);
          if (y == Z(0)) continue;
          acc[i] = (acc[i] + y).mod(hm.mz);
          hit[i] = 1;
          if (T.sol_mu[r] > 0) {
            acc[nv] = (acc[nv] + y * Z((long)T.sol_mu[r])).mod(hm.mz);
            hit[nv] = 1;
          }
        }
        for (int t = 0; t < nmat; ++t)
          if (hit[t] && !(acc[t] == Z(0))) {
            ++E->nnz;
            put(t, row, g, acc[t]);
          }
      }
    }
  }
  return E;
}

// The backings.  A slot is resident or being built by exactly one caller; the
// others wait for it (pep.hpp:55-81).  Held entries are shared, so an eviction
// never invalidates one in use.
class PepStore {
 public:
  using Builder = std::function<PepPtr(const Expo&)>;
  PepStore(Builder b, const std::string& spec, int nv, int d) : build_(std::move(b)) {
    const auto colon = spec.find(':');
    kind_ = spec.substr(0, colon);
    if (colon != std::string::npos) {
      const std::string num = spec.substr(colon + 1);
      DRZG_REQUIRE(!num.empty() && num.find_first_not_of("0123456789") == std::string::npos,
                   "pep spec: bad capacity");
      cap_ = std::stoll(num);
    }
    DRZG_REQUIRE(kind_ == "eager" || kind_ == "lazy" || kind_ == "lru" || kind_ == "lfuda",
                 "pep spec: unknown backing");
    if (kind_ == "lru" || kind_ == "lfuda") DRZG_REQUIRE(cap_ >= 1, kind_ + ": capacity must be positive");
    if (kind_ == "eager")
      for (const auto& v : monos(nv, d).mons) slots_[key(v)].entry = build_(v);
  }

  PepPtr get(const Expo& v) {
    const std::string k = key(v);
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      auto it = slots_.find(k);
      if (it != slots_.end() && it->second.entry) {
        ++hits_;
        used(k);
        return it->second.entry;
      }
      if (it != slots_.end() && it->second.building) {
        cv_.wait(lk);
        continue;
      }
      DRZG_REQUIRE(kind_ != "eager", "eager store: unknown move vector");
      slots_[k].building = true;
      ++misses_;
      lk.unlock();
      PepPtr e;
      try {
        e = build_(v);
      } catch (...) {
        lk.lock();
        slots_.erase(k);
        cv_.notify_all();
        throw;
      }
      lk.lock();
      Slot& s = slots_[k];
      s.entry = e;
      s.building = false;
      admitted(k);
      cv_.notify_all();
      return e;
    }
  }
  void stats(i64* h, i64* m, i64* e) {
    std::lock_guard<std::mutex> lk(mu_);
    *h = hits_;
    *m = misses_;
    *e = evictions_;
  }

 private:
  struct Slot {
    PepPtr entry;
    bool building = false;
  };
  static std::string key(const Expo& v) { return std::string((const char*)v.e, sizeof(int) * v.nv); }
  void drop(const std::string& k) {
    slots_.erase(k);
    ++evictions_;
  }
  // a resident key was used again
  void used(const std::string& k) {
    if (kind_ == "lru") {
      auto w = lru_pos_.find(k);
      if (w != lru_pos_.end()) lru_.splice(lru_.begin(), lru_, w->second);
    } else if (kind_ == "lfuda") {
      auto w = lf_.find(k);
      if (w != lf_.end()) w->second.second = age_ + ++w->second.first;  // priority = age + uses
    }
  }
  // a key became resident: evict down to capacity
  void admitted(const std::string& k) {
    if (kind_ == "lru") {
      lru_.push_front(k);
      lru_pos_[k] = lru_.begin();
      while ((i64)lru_.size() > cap_) {
        const std::string victim = lru_.back();
        lru_.pop_back();
        lru_pos_.erase(victim);
        drop(victim);
      }
    } else if (kind_ == "lfuda") {
      lf_[k] = {1, age_ + 1};
      while ((i64)lf_.size() > cap_) {
        // least priority goes (ties: any); the age floor rises to it
        auto victim = lf_.end();
        for (auto it = lf_.begin(); it != lf_.end(); ++it)
          if (it->first != k && (victim == lf_.end() || it->second.second < victim->second.second)) victim = it;
        age_ = std::max(age_, victim->second.second);
        const std::string vk = victim->first;
        lf_.erase(victim);
        drop(vk);
      }
    }
  }

  Builder build_;
  std::string kind_;
  i64 cap_ = 0;
  std::mutex mu_;
  std::condition_variable cv_;
  std::unordered_map<std::string, Slot> slots_;
  i64 hits_ = 0, misses_ = 0, evictions_ = 0;
  std::list<std::string> lru_;
  std::unordered_map<std::string, std::list<std::string>::iterator> lru_pos_;
  std::unordered_map<std::string, std::pair<i64, i64>> lf_;  // key -> (uses, priority)
  i64 age_ = 0;
};

}  // namespace drzg

using namespace drzg;

namespace {
template <class F>
int pguard(F&& f) {
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
struct StoreHandle {
  std::unique_ptr<PepStore> store;
  StatesCtx* ctx = nullptr;
  int nv = 0, limbs = 1, side = 0;
};
}  // namespace

extern "C" {

drzg_pep_store* drzg_pep_store_create(drzg_ctx* ctx, const char* spec) {
  StoreHandle* out = nullptr;
  pguard([&] {
    DRZG_REQUIRE(ctx && spec, "pep: null argument");
    StatesCtx* C = reinterpret_cast<StatesCtx*>(ctx);
    auto h = std::make_unique<StoreHandle>();
    h->ctx = C;
    h->nv = C->T.nv;
    h->limbs = C->sp.limbs;
    h->side = C->T.side;
    h->store = std::make_unique<PepStore>([C](const Expo& v) { return build_entry(*C, v); }, spec, C->T.nv, C->T.d);
    out = h.release();
  });
  return reinterpret_cast<drzg_pep_store*>(out);
}

drzg_pep_store* drzg_pep_store_create_stub(int32_t nv, int32_t d, const char* spec) {
  StoreHandle* out = nullptr;
  pguard([&] {
    auto h = std::make_unique<StoreHandle>();
    h->nv = nv;
    h->store = std::make_unique<PepStore>(
        [](const Expo& v) {
          auto e = std::make_shared<PepEntryHost>();
          e->v = v;
          e->nnz = v.total();
          return PepPtr(e);
        },
        spec, nv, d);
    out = h.release();
  });
  return reinterpret_cast<drzg_pep_store*>(out);
}

void drzg_pep_store_free(drzg_pep_store* s) { delete reinterpret_cast<StoreHandle*>(s); }

int drzg_pep_get(drzg_pep_store* s, const int32_t* v, uint64_t* planes_out, int64_t* nnz_out) {
  return pguard([&] {
    StoreHandle& h = *reinterpret_cast<StoreHandle*>(s);
    Expo ve(h.nv);
    for (int i = 0; i < h.nv; ++i) ve[i] = v[i];
    PepPtr e = h.store->get(ve);
    if (nnz_out) *nnz_out = e->nnz;
    if (planes_out && !e->planes.empty()) std::memcpy(planes_out, e->planes.data(), e->planes.size() * 8);
  });
}

int drzg_pep_stats(drzg_pep_store* s, int64_t* hits, int64_t* misses, int64_t* evictions) {
  return pguard([&] {
    i64 a, b, c;
    reinterpret_cast<StoreHandle*>(s)->store->stats(&a, &b, &c);
    *hits = a;
    *misses = b;
    *evictions = c;
  });
}

int drzg_pep_eval_to_linear(drzg_pep_store* s, const int32_t* v, const int32_t* x, uint64_t* A, uint64_t* B) {
  return pguard([&] {
    StoreHandle& h = *reinterpret_cast<StoreHandle*>(s);
    DRZG_REQUIRE(h.ctx, "pep: stub store has no matrices");
    StatesCtx& C = *h.ctx;
    Expo ve(h.nv);
    for (int i = 0; i < h.nv; ++i) ve[i] = v[i];
    PepPtr e = h.store->get(ve);
    const int side = h.side, limbs = h.limbs, nv = h.nv;
    const u64 beta = C.sp.beta;
    const size_t nn = (size_t)side * side;
    // A = sum_i v_i A_i, B = sum_i x_i A_i + A_{n+1} mod p^M (reduction.hpp:300-339)
    if (!C.hm.wide) {
      const u128 m = C.hm.m128;
      for (size_t rc = 0; rc < nn; ++rc) {
        u128 a = 0, b = 0;
        for (int t = 0; t <= nv; ++t) {
          u128 val = 0;
          for (int l = limbs - 1; l >= 0; --l) val = val * beta + e->planes[((size_t)t * limbs + l) * nn + rc];
          if (!val) continue;
          if (t < nv) {
            a = (a + mulm128(val, (u128)v[t], m)) % m;
            b = (b + mulm128(val, (u128)x[t], m)) % m;
          } else {
            b = (b + val) % m;
          }
        }
        for (int l = 0; l < limbs; ++l) {
          A[(size_t)l * nn + rc] = (uint64_t)(a % beta);
          B[(size_t)l * nn + rc] = (uint64_t)(b % beta);
          a /= beta;
          b /= beta;
        }
      }
      return;
    }
    for (size_t rc = 0; rc < nn; ++rc) {
      Z a(0), b(0);
      for (int t = 0; t <= nv; ++t) {
        Z val(0);
        for (int l = limbs - 1; l >= 0; --l)
          val = val * Z::from_u64(beta) + Z::from_u64(e->planes[((size_t)t * limbs + l) * nn + rc]);
        if (val == Z(0)) continue;
        if (t < nv) {
          a += val * Z((long)v[t]);
          b += val * Z((long)x[t]);
        } else {
          b += val;
        }
      }
      a = a.mod(C.hm.mz);
      b = b.mod(C.hm.mz);
      for (int l = 0; l < limbs; ++l) {
        Z ra = a.mod(Z::from_u64(beta)), rb = b.mod(Z::from_u64(beta));
        A[(size_t)l * nn + rc] = ra.to_u64();
        B[(size_t)l * nn + rc] = rb.to_u64();
        a = (a - ra).divexact(Z::from_u64(beta));
        b = (b - rb).divexact(Z::from_u64(beta));
      }
    }
  });
}

}  // extern "C"
