// Device-resident reduction engine (see engine.cuh).
#include <algorithm>
#include <tuple>
#include <functional>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>

#include "engine.cuh"
#include "host/flatmap.hpp"

#include <condition_variable>
#include <deque>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include "kernels/dixon.cuh"
#include "kernels/tc_gemm.cuh"

namespace drzg {

namespace {
inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
}  // namespace

// Block-sparse order of the Dixon system for the tensor-core carry.
//
// Jp's rows are Homog_L (monomial m) and its columns the solution indices r,
// with Jp[m, r] != 0 only for m - mu_r in the support of the generator of r
// (a quadric or cubic in every BASELINE shape): about 19 nonzeros per row of
// 3003 for the fourfold.  Rows sorted lexicographically under a well-chosen
// variable order, and columns by the mean position of their nonzero rows,
// leave most 128 x 128 blocks of Jp empty (71% for the random fourfold), so
// the carry GEMM of an M tile runs over its nonzero K blocks only.  The
// permutation is applied to every engine table at upload (Cq rows/columns,
// Jp, the gather tables and the T_x source indices); the reference-shaped
// RuvTables are not touched.  Returns new position of every m and every r.
namespace {
struct SysOrder {
  std::vector<int> pos_m, pos_r;
  std::vector<int> kb_ptr, kb_idx;  // per 128-row M tile: nonzero 128-wide K blocks
  long long blocks = 0;
};

// the T_x grouping of solution indices (DRZG_TX_GROUP=0/1)
bool tx_grouped() {
  static const bool on = [] {
    const char* e = std::getenv("DRZG_TX_GROUP");
    return e && std::string(e) == "1";
  }();
  return on;
}

SysOrder order_system(const RuvTables& T, bool search, bool group_tx) {
  const int nL = T.nL, nv = T.nv;
  constexpr int B = 128;
  const int nt = (nL + B - 1) / B;
  const auto& rowp = T.sys.rowptr;
  const auto& colv = T.sys.col;
  auto sort_pos = [&](const std::vector<double>& key) {
    std::vector<int> ord(nL), pos(nL);
    for (int i = 0; i < nL; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return key[a] < key[b]; });
    for (int i = 0; i < nL; ++i) pos[ord[i]] = i;
    return pos;
  };
  auto col_pos = [&](const std::vector<int>& pm) {
    std::vector<double> sum(nL, 0.0), cnt(nL, 0.0);
    for (int m = 0; m < nL; ++m)
      for (int e = rowp[m]; e < rowp[m + 1]; ++e) sum[colv[e]] += pm[m], cnt[colv[e]] += 1;
    for (int r = 0; r < nL; ++r) sum[r] = cnt[r] > 0 ? sum[r] / cnt[r] : 1e18 + r;
    return sort_pos(sum);
  };
  auto blocks_of = [&](const std::vector<int>& pm, const std::vector<int>& pr) {
    std::vector<char> occ((size_t)nt * nt, 0);
    long long n = 0;
    for (int m = 0; m < nL; ++m)
      for (int e = rowp[m]; e < rowp[m + 1]; ++e) {
        char& o = occ[(size_t)(pm[m] / B) * nt + pr[colv[e]] / B];
        n += !o;
        o = 1;
      }
    return std::make_pair(n, occ);
  };
  SysOrder best;
  best.pos_m.resize(nL);
  best.pos_r.resize(nL);
  for (int i = 0; i < nL; ++i) best.pos_m[i] = best.pos_r[i] = i;
  best.blocks = blocks_of(best.pos_m, best.pos_r).first;
  if (search) {
    // every variable order (and its reverse) scored on host threads (the
    // fourfold's 1440 candidates took ~0.5 s on one); the first best in
    // enumeration order wins, as it did sequentially
    const auto& Lm = monos(nv, T.L).mons;
    std::vector<std::vector<int>> perms;
    {
      std::vector<int> vp(nv);
      for (int i = 0; i < nv; ++i) vp[i] = i;
      do perms.push_back(vp);
      while (std::next_permutation(vp.begin(), vp.end()));
    }
    const int ncand = 2 * (int)perms.size();
    std::vector<long long> score(ncand);
    auto eval = [&](int c) {
      const std::vector<int>& vp = perms[c / 2];
      const int sgn = (c & 1) ? 1 : -1;
      std::vector<double> key(nL);
      for (int m = 0; m < nL; ++m) {
        double k = 0;
        for (int i = 0; i < nv; ++i) k = k * 64 + sgn * Lm[m][vp[i]];
        key[m] = k;
      }
      std::vector<int> pm = sort_pos(key), pr = col_pos(pm);
      return std::make_tuple(blocks_of(pm, pr).first, std::move(pm), std::move(pr));
    };
    const int nth = std::max(1, std::min<int>((int)call_cores(), ncand / 8));
    std::vector<std::thread> pool;
    for (int t = 0; t < nth; ++t)
      pool.emplace_back([&, t] {
        for (int c = t; c < ncand; c += nth) score[c] = std::get<0>(eval(c));
      });
    for (auto& th : pool) th.join();
    int bestc = -1;
    for (int c = 0; c < ncand; ++c)
      if (score[c] < best.blocks && (bestc < 0 || score[c] < score[bestc])) bestc = c;
    if (bestc >= 0) {
      auto r = eval(bestc);
      best.blocks = std::get<0>(r);
      best.pos_m = std::move(std::get<1>(r));
      best.pos_r = std::move(std::get<2>(r));
    }
  }
  if (group_tx) {
    // solution indices feeding one side row made adjacent (each r feeds
    // exactly one row sol_row[r]), groups in the order of their first
    // member: the T_x epilogue then reads one contiguous Y slab per range of
    // side rows
    std::vector<int> gfirst(T.side, INT32_MAX);
    for (int r = 0; r < nL; ++r) gfirst[T.sol_row[r]] = std::min(gfirst[T.sol_row[r]], best.pos_r[r]);
    std::vector<double> key(nL);
    for (int r = 0; r < nL; ++r) key[r] = (double)gfirst[T.sol_row[r]] * (double)(nL + 1) + best.pos_r[r];
    best.pos_r = sort_pos(key);
    best.blocks = blocks_of(best.pos_m, best.pos_r).first;
  }
  auto occ = blocks_of(best.pos_m, best.pos_r).second;
  best.kb_ptr.assign(1, 0);
  for (int i = 0; i < nt; ++i) {
    for (int j = 0; j < nt; ++j)
      if (occ[(size_t)i * nt + j]) best.kb_idx.push_back(j);
    best.kb_ptr.push_back((int)best.kb_idx.size());
  }
  return best;
}
}  // namespace

// debug: nonzero Jp blocks of the carry order without / with the T_x grouping
std::pair<long long, long long> debug_order_blocks(const RuvTables& T) {
  return {order_system(T, T.nL > 2 * 128, false).blocks, order_system(T, T.nL > 2 * 128, true).blocks};
}

ReductionEngine::ReductionEngine(const RuvTables& T, int n, u64 p, cudaStream_t st)
    : T_(&T), n_(n), p_(p), st_(st) {
  {
    // stream-ordered allocations stay mapped between zeta functions (the
    // default pool would hand them back to the driver at every sync)
    int dev = 0;
    DRZG_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t mp;
    DRZG_CUDA(cudaDeviceGetDefaultMemPool(&mp, dev));
    uint64_t keep = UINT64_MAX;
    DRZG_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep));
    DRZG_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, dev));
  }
  DRZG_REQUIRE(T.dp.Ld <= dev::kLdMax, "engine: too many digit planes");
  // small systems pad to whole 128-row tiles (the one-launch Dixon kernel)
  nLp_ = round_up(T.nL, 128);  // whole 128-row tiles (the one-launch kernels)
  sidep_ = round_up(T.side, 16);
  slot_stride_ = (long long)T.dp.Ld * sidep_;
  gsize_ = (int)mono_count(T.nv, T.D - 1);
  const char* g = std::getenv("DRZG_GEMM");
  const bool want_tc = !(g && std::string(g) == "dp4a");
  const char* so = std::getenv("DRZG_SPARSE_CARRY");
  sparse_carry_ = want_tc && !(so && std::string(so) == "0");
  // block-sparse order of the system (identity unless the carry uses it)
  auto to0 = std::chrono::steady_clock::now();
  SysOrder ord = order_system(T, sparse_carry_ && T.nL > 2 * 128, tx_grouped());
  if (std::getenv("DRZG_VERBOSE"))
    std::fprintf(stderr, "[drzg] system order: %lld of %lld Jp blocks nonzero (%.3f s)\n", ord.blocks,
                 (long long)((T.nL + 127) / 128) * ((T.nL + 127) / 128),
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - to0).count());
  pos_m_ = ord.pos_m;
  pos_r_ = ord.pos_r;
  const std::vector<int>& pm = ord.pos_m;
  const std::vector<int>& pr = ord.pos_r;
  kblocks_ = ord.blocks;
  // C padded to nLp x nLp: rows solution indices r, columns rows m
  std::vector<int8_t> Cp((size_t)nLp_ * nLp_, 0);
  for (int r = 0; r < T.nL; ++r)
    for (int c = 0; c < T.nL; ++c) Cp[(size_t)pr[r] * nLp_ + pm[c]] = T.sys.Cq[(size_t)r * T.nL + c];
  C_.upload(Cp, st_);
  // Jp in the new order (CSR): rows m, columns r
  std::vector<int> jptr(T.nL + 1, 0), jcol, jval;
  {
    std::vector<int> inv_m(T.nL);
    for (int m = 0; m < T.nL; ++m) inv_m[pm[m]] = m;
    for (int nm = 0; nm < T.nL; ++nm) {
      const int m = inv_m[nm];
      for (int e = T.sys.rowptr[m]; e < T.sys.rowptr[m + 1]; ++e) {
        jcol.push_back(pr[T.sys.col[e]]);
        jval.push_back(T.sys.val[e]);
      }
      jptr[nm + 1] = (int)jcol.size();
    }
  }
  // dense Jp for the tensor-core carry product (entries are exact small
  // non-negative integers; u8 operand); DRZG_GEMM=dp4a selects the CUDA-core path
  {
    int maxv = 0;
    for (int v : jval) maxv = std::max(maxv, v);
    // |c_{k+1}| <= (127 + |c_k| + R (q-1)/2) / q  =>  |c| <= (127 + R (q-1)/2) / (q-1)
    i64 R = 0;
    for (int r = 0; r < T.nL; ++r) {
      i64 rs = 0;
      for (int e2 = jptr[r]; e2 < jptr[r + 1]; ++e2) rs += std::abs(jval[e2]);
      R = std::max(R, rs);
    }
    i64 cmax = (127 + R * (T.dp.q - 1) / 2) / (T.dp.q - 1) + 1;
    // the running residual r = b + c is stored as in + q h with h in int8
    DRZG_REQUIRE((127 + cmax + T.dp.q) / T.dp.q < 127, "engine: Dixon residual high part exceeds int8");
    // multiply-high epilogues are exact when every operand is < 2^22:
    // digit GEMM |acc| <= nLp (q/2)^2, carry numerators <= 127 + cmax + R q/2,
    // T epilogue <= (terms per side row) (max weight) (q/2) + carry
    const i64 half = T.dp.q / 2;
    i64 wmax = 0;
    for (int r = 0; r < T.nL; ++r) wmax = std::max<i64>(wmax, T.sol_mu[r]);
    i64 bound = std::max<i64>((i64)nLp_ * half * half, 127 + cmax + R * half);
    i64 maxnt = 0;  // solution indices feeding one side row
    for (int g2 = 0; g2 < T.side; ++g2) maxnt = std::max<i64>(maxnt, T.t_ptr[g2 + 1] - T.t_ptr[g2]);
    bound = std::max<i64>(bound, std::max<i64>(T.nv, maxnt) * (4096 + wmax) * half + 4096);
    // (and the T_x weights x_i + mu_i, exponents below 4096, fit the 16-bit
    // halves the epilogue's dp2a products take)
    fast_ = bound < ((i64)1 << 22) && 4096 + wmax < (1 << 15);
    if (want_tc && maxv < 256) {
      std::vector<int8_t> Jd((size_t)nLp_ * nLp_, 0);
      for (int r = 0; r < T.nL; ++r)
        for (int e = jptr[r]; e < jptr[r + 1]; ++e) Jd[(size_t)r * nLp_ + jcol[e]] = (int8_t)(uint8_t)jval[e];
      Jd_.upload(Jd, st_);
      use_tc_ = true;
    }
  }
  sparse_carry_ = sparse_carry_ && use_tc_;
  DRZG_REQUIRE(dev::gather_smem_bytes(sidep_) <= 200 * 1024, "engine: side too large for the gather staging");
  // the shared-memory opt-ins are per (kernel, device) and process-wide:
  // set once per device at the largest size any engine launches (an engine
  // of another shape on a concurrent thread must not lower it under a launch)
  // -- the gather stages 32 states x sidep; the flush transpose Ld x 64 rows
  // x 32 states (50 KB at the quintic surface's 25 digit planes)
  {
    static std::mutex mu;
    static bool done[64] = {false};
    int dev = 0;
    DRZG_CUDA(cudaGetDevice(&dev));
    DRZG_REQUIRE(dev >= 0 && dev < 64, "engine: device index out of range");
    std::lock_guard<std::mutex> lk(mu);
    if (!done[dev]) {
      DRZG_CUDA(cudaFuncSetAttribute(dev::gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      DRZG_CUDA(cudaFuncSetAttribute(dev::flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     dev::kLdMax * dev::kFlushRows * dev::kFlushStates));
      done[dev] = true;
    }
  }
  const char* fz = std::getenv("DRZG_FUSED");
  fused_ = use_tc_ && dixon_fused_ok(nLp_) && !(fz && std::string(fz) == "0");
  const char* ck = std::getenv("DRZG_CHUNK");
  // whole-chunk launches are opt-in: over 58 K3 zeta functions they gave a
  // 0.244 s median against 0.230 s step by step (their T_x runs inside the
  // block's CTA, serialised with its Dixon solve)
  chunk_ = fused_ && dixon_chunk_ok(nLp_, T.dp.Ld) && ck && std::string(ck) == "1";
  const char* fl = std::getenv("DRZG_FLOW");
  flow_ = use_tc_ && sparse_carry_ && !fused_ && nLp_ % 128 == 0 && !(fl && std::string(fl) == "0");
  const char* f2e = std::getenv("DRZG_FLOW2");
  flow2_ = flow_ && !(f2e && std::string(f2e) == "0");
  if (sparse_carry_) {
    kb_ptr_.upload(ord.kb_ptr, st_);
    kb_idx_.upload(ord.kb_idx, st_);
    // pair tiles (rows 256 i .. 256 i + 255): the union of the two K-block lists
    const int nt = (int)ord.kb_ptr.size() - 1;
    std::vector<int> p2{0}, i2;
    for (int i = 0; 2 * i < nt; ++i) {
      std::vector<int> u(ord.kb_idx.begin() + ord.kb_ptr[2 * i], ord.kb_idx.begin() + ord.kb_ptr[2 * i + 1]);
      if (2 * i + 1 < nt) u.insert(u.end(), ord.kb_idx.begin() + ord.kb_ptr[2 * i + 1], ord.kb_idx.begin() + ord.kb_ptr[2 * i + 2]);
      std::sort(u.begin(), u.end());
      u.erase(std::unique(u.begin(), u.end()), u.end());
      i2.insert(i2.end(), u.begin(), u.end());
      p2.push_back((int)i2.size());
    }
    kblocks2_ = (long long)i2.size();
    kb2_ptr_.upload(p2, st_);
    kb2_idx_.upload(i2, st_);
    if (std::getenv("DRZG_VERBOSE"))
      std::fprintf(stderr, "[drzg] carry K blocks: %lld (128-row tiles), %lld (256-row pairs, x2 rows)\n", kblocks_,
                   kblocks2_);
  }
  jp_ptr_.upload(jptr, st_);
  jp_col_.upload(jcol, st_);
  jp_val_.upload(jval, st_);
  {
    std::vector<int> gi(T.gidx.size()), gv(T.ginv.size());
    for (int vi = 0; vi < T.ndir; ++vi) {
      for (int m = 0; m < T.nL; ++m) gi[(size_t)vi * T.nL + pm[m]] = T.gidx[(size_t)vi * T.nL + m];
      for (int g2 = 0; g2 < T.side; ++g2) {
        const int m = T.ginv[(size_t)vi * T.side + g2];
        gv[(size_t)vi * T.side + g2] = m >= 0 ? pm[m] : -1;
      }
    }
    gidx_.upload(gi, st_);
    ginv_.upload(gv, st_);
  }
  const auto& dl = monos(T.nv, T.d).mons;
  std::vector<int> dirs;
  for (const auto& v : dl) {
    dirs_host_.push_back(v);
    for (int i = 0; i < T.nv; ++i) dirs.push_back(v[i]);
  }
  dirs_.upload(dirs, st_);
  t_ptr_.upload(T.t_ptr, st_);
  {
    std::vector<int> ts(T.t_src.size()), si(T.nL), smu(T.nL);
    for (size_t e = 0; e < T.t_src.size(); ++e) ts[e] = pr[T.t_src[e]];
    for (int r = 0; r < T.nL; ++r) {
      si[pr[r]] = T.sol_i[r];
      smu[pr[r]] = T.sol_mu[r];
    }
    t_src_.upload(ts, st_);
    sol_i_.upload(si, st_);
    sol_mu_.upload(smu, st_);
  }
  std::vector<int> mon;
  for (const auto& e : monos(T.nv, T.D).mons)
    for (int i = 0; i < T.nv; ++i) mon.push_back(e[i]);
  mon_.upload(mon, st_);
  std::vector<unsigned long long> bt(Binom::get().tab.begin(), Binom::get().tab.end());
  btab_.upload(bt, st_);
  DRZG_CUDA(cudaEventCreate(&ev0_));
  DRZG_CUDA(cudaEventCreate(&ev1_));
}

ReductionEngine::~ReductionEngine() {
  release_pool();
  cudaEventDestroy(ev0_);
  cudaEventDestroy(ev1_);
}

void ReductionEngine::timed(double* acc, const std::function<void()>& f) {
  ++g_traffic.launches;
  if (!clock.on) {
    f();
    return;
  }
  DRZG_CUDA(cudaEventRecord(ev0_, st_));
  f();
  DRZG_CUDA(cudaEventRecord(ev1_, st_));
  DRZG_CUDA(cudaEventSynchronize(ev1_));
  float ms = 0;
  DRZG_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
  *acc += ms;
}

// The state pool lives in one reserved virtual range; growth maps more
// physical memory behind it (CUDA VMM), so existing slots never move and no
// copy (old + new pool at once) is needed
namespace {
struct Vmm {
  PFN_cuMemAddressReserve_v10020 reserve = nullptr;
  PFN_cuMemCreate_v10020 create = nullptr;
  PFN_cuMemMap_v10020 map = nullptr;
  PFN_cuMemSetAccess_v10020 access = nullptr;
  PFN_cuMemGetAllocationGranularity_v10020 gran = nullptr;
  PFN_cuMemUnmap_v10020 unmap = nullptr;
  PFN_cuMemRelease_v10020 release = nullptr;
  PFN_cuMemAddressFree_v10020 addr_free = nullptr;
  static const Vmm& get() {
    static Vmm v = [] {
      Vmm x;
      auto load = [](const char* name, void** fn) {
        cudaDriverEntryPointQueryResult q;
        DRZG_CUDA(cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q));
        DRZG_REQUIRE(q == cudaDriverEntryPointSuccess, std::string("driver entry point ") + name);
      };
      load("cuMemAddressReserve", (void**)&x.reserve);
      load("cuMemCreate", (void**)&x.create);
      load("cuMemMap", (void**)&x.map);
      load("cuMemSetAccess", (void**)&x.access);
      load("cuMemGetAllocationGranularity", (void**)&x.gran);
      load("cuMemUnmap", (void**)&x.unmap);
      load("cuMemRelease", (void**)&x.release);
      load("cuMemAddressFree", (void**)&x.addr_free);
      return x;
    }();
    return v;
  }
};
#define DRZG_CU(x)                                                                             \
  do {                                                                                         \
    CUresult r_ = (x);                                                                         \
    if (r_ != CUDA_SUCCESS)                                                                    \
      throw ::drzg::contract_error("CUDA driver error " + std::to_string((int)r_), __FILE__, __LINE__); \
  } while (0)
}  // namespace

// A released pool stays mapped for the next engine on the same device (like
// a caching allocator): unmapping and re-creating gigabytes of physical
// memory costs tens to hundreds of milliseconds per zeta function, with a
// long tail.  Slots carry no state between engines (seed_kernel writes every
// fresh slot in full).
namespace {
struct CachedPool {
  int8_t* base = nullptr;
  size_t reserved = 0, mapped = 0;
  std::vector<std::pair<size_t, std::pair<size_t, unsigned long long>>> chunks;  // off, (bytes, handle)
};
std::mutex g_pool_mu;
// per device: the pools finished engines left (one per engine that was alive
// at once: concurrent calls each keep theirs), at most half the device mapped
std::map<int, std::vector<CachedPool>> g_pool_cache;
}  // namespace

size_t cached_pool_bytes(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  size_t b = 0;
  auto it = g_pool_cache.find(dev);
  if (it != g_pool_cache.end())
    for (const auto& c : it->second) b += c.mapped;
  return b;
}

// the retained mempool keeps freed stream-ordered memory reserved (fast
// reuse across zeta functions); cudaMemGetInfo does not count it as free, so
// memory planning trims it first
void ReductionEngine::trim_mempool(int dev) {
  cudaMemPool_t mp;
  DRZG_CUDA(cudaDeviceGetDefaultMemPool(&mp, dev));
  DRZG_CUDA(cudaMemPoolTrimTo(mp, 0));
}

void ReductionEngine::grow_pool(int need) {
  const Vmm& V = Vmm::get();
  int dev = 0;
  DRZG_CUDA(cudaGetDevice(&dev));
  if (!pool_) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pool_cache.find(dev);
    if (it != g_pool_cache.end() && !it->second.empty()) {
      // the largest cached pool
      auto& v = it->second;
      auto best = std::max_element(v.begin(), v.end(),
                                   [](const CachedPool& a, const CachedPool& b) { return a.mapped < b.mapped; });
      pool_ = best->base;
      vmm_reserved_ = best->reserved;
      vmm_mapped_ = best->mapped;
      for (auto& c : best->chunks) vmm_chunks_.push_back({c.first, c.second.first, c.second.second});
      v.erase(best);
      pool_dev_ = dev;
    }
  }
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  size_t gran = 0;
  DRZG_CU(V.gran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  size_t fr = 0, tot = 0;
  if (!pool_) {
    // reserve address space for the whole device once
    tot = device_total_memory();
    if (!tot) mem_info(&fr, &tot, "engine.cu:1");
    vmm_reserved_ = (tot + gran - 1) / gran * gran;
    CUdeviceptr base = 0;
    DRZG_CU(V.reserve(&base, vmm_reserved_, gran, 0, 0));
    pool_ = reinterpret_cast<int8_t*>(base);
    vmm_mapped_ = 0;
    pool_dev_ = dev;
  }
  int ncap = std::max(need, cap_ + std::max(1024, cap_ / 2));
  size_t want = (size_t)ncap * slot_stride_;
  if (want <= vmm_mapped_) {
    // the (cached) mapping already covers it: no sync, no driver query
    int ncap2 = (int)std::min<size_t>(vmm_mapped_ / (size_t)slot_stride_, (size_t)INT32_MAX);
    for (int s = ncap2 - 1; s >= cap_; --s) free_.push_back(s);
    cap_ = ncap2;
    return;
  }
  DRZG_CUDA(cudaStreamSynchronize(st_));
  if (want > vmm_mapped_) trim_mempool(dev);  // unused stream-ordered reserve back to the driver
  mem_info(&fr, &tot, "engine.cu:2");
  if (want > vmm_mapped_ + fr / 2) {
    // other engines' cached pools give their memory back before this one
    // settles for less
    std::vector<CachedPool> drop;
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      drop.swap(g_pool_cache[dev]);
    }
    for (auto& c : drop) {
      for (auto& k : c.chunks) {
        V.unmap(reinterpret_cast<CUdeviceptr>(c.base) + k.first, k.second.first);
        V.release((CUmemGenericAllocationHandle)k.second.second);
      }
      V.addr_free(reinterpret_cast<CUdeviceptr>(c.base), c.reserved);
    }
    if (!drop.empty()) mem_info(&fr, &tot, "engine.cu:2b");
  }
  size_t margin = (size_t)2 << 30;
  std::unique_lock<std::mutex> tmp_lock(tmp_mu_, std::defer_lock);
  if (want > vmm_mapped_ + (fr > margin ? fr - margin : 0)) tmp_lock.lock();  // no sweep is launching now
  if (want > vmm_mapped_ + (fr > margin ? fr - margin : 0) && bcap_ > 0) {
    // give the batch temporaries back first; they are re-sized on demand
    // (stream-ordered frees: kernels already queued on st_ still see them)
    Bg_.release();
    Y_.release();
    IN_.release();
    H_.release();
    W_.release();
    bcap_ = 0;
    DRZG_CUDA(cudaStreamSynchronize(st_));
    trim_mempool(dev);
    mem_info(&fr, &tot, "engine.cu:3");
  }
  size_t room = vmm_mapped_ + (fr > margin ? fr - margin : 0);
  if (want > room) want = std::max<size_t>(room, (size_t)need * (size_t)slot_stride_);  // settle for what fits
  DRZG_REQUIRE(want <= room && want <= vmm_reserved_,
               "engine: state pool exceeds device memory (" + std::to_string(need) + " slots)");
  size_t target = (want + gran - 1) / gran * gran;
  target = std::min(target, vmm_reserved_);
  while (vmm_mapped_ < target) {
    size_t chunk = std::min<size_t>(target - vmm_mapped_, (size_t)4 << 30);
    chunk = (chunk + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h;
    DRZG_CU(V.create(&h, chunk, &prop, 0));
    CUdeviceptr at = reinterpret_cast<CUdeviceptr>(pool_) + vmm_mapped_;
    DRZG_CU(V.map(at, chunk, 0, h, 0));
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    DRZG_CU(V.access(at, chunk, &acc, 1));
    vmm_chunks_.push_back({vmm_mapped_, chunk, (unsigned long long)h});
    vmm_mapped_ += chunk;
  }
  int ncap2 = (int)std::min<size_t>(vmm_mapped_ / (size_t)slot_stride_, (size_t)INT32_MAX);
  for (int s = ncap2 - 1; s >= cap_; --s) free_.push_back(s);
  cap_ = ncap2;
}

void ReductionEngine::release_pool() {
  if (!pool_) return;
  cudaStreamSynchronize(st_);
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto& v = g_pool_cache[pool_dev_];
    size_t cached = 0;
    for (const auto& c0 : v) cached += c0.mapped;
    const size_t tot = device_total_memory();
    if (!std::getenv("DRZG_NO_POOL_CACHE") && (v.empty() || !tot || cached + vmm_mapped_ <= tot / 2)) {
      CachedPool c;
      c.base = pool_;
      c.reserved = vmm_reserved_;
      c.mapped = vmm_mapped_;
      for (auto& k : vmm_chunks_) c.chunks.push_back({k.off, {k.bytes, k.handle}});
      v.push_back(std::move(c));
      vmm_chunks_.clear();
      pool_ = nullptr;
      return;
    }
  }
  const Vmm& V = Vmm::get();
  for (auto& c : vmm_chunks_) {
    V.unmap(reinterpret_cast<CUdeviceptr>(pool_) + c.off, c.bytes);
    V.release((CUmemGenericAllocationHandle)c.handle);
  }
  V.addr_free(reinterpret_cast<CUdeviceptr>(pool_), vmm_reserved_);
  vmm_chunks_.clear();
  pool_ = nullptr;
}

int ReductionEngine::alloc_slot() {
  if (free_.empty()) grow_pool(cap_ + 1);
  int s = free_.back();
  free_.pop_back();
  peak_live_ = std::max<i64>(peak_live_, (i64)cap_ - (i64)free_.size());
  return s;
}

void ReductionEngine::ensure_batch(int B) {
  if (B <= bcap_) return;
  const int Ld = T_->dp.Ld;
  size_t per = (size_t)(2 * Ld + 1) * nLp_ + sizeof(int16_t) * nLp_ + (size_t)Ld * sidep_;
  size_t fr = 0, tot = 0;
  const size_t tot_mem = device_total_memory();
  if (tot_mem && (double)round_up(B, 64) * (double)per < 0.02 * (double)tot_mem) {
    // small batches: temporaries for exactly this batch, no driver query
    fr = tot = tot_mem;
  } else {
    mem_info(&fr, &tot, "engine.cu:4");
  }
  if (fr * 0.8 < tot * 0.12) {
    int dev = 0;
    DRZG_CUDA(cudaGetDevice(&dev));
    DRZG_CUDA(cudaStreamSynchronize(st_));
    trim_mempool(dev);
    mem_info(&fr, &tot, "engine.cu:5");
  }
  // temporaries get at most half of what is free, in multiples of 64 states
  // temporaries: at most 80% of what is free and 12% of the device, so the
  // state pool keeps room to grow
  size_t lim = std::max<size_t>(64, std::min<size_t>((size_t)(fr * 0.8), (size_t)(tot * 0.12)) / per / 64 * 64);
  lim = std::min<size_t>(lim, (size_t)1 << 21);  // grid.y = states / 32 stays < 65536
  int nb = (int)std::min<size_t>(lim, (size_t)round_up(B, 64));
  if (nb <= bcap_) return;
  bcap_ = nb;
  // state-contiguous layouts with pitch bcap_: Bg/Y Ld x nLp x P, IN/H nLp x P
  Bg_.alloc((size_t)bcap_ * Ld * nLp_, st_);
  Y_.alloc((size_t)bcap_ * Ld * nLp_, st_);
  IN_.alloc((size_t)bcap_ * nLp_, st_);
  H_.alloc((size_t)bcap_ * nLp_, st_);
  W_.alloc((size_t)bcap_ * Ld * sidep_, st_);
  // K padding of Bg / IN / Y must read as zero
  DRZG_CUDA(cudaMemsetAsync(Bg_.p, 0, Bg_.n, st_));
  DRZG_CUDA(cudaMemsetAsync(Y_.p, 0, Y_.n, st_));
  DRZG_CUDA(cudaMemsetAsync(IN_.p, 0, IN_.n, st_));
  DRZG_CUDA(cudaMemsetAsync(H_.p, 0, H_.n, st_));
}

dev::StepArgs ReductionEngine::make_args(int b0, int nb, int y) {
  const RuvTables& T = *T_;
  dev::StepArgs a;
  a.C = C_.p;
  a.jp_ptr = jp_ptr_.p;
  a.jp_col = jp_col_.p;
  a.jp_val = jp_val_.p;
  a.gidx = gidx_.p;
  a.ginv = ginv_.p;
  a.ks = d_k_.p + b0;
  a.dirs = dirs_.p;
  a.t_ptr = t_ptr_.p;
  a.t_src = t_src_.p;
  a.sol_i = sol_i_.p;
  a.sol_mu = sol_mu_.p;
  a.nv = T.nv;
  a.nL = T.nL;
  a.nLp = nLp_;
  a.side = T.side;
  a.sidep = sidep_;
  a.Ld = T.dp.Ld;
  a.q = T.dp.q;
  a.fq = FastQ::make(T.dp.q);
  a.fast = fast_ ? 1 : 0;
  a.pool = pool_;
  a.slot_stride = slot_stride_;
  a.slot = d_slot_.p + b0;
  a.vdir = d_vdir_.p + b0;
  a.u0 = d_u0_.p + (size_t)b0 * T.nv;
  a.y = y;
  a.B = nb;
  a.P = bcap_;
  a.Bg = Bg_.p;
  a.IN = IN_.p;
  a.H = H_.p;
  a.Y = Y_.p;
  a.W = W_.p;
  return a;
}

// Dixon solve of the batch's gathered digits (Bg, in_0, c_0 = 0) into Y
void ReductionEngine::dixon(dev::StepArgs& a) {
  const RuvTables& T = *T_;
  const int nb = a.B;
  dim3 gG((nb + 63) / 64, nLp_ / 64);
  dim3 gC((nb + 127) / 128, T.nL);
  if (fused_) {
    // small systems: the whole solve of every state in one launch
    FusedArgs f;
    f.nL = T.nL;
    f.nLp = nLp_;
    f.N = nb;
    f.P = bcap_;
    f.Ld = T.dp.Ld;
    f.q = T.dp.q;
    f.fq = FastQ::make(T.dp.q);
    f.fast = fast_ ? 1 : 0;
    f.Bg = Bg_.p;
    f.Y = Y_.p;
    if (chunk_now_) {
      // every step of the sub-batch's chunks in this launch (T_x in-kernel)
      f.chunk = 1;
      f.ks = a.ks;
      f.vdir = a.vdir;
      f.u0 = a.u0;
      f.dirs = a.dirs;
      f.t_ptr = a.t_ptr;
      f.t_src = a.t_src;
      f.sol_i = a.sol_i;
      f.sol_mu = a.sol_mu;
      f.ginv = a.ginv;
      f.W = a.W;
      f.side = a.side;
      f.sidep = a.sidep;
      f.nv = a.nv;
    }
    static int traces = std::getenv("DRZG_FUSED_TRACE") ? 6 : 0;
    DevBuf<long long> tb;
    if (traces > 0 && nb <= 2048) {
      tb.alloc(4 * T.dp.Ld + 2, st_);
      DRZG_CUDA(cudaMemsetAsync(tb.p, 0, tb.n * 8, st_));
      f.trace = tb.p;
    }
    timed(&clock.gemm_ms, [&] { dixon_fused(C_.p, Jd_.p, f, st_); });
    if (f.trace) {
      --traces;
      std::vector<long long> h(tb.n);
      DRZG_CUDA(cudaMemcpyAsync(h.data(), tb.p, tb.n * 8, cudaMemcpyDeviceToHost, st_));
      DRZG_CUDA(cudaStreamSynchronize(st_));
      std::fprintf(stderr, "[drzg] fused trace N=%d (us from epilogue start):", nb);
      for (int k = 0; k < T.dp.Ld; ++k)
        std::fprintf(stderr, " k%d[D %.1f Y %.1f C %.1f I %.1f]", k, (h[1 + 4 * k] - h[0]) / 1e3,
                     (h[2 + 4 * k] - h[0]) / 1e3, h[3 + 4 * k] ? (h[3 + 4 * k] - h[0]) / 1e3 : 0.0,
                     h[4 + 4 * k] ? (h[4 + 4 * k] - h[0]) / 1e3 : 0.0);
      std::fprintf(stderr, "\n");
    }
    ++clock.gemm_launches;
    clock.gemm_macs += (double)T.dp.Ld * T.nL * T.nL * chunk_steps_;
    clock.carry_macs += (double)(T.dp.Ld - 1) * T.nL * T.nL * chunk_steps_;
    static const bool hist = std::getenv("DRZG_FUSED_HIST") != nullptr;
    if (hist) {
      // state-steps by 64-state blocks per SM of the launch (0: < 1 ... 4: >= 8)
      static double h[5] = {0, 0, 0, 0, 0};
      static long long calls = 0;
      const double per = (double)nb / 64.0 / sms_;
      h[per < 1 ? 0 : per < 2 ? 1 : per < 4 ? 2 : per < 8 ? 3 : 4] += nb;
      if (++calls % 985 == 0)
        std::fprintf(stderr, "[drzg] fused launch states by 64-blocks per SM: <1 %.0f, 1-2 %.0f, 2-4 %.0f, 4-8 %.0f, >=8 %.0f\n",
                     h[0], h[1], h[2], h[3], h[4]);
    }
    return;
  }
  if (flow_) {
    // larger systems: every digit and carry product of the batch in one
    // persistent dataflow launch
    FlowArgs f;
    TcEpiArgs& e = f.epi;
    e.M = T.nL;
    e.N = nb;
    e.q = T.dp.q;
    e.fq = FastQ::make(T.dp.q);
    e.fast = fast_ ? 1 : 0;
    e.Ld = T.dp.Ld;
    e.nLp = nLp_;
    e.nL = T.nL;
    e.P = bcap_;
    e.Y = Y_.p;
    e.Bg = Bg_.p;
    e.H = H_.p;
    e.IN = IN_.p;
    e.kb_ptr = kb_ptr_.p;
    e.kb_idx = kb_idx_.p;
    const size_t nctr = (size_t)(2 * T.dp.Ld - 1) * ((nb + 255) / 256);
    flow_ctr_.alloc(std::max<size_t>(nctr, (size_t)(2 * T.dp.Ld - 1) * ((bcap_ + 255) / 256)), st_);
    f.counters = flow_ctr_.p;
    f.kb2_ptr = kb2_ptr_.p;
    f.kb2_idx = kb2_idx_.p;
    if (flow2_)
      timed(&clock.gemm_ms, [&] { dixon_flow2(C_.p, Jd_.p, f, st_); });
    else
      timed(&clock.gemm_ms, [&] { dixon_flow(C_.p, Jd_.p, f, st_); });
    ++clock.gemm_launches;
    clock.gemm_macs += (double)T.dp.Ld * T.nL * T.nL * nb;
    // useful carry work: Jp's nonzero 128 x 128 blocks (the pair kernel
    // also multiplies the zero blocks its union lists bring in)
    clock.carry_macs += (double)(T.dp.Ld - 1) * kblocks_ * 128 * 128 * nb;
    return;
  }
  for (int k = 0; k < T.dp.Ld; ++k) {
    if (use_tc_) {
      // y_k = bal(Cq . in_k): tcgen05 int8, digit epilogue
      TcEpiArgs e;
      e.mode = (int)TcEpilogue::digit;
      e.M = T.nL;
      e.N = nb;
      e.q = T.dp.q;
      e.fq = FastQ::make(T.dp.q);
      e.fast = fast_ ? 1 : 0;
      e.Ld = T.dp.Ld;
      e.k = k;
      e.nLp = nLp_;
      e.nL = T.nL;
      e.Y = Y_.p;
      e.b_mn = 1;
      e.P = bcap_;
      // in_0 = bal(b_0 + 0) = b_0: digit 0 reads the gathered plane directly
      const int8_t* in = k ? IN_.p : Bg_.p;
      timed(&clock.gemm_ms, [&] { tc_gemm_i8(C_.p, nLp_, nLp_, in, nb, bcap_, nLp_, e, st_); });
      ++clock.gemm_launches;
      clock.gemm_macs += (double)T.nL * T.nL * nb;
      if (k + 1 < T.dp.Ld) {
        // c_{k+1} = (b_k + c_k - Jp . y_k) / q, in_{k+1}: tcgen05 int8 (u8 Jp), carry epilogue
        e.mode = (int)TcEpilogue::carry;
        e.a_unsigned = 1;
        e.Bg = Bg_.p;
        e.H = H_.p;
        e.IN = IN_.p;
        if (sparse_carry_) {
          e.kb_ptr = kb_ptr_.p;
          e.kb_idx = kb_idx_.p;
        }
        timed(&clock.carry_ms, [&] {
          tc_gemm_i8(Jd_.p, nLp_, nLp_, Y_.p + (size_t)k * nLp_ * bcap_, nb, bcap_, nLp_, e, st_);
        });
        ++clock.carry_launches;
        clock.carry_macs += sparse_carry_ ? (double)kblocks_ * 128 * 128 * nb : (double)T.nL * T.nL * nb;
      }
    } else {
      timed(&clock.gemm_ms, [&] { dev::dixon_gemm_kernel<<<gG, 256, 0, st_>>>(a, k); });
      ++clock.gemm_launches;
      clock.gemm_macs += (double)T.nL * T.nL * nb;
      timed(&clock.carry_ms, [&] { dev::dixon_carry_kernel<<<gC, 128, 0, st_>>>(a, k); });
    }
  }
}

int ReductionEngine::chunk_max_states() const {
  static const int mult = [] {
    const char* e = std::getenv("DRZG_CHUNK_MAX");  // states per SM (A/B experiments)
    return e ? std::atoi(e) : 64;
  }();
  return mult * sms_;
}

i64 ReductionEngine::run_sweep(const std::vector<i64>& ks) {
  const RuvTables& T = *T_;
  const int B = (int)ks.size();
  if (B == 0) return 0;
  std::lock_guard<std::mutex> tmp_lock(tmp_mu_);  // grow_pool on the policy thread may release them
  ensure_batch(B);
  i64 mv = 0;
  for (int b0 = 0; b0 < B; b0 += bcap_) {
    const int nb = std::min(bcap_, B - b0);
    // (only batches that fit one round of 32-state blocks: larger ones run
    // 64-state blocks step by step, which a whole-chunk launch cannot hold in
    // shared memory together with the block's y planes)
    if (fused_ && chunk_ && nb <= chunk_max_states()) {
      // small systems: gather, every step of every chunk in one launch (the
      // fused Dixon solve with T_x in-kernel), then W -> pool for all
      dev::StepArgs a = make_args(b0, nb, 1);
      const int gb = (nb + dev::kGatherStates - 1) / dev::kGatherStates;
      const size_t gsm = dev::gather_smem_bytes(sidep_);
      timed(&clock.gather_ms, [&] { dev::gather_kernel<<<gb, dev::kGatherThreads, gsm, st_>>>(a); });
      i64 steps = 0;
      for (int i = 0; i < nb; ++i) steps += ks[b0 + i];
      chunk_now_ = true;
      chunk_steps_ = (double)steps;
      dixon(a);
      chunk_now_ = false;
      chunk_steps_ = 0;
      dim3 gF((nb + dev::kFlushStates - 1) / dev::kFlushStates, (T.side + dev::kFlushRows - 1) / dev::kFlushRows);
      size_t fsm = (size_t)T.dp.Ld * dev::kFlushRows * dev::kFlushStates;
      const double e0f = clock.epi_ms;
      timed(&clock.epi_ms, [&] { dev::flush_kernel<<<gF, 256, fsm, st_>>>(a, 0, nb); });
      clock.flush_ms += clock.epi_ms - e0f;
      DRZG_CUDA(cudaGetLastError());
      mv += steps;
      continue;
    }
    // prefix sizes: states of this sub-batch still stepping at y
    auto count_ge = [&](i64 y) {
      int c = 0;
      while (c < nb && ks[b0 + c] >= y) ++c;
      return c;
    };
    const i64 kmax = ks[b0];
    int By = nb;
    for (i64 y = 1; y <= kmax; ++y) {
      dev::StepArgs a = make_args(b0, By, (int)y);
      if (y == 1) {
        const int gb = (By + dev::kGatherStates - 1) / dev::kGatherStates;
        const size_t gsm = dev::gather_smem_bytes(sidep_);
        timed(&clock.gather_ms, [&] { dev::gather_kernel<<<gb, dev::kGatherThreads, gsm, st_>>>(a); });
      }  // later steps: the previous epilogue already wrote this step's operand
      chunk_steps_ = (double)By;
      dixon(a);
      a.epi_rows = dev::epi_rows_for(By, T.side, sms_);
      dim3 gE((By + 127) / 128, (T.side + a.epi_rows - 1) / a.epi_rows);
      timed(&clock.epi_ms, [&] { dev::launch_epilogue(a, gE, st_); });
      mv += By;
      const int Bn = count_ge(y + 1);
      if (Bn < By) {
        dim3 gF((By - (Bn & ~3) + dev::kFlushStates - 1) / dev::kFlushStates, (T.side + dev::kFlushRows - 1) / dev::kFlushRows);
        size_t fsm = (size_t)T.dp.Ld * dev::kFlushRows * dev::kFlushStates;
        const double e0f = clock.epi_ms;
        timed(&clock.epi_ms, [&] { dev::flush_kernel<<<gF, 256, fsm, st_>>>(a, Bn, By); });
        clock.flush_ms += clock.epi_ms - e0f;
      }
      By = Bn;
      DRZG_CUDA(cudaGetLastError());
    }
  }
  return mv;
}

namespace {
// one seed bucket (column c, pole P), grouped: group gi is a state (one key),
// entries [eptr[gi], eptr[gi+1]) its distinct side rows with Ld carried digits
struct PrepBucket {
  int col = 0, pole = 0;
  bool first = false;
  std::vector<u64> key;
  std::vector<int> u;  // nv per group
  std::vector<int> eptr{0}, eg;
  std::vector<int8_t> ed;
  i64 combines = 0;  // seeds folded into an earlier seed of the same group
  bool ready = false;
};

class SeedPreparer {
 public:
  template <class KeyFn>
  SeedPreparer(std::vector<ColumnSeeds>& cols, const std::vector<int>& top0, KeyFn keyfn, int nv, int Ld, int q,
               unsigned threads)
      : nv_(nv), Ld_(Ld), q_(q) {
    for (int c = 0; c < (int)cols.size(); ++c)
      for (auto& kv : cols[c].by_pole) {
        auto pb = std::make_unique<PrepBucket>();
        pb->col = c;
        pb->pole = kv.first;
        pb->first = top0[c] == kv.first;
        order_.push_back({kv.first, c, &kv.second, pb.get()});
        index_[((u64)(u32)kv.first << 32) | (u32)c] = pb.get();
        owned_.push_back(std::move(pb));
      }
    std::stable_sort(order_.begin(), order_.end(), [](const Job& a, const Job& b) {
      return a.pole != b.pole ? a.pole > b.pole : a.col < b.col;
    });
    key_ = [keyfn](int c, const Expo& u) { return keyfn(c, u); };
    for (unsigned t = 0; t < threads; ++t) workers_.emplace_back([this] { work(); });
  }
  ~SeedPreparer() {
    stop_ = true;
    for (auto& w : workers_) w.join();
  }
  PrepBucket& wait(int c, int P) {
    PrepBucket* pb = index_.at(((u64)(u32)P << 32) | (u32)c);
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return pb->ready || err_; });
    if (err_) std::rethrow_exception(err_);
    return *pb;
  }
  void release(int c, int P) {
    PrepBucket* pb = index_.at(((u64)(u32)P << 32) | (u32)c);
    PrepBucket empty;
    std::swap(pb->key, empty.key);
    std::swap(pb->u, empty.u);
    std::swap(pb->eptr, empty.eptr);
    std::swap(pb->eg, empty.eg);
    std::swap(pb->ed, empty.ed);
  }

 private:
  struct Job {
    int pole, col;
    SeedBucket* bk;
    PrepBucket* pb;
  };
  void work() {
    for (;;) {
      if (stop_) return;
      const size_t j = next_.fetch_add(1);
      if (j >= order_.size()) return;
      try {
        prepare(order_[j]);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu_);
        if (!err_) err_ = std::current_exception();
        cv_.notify_all();
        return;
      }
      {
        std::lock_guard<std::mutex> lk(mu_);
        order_[j].pb->ready = true;
      }
      cv_.notify_all();
    }
  }
  void prepare(const Job& jb) {
    SeedBucket& bk = *jb.bk;
    PrepBucket& pb = *jb.pb;
    const int nv = nv_, Ld = Ld_, q = q_;
    const size_t ns = bk.size();
    if (pb.first) {
      // a column's first sweep keeps its seeds apart: every seed is its own
      // group with its one side row, and its digits are already balanced
      // (expand_column), so the bucket is taken over as it stands
      pb.u = std::move(bk.u);
      pb.eg = std::move(bk.g);
      pb.ed = std::move(bk.dig);
      pb.eptr.resize(ns + 1);
      for (size_t i = 0; i <= ns; ++i) pb.eptr[i] = (int)i;
      SeedBucket().u.swap(bk.u);
      SeedBucket().g.swap(bk.g);
      SeedBucket().dig.swap(bk.dig);
      return;
    }
    std::vector<u64> kv(ns);
    for (size_t i = 0; i < ns; ++i) {
      Expo u(nv);
      for (int j = 0; j < nv; ++j) u[j] = bk.u[i * nv + j];
      kv[i] = key_(jb.col, u);
    }
    std::vector<int> ord(ns);
    for (size_t i = 0; i < ns; ++i) ord[i] = (int)i;
    if (!pb.first)
      std::sort(ord.begin(), ord.end(), [&](int a, int b) { return kv[a] != kv[b] ? kv[a] < kv[b] : bk.g[a] < bk.g[b]; });
    std::vector<int> acc(Ld);
    size_t i = 0;
    while (i < ns) {
      size_t j = i + 1;
      if (!pb.first)
        while (j < ns && kv[ord[j]] == kv[ord[i]]) ++j;
      const int s0i = ord[i];
      pb.key.push_back(kv[s0i]);
      for (int t = 0; t < nv; ++t) pb.u.push_back(bk.u[(size_t)s0i * nv + t]);
      pb.combines += (i64)(j - i - 1);
      for (size_t a = i; a < j;) {
        size_t b2 = a + 1;
        while (b2 < j && bk.g[ord[b2]] == bk.g[ord[a]]) ++b2;
        std::fill(acc.begin(), acc.end(), 0);
        for (size_t x = a; x < b2; ++x)
          for (int t = 0; t < Ld; ++t) acc[t] += bk.dig[(size_t)ord[x] * Ld + t];
        int carry = 0;
        for (int t = 0; t < Ld; ++t) {
          int v = acc[t] + carry;
          int r = ((v % q) + q) % q;
          if (r > q / 2) r -= q;
          carry = (v - r) / q;
          pb.ed.push_back((int8_t)r);
        }
        pb.eg.push_back(bk.g[ord[a]]);
        a = b2;
      }
      pb.eptr.push_back((int)pb.eg.size());
      i = j;
    }
    SeedBucket().u.swap(bk.u);  // release host memory
    SeedBucket().g.swap(bk.g);
    SeedBucket().dig.swap(bk.dig);
  }

  int nv_, Ld_, q_;
  std::function<u64(int, const Expo&)> key_;
  std::vector<Job> order_;
  std::unordered_map<u64, PrepBucket*> index_;
  std::vector<std::unique_ptr<PrepBucket>> owned_;
  std::vector<std::thread> workers_;
  std::atomic<size_t> next_{0};
  std::atomic<bool> stop_{false};
  std::mutex mu_;
  std::condition_variable cv_;
  std::exception_ptr err_;
};
}  // namespace

namespace {
// seed-preparer threads (DRZG_PREP_THREADS overrides; default a quarter of
// the cores, at most 4)
unsigned prep_threads_for(unsigned host_threads) {
  static const int env = [] {
    const char* e = std::getenv("DRZG_PREP_THREADS");
    return e ? std::atoi(e) : 0;
  }();
  if (env > 0) return (unsigned)env;
  return std::max(1u, std::min(host_threads / 4, 4u));
}
}  // namespace

void ReductionEngine::run_pchunk(std::vector<ColumnSeeds>& cols, std::vector<std::vector<i64>>& G, Ledger& led) {
  const RuvTables& T = *T_;
  const int nv = T.nv, Ld = T.dp.Ld, ncol = (int)cols.size();
  // DRZG_VERBOSE: wall-clock marks of the run's stages (long-tail hunting)
  const auto wm0 = std::chrono::steady_clock::now();
  double wmark[5] = {0, 0, 0, 0, 0};
  auto wsince = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - wm0).count(); };
  // declared first, destroyed last: the time the locals' destructors take
  struct ExitMark {
    std::chrono::steady_clock::time_point t0;
    bool on;
    ~ExitMark() {
      if (on)
        std::fprintf(stderr, "[drzg] pchunk wall: exit %.3f\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
  } exit_mark{wm0, std::getenv("DRZG_VERBOSE") != nullptr};
  // key packing for combine_states' (u, pole) identity, per column
  i64 maxpole = 0;
  size_t total_seeds = 0;
  std::vector<int> top0(ncol, 0);
  for (int c = 0; c < ncol; ++c) {
    if (!cols[c].by_pole.empty()) top0[c] = cols[c].by_pole.rbegin()->first;
    maxpole = std::max<i64>(maxpole, top0[c]);
    for (auto& kv : cols[c].by_pole) total_seeds += kv.second.size();
  }
  int bits = 1;
  while (((i64)1 << bits) <= (i64)T.d * maxpole + 1) ++bits;
  int colbits = 1;
  while ((1 << colbits) < ncol) ++colbits;
  DRZG_REQUIRE(nv * bits + colbits <= 64, "engine: state key does not fit 64 bits");
  // the fp32 epilogue bound assumed exponents below 4096
  if ((i64)T.d * maxpole >= 4096) fast_ = false;
  auto key = [&](int c, const Expo& u) { return ((u64)c << (nv * bits)) | u.pack(bits); };

  cudaEvent_t run0, run1;
  DRZG_CUDA(cudaEventCreate(&run0));
  DRZG_CUDA(cudaEventCreate(&run1));
  DRZG_CUDA(cudaEventRecord(run0, st_));
  wmark[0] = wsince();
  DevBuf<long long> dG;
  dG.alloc((size_t)ncol * Ld * gsize_, st_);
  DRZG_CUDA(cudaMemsetAsync(dG.p, 0, dG.n * sizeof(long long), st_));
  DevBuf<int> d_err;
  d_err.alloc(1, st_);
  DRZG_CUDA(cudaMemsetAsync(d_err.p, 0, sizeof(int), st_));
  if (cap_ == 0) {
    // live states never exceed the seeds materialised so far: size the pool
    // for all of them when that fits 60% of free HBM (the rest feeds the
    // batch temporaries), else take the 60% and grow only if needed
    const size_t want = std::max<size_t>(1024, total_seeds / 3 + 1);
    const size_t tot_mem = device_total_memory();
    if (tot_mem && (double)want * (double)slot_stride_ < 0.05 * (double)tot_mem) {
      grow_pool((int)want);  // small: no need to ask the driver what is free
    } else {
      size_t fr = 0, tot = 0;
      mem_info(&fr, &tot, "engine.cu:6");
      size_t budget = (size_t)(fr * 0.40) / (size_t)slot_stride_;
      grow_pool((int)std::max<size_t>(1024, std::min<size_t>(want, budget)));
    }
  }

  // DRZG_TIMELINE: device time of every sweep and the device idle time
  // between sweeps (the host policy falling behind), summarised at the end
  const bool timeline = std::getenv("DRZG_TIMELINE") != nullptr;
  struct SweepMark {
    cudaEvent_t e0, e1;
    int pole;
    i64 states, matvecs;
    double t_push, t_pop, t_launched;  // host seconds since the run started
    double t_seeded, t_staged;         // ... seed work issued, sweep inputs staged
  };
  std::vector<SweepMark> tl;
  std::map<int, std::vector<HS>, std::greater<int>> landed;
  // per pole: key -> position in landed[pole]; a state landing on a key that
  // is already there is combined at once (the reference combines after every
  // sweep, reduction.hpp:502, so the ledger is unchanged)
  std::map<int, FlatMap> landed_idx;
  std::vector<FlatMap> floor_keys(ncol);
  std::vector<i64> floor_arrivals(ncol, 0);
  std::vector<std::map<int, SeedBucket>::reverse_iterator> sit(ncol);
  for (int c = 0; c < ncol; ++c) sit[c] = cols[c].by_pole.rbegin();

  // separate device buffers per use within a sweep: with the host running
  // ahead, a restaged buffer must not be one an earlier kernel of the same
  // sweep still reads (the stream orders copies and kernels, so reuse across
  // uses is safe; distinct buffers just avoid needless reallocations)
  // background preparation of every seed bucket, in consumption order
  // (descending pole): key sort, grouping by (column, u) and by side row g,
  // and the carried digit sums of each group's entries
  auto prep_owner = std::make_unique<SeedPreparer>(cols, top0, [&](int c, const Expo& u) { return key(c, u); }, nv, Ld,
                                                   T.dp.q, prep_threads_for(host_threads_));
  SeedPreparer& prep = *prep_owner;
  // The policy (moves, landing, combines, seeds, slot bookkeeping) never
  // needs a device result, so it runs on its own thread as far ahead as it
  // likes and hands every sweep to this thread as a command; this thread only
  // stages inputs and launches kernels (and is the one the CUDA launch queue
  // throttles).  The device never waits on host bookkeeping after the first
  // sweep unless the policy is slower than the device in total.
  struct SweepCmd {
    int pole = 0;
    bool done = false;
    std::vector<int> s_new, p_new, g_new, s_add, p_add, g_add;
    std::vector<int8_t> d_new, d_add;
    std::vector<int> hslot, hvdir, hu0;
    std::vector<i64> ks;
    i64 matvecs = 0;
    std::vector<int> gptr, mem;  // merges
    std::vector<int> fs, fc, fu; // floor arrivals
    double t_push = 0;           // DRZG_TIMELINE: host time the policy handed it over
  };
  std::mutex qmu;
  std::condition_variable qcv;
  std::deque<std::unique_ptr<SweepCmd>> queue;
  std::exception_ptr perr;
  auto push = [&](std::unique_ptr<SweepCmd> c) {
    if (timeline) c->t_push = wsince();
    {
      std::lock_guard<std::mutex> lk(qmu);
      queue.push_back(std::move(c));
    }
    qcv.notify_one();
  };
  // leave cores to the launcher and the seed preparers (an oversubscribed
  // launcher starves the device)
  ForkJoin move_pool((int)(host_threads_ > 6 ? host_threads_ - 4 : 2));
  std::thread policy([&] {
    const auto pol0 = std::chrono::steady_clock::now();
    struct PolicyWall {
      std::chrono::steady_clock::time_point t0;
      double* acc;
      ~PolicyWall() { *acc += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
    } policy_wall{pol0, &policy_wall_s_};
    try {
  for (;;) {
    int P = -1;
    if (!landed.empty()) P = landed.begin()->first;
    for (int c = 0; c < ncol; ++c)
      if (sit[c] != cols[c].by_pole.rend()) P = std::max(P, sit[c]->first);
    if (P <= n_) break;
    std::vector<HS> front;
    if (!landed.empty() && landed.begin()->first == P) {
      front = std::move(landed.begin()->second);
      landed.erase(landed.begin());
    }
    FlatMap front_idx(16);  // key -> position in front (states landed at P)
    {
      auto li = landed_idx.find(P);
      if (li != landed_idx.end()) front_idx.swap(li->second);
      landed_idx.erase(P);
    }
    auto hp0 = std::chrono::steady_clock::now();
    // materialise the seeds whose pole is P.  Seeds sharing (column, u) form
    // one state (the reference's combine_states of those seeds, counted in
    // the ledger); a state already landed at P absorbs them in place; a
    // column's first sweep keeps its seeds apart, as the reference does.
    // Landed states are unique per key (combined as they land), so after
    // this no two live states at P share a key.  The grouping and digit sums
    // of every seed bucket were prepared by the background workers; only
    // the (u, pole) lookups against landed states and slot allocation run here.
    auto cmd = std::make_unique<SweepCmd>();
    cmd->pole = P;
    {
      std::vector<int>& s_new = cmd->s_new; std::vector<int>& p_new = cmd->p_new; std::vector<int>& g_new = cmd->g_new;
      std::vector<int>& s_add = cmd->s_add; std::vector<int>& p_add = cmd->p_add; std::vector<int>& g_add = cmd->g_add;
      std::vector<int8_t>& d_new = cmd->d_new; std::vector<int8_t>& d_add = cmd->d_add;
      p_new.assign(1, 0);
      p_add.assign(1, 0);
      // the lookups of this pole's seed groups against the landed states
      // (cache-missing probes of a large index) on the move pool's threads
      // first, when there are many (K3's seed poles p(m+j): ~10 ms of the
      // device's wait otherwise); the index is only read
      std::vector<std::vector<int>> fposv(ncol);
      {
        std::vector<int> heavy;
        size_t total = 0;
        for (int c = 0; c < ncol; ++c) {
          if (sit[c] == cols[c].by_pole.rend() || sit[c]->first != P) continue;
          PrepBucket& pb = prep.wait(c, P);
          if (pb.first || front_idx.empty()) continue;
          heavy.push_back(c);
          total += pb.key.size();
        }
        if (total >= 16384 && move_pool.size() > 1) {
          const int nth = move_pool.size();
          move_pool.run(nth, [&](int t) {
            for (size_t h2 = t; h2 < heavy.size(); h2 += nth) {
              const int c = heavy[h2];
              PrepBucket& pb = prep.wait(c, P);
              std::vector<int>& fp = fposv[c];
              fp.resize(pb.key.size());
              for (size_t gi = 0; gi < pb.key.size(); ++gi) fp[gi] = front_idx.find(pb.key[gi]);
            }
          });
        }
      }
      for (int c = 0; c < ncol; ++c) {
        if (sit[c] == cols[c].by_pole.rend() || sit[c]->first != P) continue;
        const auto hw0 = std::chrono::steady_clock::now();
        PrepBucket& pb = prep.wait(c, P);
        prep_wait_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - hw0).count();
        led.combines += pb.combines;
        const size_t ng = pb.eptr.size() - 1;  // (first buckets carry no keys: never looked up)
        if (pb.first) {
          // a column's first bucket: every seed is its own fresh state (no
          // lookups), one side row each -- bulk copies, slots taken at once
          if (free_.size() < ng) grow_pool(cap_ + (int)(ng - free_.size()));
          const size_t f0n = front.size(), s0n = s_new.size();
          const int g0n = (int)g_new.size();
          front.resize(f0n + ng);
          s_new.resize(s0n + ng);
          for (size_t gi = 0; gi < ng; ++gi) {
            HS& h = front[f0n + gi];
            h.col = c;
            h.u = Expo(nv);
            for (int t = 0; t < nv; ++t) h.u[t] = pb.u[gi * nv + t];
            h.pole = P;
            h.slot = alloc_slot();
            s_new[s0n + gi] = h.slot;
          }
          g_new.insert(g_new.end(), pb.eg.begin(), pb.eg.end());
          d_new.insert(d_new.end(), pb.ed.begin(), pb.ed.end());
          p_new.reserve(p_new.size() + ng);
          for (size_t gi = 0; gi < ng; ++gi) p_new.push_back(g0n + pb.eptr[gi + 1]);
          prep.release(c, P);
          ++sit[c];
          continue;
        }
        // the landed-state index outgrows the caches: probe lines prefetched ahead
        constexpr size_t kPf = 8;
        if (!pb.first)
          for (size_t gi = 0; gi < std::min(ng, kPf); ++gi) front_idx.prefetch(pb.key[gi]);
        const std::vector<int>& fp = fposv[c];
        for (size_t gi = 0; gi < ng; ++gi) {
          if (fp.empty() && !pb.first && gi + kPf < ng) front_idx.prefetch(pb.key[gi + kPf]);
          const int fpos = !fp.empty() ? fp[gi] : pb.first ? -1 : front_idx.find(pb.key[gi]);
          const int e0 = pb.eptr[gi], e1 = pb.eptr[gi + 1];
          if (fpos >= 0) {
            led.combines += 1;
            s_add.push_back(front[fpos].slot);
            g_add.insert(g_add.end(), pb.eg.begin() + e0, pb.eg.begin() + e1);
            d_add.insert(d_add.end(), pb.ed.begin() + (size_t)e0 * Ld, pb.ed.begin() + (size_t)e1 * Ld);
            p_add.push_back((int)g_add.size());
          } else {
            HS h;
            h.col = c;
            h.u = Expo(nv);
            for (int t = 0; t < nv; ++t) h.u[t] = pb.u[gi * nv + t];
            h.pole = P;
            h.slot = alloc_slot();
            front.push_back(h);
            s_new.push_back(h.slot);
            g_new.insert(g_new.end(), pb.eg.begin() + e0, pb.eg.begin() + e1);
            d_new.insert(d_new.end(), pb.ed.begin() + (size_t)e0 * Ld, pb.ed.begin() + (size_t)e1 * Ld);
            p_new.push_back((int)g_new.size());
          }
        }
        prep.release(c, P);
        ++sit[c];
      }
    }
    auto hp1 = std::chrono::steady_clock::now();
    auto hp2 = hp1;
    // the front is handed to the launcher in chunks of states (each sorted
    // by (k, v) on its own), so the device starts on a sweep before the
    // policy has finished it; the seed work of pole P rides with chunk 0
    // (DRZG_CHUNK0 < 17: chunks double from 2^CHUNK0 states, so the device
    // gets a pole's first states after a shorter policy step; measured no
    // better on K3, whose smaller batches cost more than the wait saves)
    const size_t nfront = front.size();
    constexpr size_t kChunk = (size_t)1 << 17;
    static const int chunk0 = [] {
      const char* e = std::getenv("DRZG_CHUNK0");  // A/B: log2 of a pole's first chunk
      return e ? std::min(17, std::max(8, std::atoi(e))) : 17;  // K3: 2^17 beat 2^13 (0.221 vs 0.229 s)
    }();
    size_t chunk = (size_t)1 << chunk0;
    for (size_t f0 = 0, nf = 0; f0 < nfront; f0 += nf, chunk = std::min(kChunk, 2 * chunk)) {
      if (f0) {
        cmd = std::make_unique<SweepCmd>();
        cmd->pole = P;
      }
      nf = std::min(nfront, f0 + chunk) - f0;
      // moves (reduction.hpp:486-496) for every state, on host threads
      const auto hp1m = std::chrono::steady_clock::now();
      std::vector<int> vd(nf);
      std::vector<i64> kk(nf);
      {
        const int nth = (int)std::max<size_t>(1, std::min<size_t>(move_pool.size(), nf / 4096 + 1));
        std::vector<std::exception_ptr> errs(nth);
        auto moves = [&](int t) {
          try {
            for (size_t i = t * nf / nth; i < (t + 1) * nf / nth; ++i) {
              Expo v;
              i64 k;
              pchunk_move(T.d, n_, (i64)p_, front[f0 + i].u, front[f0 + i].pole, T.S, &v, &k);
              DRZG_REQUIRE(k >= 1, "p-chunk: no admissible move");
              DRZG_REQUIRE(legal(T.d, front[f0 + i].u, v, k, T.S), "reduce_chunk: illegal move");
              vd[i] = (int)rank_of(v);
              kk[i] = k;
            }
          } catch (...) {
            errs[t] = std::current_exception();
          }
        };
        if (nth == 1)
          moves(0);  // small sweeps: no hand-off on the policy's critical path
        else
          move_pool.run(nth, moves);
        for (auto& e2 : errs)
          if (e2) std::rethrow_exception(e2);
      }
      const auto hm1 = std::chrono::steady_clock::now();
      moves_only_s_ += std::chrono::duration<double>(hm1 - hp1m).count();
      // longest chunks first, then by direction: counting sort on (k, v)
      // (the front is read in its own order and the sorted arrays written by
      // position: sequential reads of the 40-byte states, not random ones)
      std::vector<int> order(nf), pos(nf);
      {
        const int ndir = T.ndir;
        i64 kmx = 1;
        for (i64 k : kk) kmx = std::max(kmx, k);
        std::vector<int> cnt((size_t)(kmx + 1) * ndir + 1, 0);
        auto bucket = [&](size_t i) { return (size_t)(kmx - kk[i]) * ndir + vd[i]; };
        for (size_t i = 0; i < nf; ++i) ++cnt[bucket(i) + 1];
        for (size_t b = 1; b < cnt.size(); ++b) cnt[b] += cnt[b - 1];
        for (size_t i = 0; i < nf; ++i) {
          const int o = cnt[bucket(i)]++;
          pos[i] = o;
          order[o] = (int)i;
        }
      }
      std::vector<int>& hslot = cmd->hslot;
      std::vector<int>& hvdir = cmd->hvdir;
      std::vector<int>& hu0 = cmd->hu0;
      std::vector<i64>& ks = cmd->ks;
      hslot.resize(nf);
      hvdir.resize(nf);
      hu0.resize(nf * nv);
      ks.resize(nf);
      for (size_t i = 0; i < nf; ++i) {
        const int o = pos[i];
        const HS& h = front[f0 + i];
        hslot[o] = h.slot;
        hvdir[o] = vd[i];
        ks[o] = kk[i];
        for (int j = 0; j < nv; ++j) hu0[(size_t)o * nv + j] = h.u[j];
      }
      auto hp3 = std::chrono::steady_clock::now();
      for (i64 k : ks) cmd->matvecs += k;  // run_sweep: one matvec per state per step
      led.matvecs += cmd->matvecs;
      auto hp4 = std::chrono::steady_clock::now();
      led.startups += (i64)nf;
      // the sweep goes to the launcher now; its landing (merges, floor
      // arrivals) follows as a second command, so the device starts on the
      // chunk while the policy lands it
      push(std::move(cmd));
      cmd = std::make_unique<SweepCmd>();
      cmd->pole = P;
      // land every state at pole P - k; a state landing on a key already there
      // is combined at once (reduction.hpp:502 combines after every sweep)
      std::vector<int>& fs = cmd->fs;
      std::vector<int>& fc = cmd->fc;
      std::vector<int>& fu = cmd->fu;
      std::vector<std::pair<int, int>> merges;  // (dst slot, src slot)
      // states are landed in the front's own order (sequential reads); the
      // landing pole's index and list are looked up once per chunk length k,
      // and the probe lines of the keys kPf states ahead are prefetched (the
      // per-pole maps outgrow the caches)
      i64 kmax_c = 1;
      for (i64 k : kk) kmax_c = std::max(kmax_c, k);
      std::vector<FlatMap*> kidx((size_t)kmax_c + 1, nullptr);
      std::vector<std::vector<HS>*> klst((size_t)kmax_c + 1, nullptr);
      std::vector<char> kseen((size_t)kmax_c + 1, 0);
      for (i64 k : kk) kseen[k] = 1;
      for (i64 k = 1; k <= kmax_c; ++k)
        if (kseen[k] && P - (int)k != n_) {
          kidx[k] = &landed_idx[P - (int)k];
          klst[k] = &landed[P - (int)k];
        }
      std::vector<u64> lkey(nf);
      for (size_t i = 0; i < nf; ++i) {
        Expo u = front[f0 + i].u;
        const Expo& v = dirs_host_[vd[i]];
        for (int j = 0; j < nv; ++j) u[j] -= (int)(kk[i] * v[j]);
        lkey[i] = key(front[f0 + i].col, u);
      }
      constexpr size_t kPf = 8;
      for (size_t i = 0; i < nf; ++i) {
        if (i + kPf < nf && kidx[kk[i + kPf]]) kidx[kk[i + kPf]]->prefetch(lkey[i + kPf]);
        HS h = front[f0 + i];
        const Expo& v = dirs_host_[vd[i]];
        for (int j = 0; j < nv; ++j) h.u[j] -= (int)(kk[i] * v[j]);
        h.pole -= (int)kk[i];
        const u64 kh = lkey[i];
        if (h.pole == n_) {
          fs.push_back(h.slot);
          fc.push_back(h.col);
          for (int j = 0; j < nv; ++j) fu.push_back(h.u[j]);
          floor_arrivals[h.col]++;
          floor_keys[h.col].insert(kh, 0);
        } else {
          FlatMap& idx = *kidx[kk[i]];
          std::vector<HS>& lst = *klst[kk[i]];
          const int pos_l = idx.insert(kh, (int)lst.size());
          if (pos_l == (int)lst.size()) {
            lst.push_back(h);
          } else {
            merges.emplace_back(lst[pos_l].slot, h.slot);
            led.combines += 1;
          }
        }
      }
      if (!merges.empty()) {
        std::sort(merges.begin(), merges.end());
        std::vector<int>& gptr = cmd->gptr;
        std::vector<int>& mem = cmd->mem;
        gptr.assign(1, 0);
        for (size_t a = 0; a < merges.size();) {
          size_t b2 = a;
          mem.push_back(merges[a].first);
          while (b2 < merges.size() && merges[b2].first == merges[a].first) mem.push_back(merges[b2++].second);
          gptr.push_back((int)mem.size());
          a = b2;
        }
        for (auto& m : merges) free_slot(m.second);
      }
      auto hp5 = std::chrono::steady_clock::now();
      {
        auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        host_t_[0] += sec(hp0, hp1);
        host_t_[1] += sec(hp1, hp2);
        host_t_[2] += sec(hp1m, hp3);  // this chunk's moves, sort and command arrays
        (void)hp2;
        (void)hp4;  // launch time is accounted by the launcher
        host_t_[4] += sec(hp4, hp5);
      }
      for (int s : fs) free_slot(s);
      push(std::move(cmd));
    }
    if (cmd) push(std::move(cmd));  // seeds of a pole with no states left (none expected)
  }
    } catch (...) {
      perr = std::current_exception();
    }
    auto fin = std::make_unique<SweepCmd>();
    fin->done = true;
    push(std::move(fin));
  });
  // launcher: stage and launch every sweep's work in policy order
  DevBuf<int> d_a, d_b, d_c, d_s2, d_p2, d_g2, d_mp, d_mm;
  DevBuf<int8_t> d_dig, d_dig2;
  try {
    for (;;) {
      std::unique_ptr<SweepCmd> cmd;
      {
        std::unique_lock<std::mutex> lk(qmu);
        qcv.wait(lk, [&] { return !queue.empty(); });
        cmd = std::move(queue.front());
        queue.pop_front();
      }
      if (cmd->done) break;
      auto hl0 = std::chrono::steady_clock::now();
      // fresh slots are zeroed and written; absorbed groups add in place
      if (!cmd->s_new.empty()) {
        d_a.stage(cmd->s_new, stager_, st_);
        d_b.stage(cmd->p_new, stager_, st_);
        d_c.stage(cmd->g_new, stager_, st_);
        d_dig.stage(cmd->d_new, stager_, st_);
        const int ns = (int)cmd->s_new.size();
        timed(&clock.other_ms, [&] {
          dev::seed_kernel<<<ns, 128, 0, st_>>>(pool_, slot_stride_, sidep_, Ld, d_a.p, d_b.p, d_c.p, d_dig.p, ns);
        });
      }
      if (!cmd->s_add.empty()) {
        d_s2.stage(cmd->s_add, stager_, st_);
        d_p2.stage(cmd->p_add, stager_, st_);
        d_g2.stage(cmd->g_add, stager_, st_);
        d_dig2.stage(cmd->d_add, stager_, st_);
        const int ns = (int)cmd->s_add.size();
        timed(&clock.other_ms, [&] {
          dev::add_entries_kernel<<<ns, 128, 0, st_>>>(pool_, slot_stride_, sidep_, Ld, T.dp.q, d_s2.p, d_p2.p,
                                                      d_g2.p, d_dig2.p, ns);
        });
      }
      const double t_seeded = timeline ? wsince() : 0;
      if (!cmd->ks.empty()) {
        d_slot_.stage(cmd->hslot, stager_, st_);
        d_vdir_.stage(cmd->hvdir, stager_, st_);
        d_u0_.stage(cmd->hu0, stager_, st_);
        d_k_.stage(cmd->ks, stager_, st_);
        if (timeline) {
          cudaEvent_t e0, e1;
          DRZG_CUDA(cudaEventCreate(&e0));
          DRZG_CUDA(cudaEventCreate(&e1));
          const double tp = std::chrono::duration<double>(hl0 - wm0).count();
          const double t_staged = wsince();
          DRZG_CUDA(cudaEventRecord(e0, st_));
          run_sweep(cmd->ks);
          DRZG_CUDA(cudaEventRecord(e1, st_));
          tl.push_back({e0, e1, cmd->pole, (i64)cmd->ks.size(), cmd->matvecs, cmd->t_push, tp, wsince(), t_seeded,
                        t_staged});
        } else {
          run_sweep(cmd->ks);
        }
      }
      if (cmd->gptr.size() > 1) {
        d_mp.stage(cmd->gptr, stager_, st_);
        d_mm.stage(cmd->mem, stager_, st_);
        const size_t ng = cmd->gptr.size() - 1;
        timed(&clock.other_ms, [&] {
          dev::launch_merge(pool_, slot_stride_, T.side, sidep_, Ld, FastQ::make(T.dp.q), d_mp.p, d_mm.p, (int)ng, st_);
        });
      }
      if (!cmd->fs.empty()) {
        d_a.stage(cmd->fs, stager_, st_);
        d_b.stage(cmd->fc, stager_, st_);
        d_c.stage(cmd->fu, stager_, st_);
        dim3 gf((unsigned)((T.side + 127) / 128) * cmd->fs.size());
        timed(&clock.other_ms, [&] {
          dev::floor_kernel<<<gf, 128, 0, st_>>>(pool_, slot_stride_, T.side, sidep_, Ld, nv, d_a.p, d_b.p, d_c.p,
                                                 mon_.p, btab_.p, dG.p, gsize_, d_err.p);
        });
      }
      host_t_[3] += std::chrono::duration<double>(std::chrono::steady_clock::now() - hl0).count();
    }
  } catch (...) {
    // drain: let the policy thread finish before unwinding
    for (;;) {
      std::unique_lock<std::mutex> lk(qmu);
      qcv.wait(lk, [&] { return !queue.empty(); });
      bool d = queue.back()->done;
      queue.clear();
      if (d) break;
    }
    policy.join();
    throw;
  }
  wmark[1] = wsince();
  policy.join();
  wmark[2] = wsince();
  if (perr) std::rethrow_exception(perr);
  for (int c = 0; c < ncol; ++c) led.combines += floor_arrivals[c] - (i64)floor_keys[c].size();
  if (timeline && !tl.empty()) {
    DRZG_CUDA(cudaStreamSynchronize(st_));
    double busy = 0, idle = 0, lead = 0;
    float ms = 0;
    DRZG_CUDA(cudaEventElapsedTime(&ms, run0, tl[0].e0));
    lead = ms;
    std::map<int, std::pair<double, double>> by_pole;  // pole -> (busy, idle before)
    for (size_t i = 0; i < tl.size(); ++i) {
      DRZG_CUDA(cudaEventElapsedTime(&ms, tl[i].e0, tl[i].e1));
      busy += ms;
      by_pole[tl[i].pole].first += ms;
      if (i) {
        float g2 = 0;
        DRZG_CUDA(cudaEventElapsedTime(&g2, tl[i - 1].e1, tl[i].e0));
        idle += g2;
        by_pole[tl[i].pole].second += g2;
      }
    }
    std::fprintf(stderr, "[drzg] timeline: %zu sweeps, before first %.1f ms, sweeps %.1f ms, between sweeps %.1f ms\n",
                 tl.size(), lead, busy, idle);
    std::fprintf(stderr, "[drzg]   host waits (process, ms): ring %.1f pinned %.1f copy %.1f malloc %.1f\n",
                 g_waits.ring_ns / 1e6, g_waits.pinned_ns / 1e6, g_waits.copy_ns / 1e6, g_waits.malloc_ns / 1e6);
    g_waits.reset();
    // the largest device gaps, with the host times (ms since the run began,
    // device times on the same base via run0) of the sweep that ended them
    {
      const double r0 = wmark[0] * 1e3;
      std::vector<std::pair<float, size_t>> gaps;
      for (size_t i = 1; i < tl.size(); ++i) {
        float g2 = 0;
        DRZG_CUDA(cudaEventElapsedTime(&g2, tl[i - 1].e1, tl[i].e0));
        gaps.push_back({g2, i});
      }
      std::sort(gaps.rbegin(), gaps.rend());
      for (size_t j = 0; j < gaps.size() && j < 6 && gaps[j].first > 1.0f; ++j) {
        const size_t i = gaps[j].second;
        float d0 = 0, d1 = 0;
        DRZG_CUDA(cudaEventElapsedTime(&d0, run0, tl[i - 1].e1));
        DRZG_CUDA(cudaEventElapsedTime(&d1, run0, tl[i].e0));
        std::fprintf(stderr,
                     "[drzg]   gap %.2f ms before sweep %zu (pole %d, %lld states): device idle %.2f..%.2f, "
                     "policy pushed %.2f, launcher popped %.2f, seeded %.2f, staged %.2f, launched %.2f (prev "
                     "launched %.2f)\n",
                     gaps[j].first, i, tl[i].pole, (long long)tl[i].states, d0 + r0, d1 + r0, tl[i].t_push * 1e3,
                     tl[i].t_pop * 1e3, tl[i].t_seeded * 1e3, tl[i].t_staged * 1e3, tl[i].t_launched * 1e3,
                     tl[i - 1].t_launched * 1e3);
      }
    }
    for (auto& kv : by_pole)
      if (kv.second.first + kv.second.second > 20)
        std::fprintf(stderr, "[drzg]   pole %d: sweep %.1f ms, gap before %.1f ms\n", kv.first, kv.second.first,
                     kv.second.second);
    for (auto& m : tl) {
      cudaEventDestroy(m.e0);
      cudaEventDestroy(m.e1);
    }
  }
  if (std::getenv("DRZG_VERBOSE"))
    std::fprintf(stderr, "[drzg] host s: seeds %.3f (waiting for the preparers %.3f) combine %.3f moves %.3f (the moves themselves %.3f) launch %.3f land %.3f; policy thread wall %.3f\n",
                 host_t_[0], prep_wait_s_, host_t_[1], host_t_[2], moves_only_s_, host_t_[3], host_t_[4], policy_wall_s_);
  std::vector<long long> hG(dG.n);
  DRZG_CUDA(cudaMemcpyAsync(hG.data(), dG.p, dG.n * sizeof(long long), cudaMemcpyDeviceToHost, st_));
  g_traffic.d2h += (long long)(dG.n * sizeof(long long));
  DRZG_CUDA(cudaEventRecord(run1, st_));
  wmark[3] = wsince();
  DRZG_CUDA(cudaStreamSynchronize(st_));
  wmark[4] = wsince();
  if (std::getenv("DRZG_VERBOSE"))
    std::fprintf(stderr, "[drzg] pchunk wall: run0 %.3f loop %.3f join %.3f run1 %.3f sync %.3f\n", wmark[0], wmark[1],
                 wmark[2], wmark[3], wmark[4]);
  {
    float ms = 0;
    DRZG_CUDA(cudaEventElapsedTime(&ms, run0, run1));
    clock.device_ms += ms;
    cudaEventDestroy(run0);
    cudaEventDestroy(run1);
  }
  DRZG_CUDA(cudaGetLastError());
  G.assign(ncol, {});
  for (int c = 0; c < ncol; ++c)
    G[c].assign(hG.begin() + (size_t)c * Ld * gsize_, hG.begin() + (size_t)(c + 1) * Ld * gsize_);
  if (exit_mark.on) {
    // which local's destruction is slow (long-tail hunting)
    const double a0 = wsince();
    prep_owner.reset();
    const double a1 = wsince();
    { auto tmp = std::move(landed); }
    { auto tmp = std::move(landed_idx); }
    const double a2 = wsince();
    { auto tmp = std::move(floor_keys); }
    const double a3 = wsince();
    d_a.release(); d_b.release(); d_c.release(); d_s2.release(); d_p2.release(); d_g2.release();
    d_mp.release(); d_mm.release(); d_dig.release(); d_dig2.release();
    const double a4 = wsince();
    dG.release(); d_err.release();
    const double a5 = wsince();
    std::fprintf(stderr, "[drzg] pchunk wall: return %.3f prep %.3f landed %.3f floor %.3f devbufs %.3f dG %.3f\n", a0,
                 a1 - a0, a2 - a1, a3 - a2, a4 - a3, a5 - a4);
  }
}

void ReductionEngine::chunk_batch(const std::vector<Expo>& u, const std::vector<int>& vdir, const std::vector<i64>& k,
                                  std::vector<i8>& w_digits, Ledger& led) {
  const RuvTables& T = *T_;
  const int nv = T.nv, Ld = T.dp.Ld, B = (int)u.size();
  DRZG_REQUIRE(w_digits.size() == (size_t)B * Ld * T.side, "chunk_batch: digit array size");
  while ((int)free_.size() < B) grow_pool(cap_ + B);
  std::vector<int> slots(B);
  for (int i = 0; i < B; ++i) slots[i] = alloc_slot();
  // upload digits slot by slot (pitch sidep)
  std::vector<int8_t> stage((size_t)slot_stride_, 0);
  for (int i = 0; i < B; ++i) {
    std::fill(stage.begin(), stage.end(), 0);
    for (int t = 0; t < Ld; ++t)
      for (int g = 0; g < T.side; ++g) stage[(size_t)t * sidep_ + g] = w_digits[((size_t)i * Ld + t) * T.side + g];
    DRZG_CUDA(cudaMemcpy(pool_ + (size_t)slots[i] * slot_stride_, stage.data(), stage.size(), cudaMemcpyHostToDevice));
  }
  std::vector<int> order(B);
  for (int i = 0; i < B; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return k[a] != k[b] ? k[a] > k[b] : vdir[a] < vdir[b]; });
  std::vector<int> hslot, hvdir, hu0;
  std::vector<i64> ks;
  for (int i : order) {
    ks.push_back(k[i]);
    DRZG_REQUIRE(k[i] >= 1, "reduce_chunk: empty chunk");
    DRZG_REQUIRE(legal(T.d, u[i], dirs_host_[vdir[i]], k[i], T.S), "reduce_chunk: illegal move");
    hslot.push_back(slots[i]);
    hvdir.push_back(vdir[i]);
    for (int j = 0; j < nv; ++j) hu0.push_back(u[i][j]);
  }
  d_slot_.stage(hslot, stager_, st_);
  d_vdir_.stage(hvdir, stager_, st_);
  d_u0_.stage(hu0, stager_, st_);
  d_k_.stage(ks, stager_, st_);
  led.matvecs += run_sweep(ks);
  led.startups += B;
  for (int i = 0; i < B; ++i) {
    DRZG_CUDA(cudaMemcpyAsync(stage.data(), pool_ + (size_t)slots[i] * slot_stride_, stage.size(),
                              cudaMemcpyDeviceToHost, st_));
    DRZG_CUDA(cudaStreamSynchronize(st_));
    for (int t = 0; t < Ld; ++t)
      for (int g = 0; g < T.side; ++g) w_digits[((size_t)i * Ld + t) * T.side + g] = stage[(size_t)t * sidep_ + g];
    free_slot(slots[i]);
  }
}


// ---------------------------------------------------------------------------
// State-level primitives and the round-based policies.

std::vector<int> ReductionEngine::seed_states(const std::vector<int>& eptr, const std::vector<int>& eg,
                                              const std::vector<i8>& edig) {
  const int ns = (int)eptr.size() - 1;
  std::vector<int> slots(ns);
  if (ns <= 0) return slots;
  while ((int)free_.size() < ns) grow_pool(cap_ + ns);
  for (int i = 0; i < ns; ++i) slots[i] = alloc_slot();
  DevBuf<int> da, db, dc;
  DevBuf<int8_t> dd;
  da.upload(slots, st_);
  db.upload(eptr, st_);
  dc.upload(eg, st_);
  dd.upload(std::vector<int8_t>(edig.begin(), edig.end()), st_);
  timed(&clock.other_ms, [&] {
    dev::seed_kernel<<<ns, 128, 0, st_>>>(pool_, slot_stride_, sidep_, T_->dp.Ld, da.p, db.p, dc.p, dd.p, ns);
  });
  DRZG_CUDA(cudaGetLastError());
  DRZG_CUDA(cudaStreamSynchronize(st_));
  return slots;
}

void ReductionEngine::step_states(const std::vector<Live*>& sts, const std::vector<int>& vdir,
                                  const std::vector<i64>& k, Ledger& led) {
  const RuvTables& T = *T_;
  const int B = (int)sts.size();
  if (!B) return;
  std::vector<int> order(B);
  for (int i = 0; i < B; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return k[a] != k[b] ? k[a] > k[b] : vdir[a] < vdir[b]; });
  std::vector<int> hslot, hvdir, hu0;
  std::vector<i64> ks;
  i64 maxpole = 0;
  for (int i : order) {
    const Live& s = *sts[i];
    const Expo& v = dirs_host_.at(vdir[i]);
    DRZG_REQUIRE(k[i] >= 1, "reduce_chunk: empty chunk");
    DRZG_REQUIRE(legal(T.d, s.u, v, k[i], T.S), "reduce_chunk: illegal move");
    DRZG_REQUIRE(s.pole - k[i] >= n_, "reduce_chunk: chunk passes the floor");
    maxpole = std::max<i64>(maxpole, s.pole);
    ks.push_back(k[i]);
    hslot.push_back(s.slot);
    hvdir.push_back(vdir[i]);
    for (int j = 0; j < T.nv; ++j) hu0.push_back(s.u[j]);
  }
  // the multiply-high T_x epilogue assumes exponents below 4096 (x = u - y v < d * pole)
  const bool fast_saved = fast_;
  if ((i64)T.d * maxpole >= 4096) fast_ = false;
  d_slot_.stage(hslot, stager_, st_);
  d_vdir_.stage(hvdir, stager_, st_);
  d_u0_.stage(hu0, stager_, st_);
  d_k_.stage(ks, stager_, st_);
  led.matvecs += run_sweep(ks);
  led.startups += B;
  fast_ = fast_saved;
  for (int i = 0; i < B; ++i) {
    Live& s = *sts[i];
    const Expo& v = dirs_host_[vdir[i]];
    for (int j = 0; j < T.nv; ++j) s.u[j] -= (int)(k[i] * v[j]);
    s.pole -= (int)k[i];
  }
}

void ReductionEngine::combine_live(std::vector<Live>& sts, Ledger& led) {
  const RuvTables& T = *T_;
  std::unordered_map<std::string, int> first;  // key -> position in out
  std::vector<Live> out;
  std::vector<std::vector<int>> groups;        // per out position: merged slots (first = keeper)
  out.reserve(sts.size());
  for (auto& s : sts) {
    std::string key((const char*)s.u.e, sizeof(int) * s.u.nv);
    key.append((const char*)&s.pole, sizeof(int));
    key.append((const char*)&s.col, sizeof(int));
    auto it = first.find(key);
    if (it == first.end()) {
      first.emplace(std::move(key), (int)out.size());
      groups.push_back({s.slot});
      out.push_back(s);
    } else {
      groups[it->second].push_back(s.slot);
      led.combines += 1;
    }
  }
  std::vector<int> gptr{0}, mem, freed;
  for (auto& g : groups) {
    if (g.size() < 2) continue;
    mem.insert(mem.end(), g.begin(), g.end());
    gptr.push_back((int)mem.size());
    freed.insert(freed.end(), g.begin() + 1, g.end());
  }
  if (gptr.size() > 1) {
    DevBuf<int> dp, dm;
    dp.upload(gptr, st_);
    dm.upload(mem, st_);
    const size_t ng = gptr.size() - 1;
    timed(&clock.other_ms, [&] {
      dev::launch_merge(pool_, slot_stride_, T.side, sidep_, T.dp.Ld, FastQ::make(T.dp.q), dp.p, dm.p, (int)ng, st_);
    });
    DRZG_CUDA(cudaGetLastError());
    DRZG_CUDA(cudaStreamSynchronize(st_));
  }
  for (int f : freed) free_slot(f);
  sts.swap(out);
}

void ReductionEngine::run_policy_live(std::vector<Live>& sts, Policy pol, Ledger& led) {
  const RuvTables& T = *T_;
  const int n = n_, d = T.d;
  auto active = [&](const Live& s) { return s.pole > n; };
  std::vector<Live*> batch;
  std::vector<int> vd;
  std::vector<i64> kk;
  auto flush = [&] {
    step_states(batch, vd, kk, led);
    batch.clear();
    vd.clear();
    kk.clear();
  };
  if (pol == Policy::depth_first) {
    // every state chunk after chunk to the floor, never combined
    // (reduction.hpp:472-483); states move in lockstep rounds, which changes
    // no state's trajectory
    for (;;) {
      for (auto& s : sts) {
        if (!active(s)) continue;
        Expo v = choose_v_greedy(d, s.u, T.S);
        repair_v(s.u, v, T.S);
        const i64 k = std::min<i64>(k_max_legal(s.u, v, T.S), (i64)s.pole - n);
        DRZG_REQUIRE(k >= 1, "depth-first: no admissible move");
        batch.push_back(&s);
        vd.push_back((int)rank_of(v));
        kk.push_back(k);
      }
      if (batch.empty()) break;
      flush();
    }
    return;
  }
  if (pol == Policy::p_chunk) {
    // reduction.hpp:486-503: per sweep the states at the top |u| take
    // k = min(p, pole - n, k_max) along the greedy v, then combine_states
    for (;;) {
      int top = -1;
      for (auto& s : sts)
        if (active(s)) top = std::max(top, s.u.total());
      if (top < 0) break;
      for (auto& s : sts) {
        if (!active(s) || s.u.total() != top) continue;
        Expo v;
        i64 k;
        pchunk_move(d, n, (i64)p_, s.u, s.pole, T.S, &v, &k);
        DRZG_REQUIRE(k >= 1, "p-chunk: no admissible move");
        batch.push_back(&s);
        vd.push_back((int)rank_of(v));
        kk.push_back(k);
      }
      flush();
      combine_live(sts, led);
    }
    return;
  }
  // var-by-var (reduction.hpp:507-532): stages t = n..0 over S = {n}; u_t is
  // driven to 0 (t in S) or 1, with a combine between stages
  DRZG_REQUIRE(T.S == (1u << n), "var-by-var: working set must be {n}");
  for (int t = n; t >= 0; --t) {
    const int target = ((T.S >> t) & 1u) ? 0 : 1;
    const unsigned stage = 1u << t;
    for (;;) {
      for (auto& s : sts) {
        if (!active(s) || s.u[t] <= target) continue;
        Expo v = choose_v_greedy(d, s.u, stage);
        repair_v(s.u, v, T.S);
        i64 k = std::min<i64>(k_max_legal(s.u, v, T.S), (i64)s.pole - n);
        if (v[t] > 0) k = std::min<i64>(k, ((i64)s.u[t] - target) / v[t]);
        DRZG_REQUIRE(k >= 1, "var-by-var: no admissible move");
        batch.push_back(&s);
        vd.push_back((int)rank_of(v));
        kk.push_back(k);
      }
      if (batch.empty()) break;
      flush();
    }
    combine_live(sts, led);
  }
  for (auto& s : sts) DRZG_REQUIRE(!active(s), "var-by-var: states left above the floor");
}

void ReductionEngine::floor_accumulate(const std::vector<Live>& sts, long long* dG, int ncols) {
  const RuvTables& T = *T_;
  if (sts.empty()) return;
  std::vector<int> fs, fc, fu;
  for (auto& s : sts) {
    DRZG_REQUIRE(s.pole == n_, "floor_to_numerator: not at the floor");
    DRZG_REQUIRE(s.col >= 0 && s.col < ncols, "floor_accumulate: column out of range");
    fs.push_back(s.slot);
    fc.push_back(s.col);
    for (int j = 0; j < T.nv; ++j) fu.push_back(s.u[j]);
  }
  DevBuf<int> da, db, dc, derr;
  da.upload(fs, st_);
  db.upload(fc, st_);
  dc.upload(fu, st_);
  derr.alloc(1, st_);
  DRZG_CUDA(cudaMemsetAsync(derr.p, 0, sizeof(int), st_));
  dim3 gf((unsigned)((T.side + 127) / 128) * fs.size());
  timed(&clock.other_ms, [&] {
    dev::floor_kernel<<<gf, 128, 0, st_>>>(pool_, slot_stride_, T.side, sidep_, T.dp.Ld, T.nv, da.p, db.p, dc.p,
                                           mon_.p, btab_.p, dG, gsize_, derr.p);
  });
  DRZG_CUDA(cudaGetLastError());
  DRZG_CUDA(cudaStreamSynchronize(st_));
}

std::vector<i8> ReductionEngine::read_states(const std::vector<int>& slots) {
  const RuvTables& T = *T_;
  const int Ld = T.dp.Ld;
  std::vector<i8> out((size_t)slots.size() * Ld * T.side);
  std::vector<int8_t> stage((size_t)slot_stride_);
  for (size_t i = 0; i < slots.size(); ++i) {
    DRZG_CUDA(cudaMemcpyAsync(stage.data(), pool_ + (size_t)slots[i] * slot_stride_, stage.size(),
                              cudaMemcpyDeviceToHost, st_));
    DRZG_CUDA(cudaStreamSynchronize(st_));
    for (int t = 0; t < Ld; ++t)
      for (int g = 0; g < T.side; ++g) out[(i * Ld + t) * T.side + g] = stage[(size_t)t * sidep_ + g];
  }
  g_traffic.d2h += (long long)(slots.size() * slot_stride_);
  return out;
}

void ReductionEngine::write_state(int slot, const std::vector<i8>& digits) {
  const RuvTables& T = *T_;
  const int Ld = T.dp.Ld;
  DRZG_REQUIRE(digits.size() == (size_t)Ld * T.side, "write_state: digit array size");
  std::vector<int8_t> stage((size_t)slot_stride_, 0);
  for (int t = 0; t < Ld; ++t)
    for (int g = 0; g < T.side; ++g) stage[(size_t)t * sidep_ + g] = digits[(size_t)t * T.side + g];
  DRZG_CUDA(cudaMemcpyAsync(pool_ + (size_t)slot * slot_stride_, stage.data(), stage.size(), cudaMemcpyHostToDevice,
                            st_));
  DRZG_CUDA(cudaStreamSynchronize(st_));
  g_traffic.h2d += (long long)stage.size();
}

void ReductionEngine::release_slots(const std::vector<int>& slots) {
  for (int s : slots) free_slot(s);
}

void ReductionEngine::run_rounds(std::vector<ColumnSeeds>& cols, std::vector<std::vector<i64>>& G, Ledger& led,
                                 Policy pol) {
  const RuvTables& T = *T_;
  const int nv = T.nv, Ld = T.dp.Ld, ncol = (int)cols.size();
  cudaEvent_t run0, run1;
  DRZG_CUDA(cudaEventCreate(&run0));
  DRZG_CUDA(cudaEventCreate(&run1));
  DRZG_CUDA(cudaEventRecord(run0, st_));
  DevBuf<long long> dG;
  dG.alloc((size_t)ncol * Ld * gsize_, st_);
  DRZG_CUDA(cudaMemsetAsync(dG.p, 0, dG.n * sizeof(long long), st_));
  // every seed is its own state (the reference seeds one GameState per term,
  // zeta.hpp:66-69); depth-first never combines, so its states may run in
  // waves that fit the pool; var-by-var combines across all of a column's
  // states, so a column runs whole
  size_t fr = 0, tot = 0;
  mem_info(&fr, &tot, "engine.cu:7");
  const size_t wave = std::max<size_t>(1024, (size_t)(fr * 0.4) / (size_t)slot_stride_);
  for (int c = 0; c < ncol; ++c) {
    std::vector<Live> sts;
    std::vector<int> eptr{0}, eg;
    std::vector<i8> ed;
    auto run_wave = [&] {
      if (sts.empty()) return;
      std::vector<int> slots = seed_states(eptr, eg, ed);
      for (size_t i = 0; i < sts.size(); ++i) sts[i].slot = slots[i];
      run_policy_live(sts, pol, led);
      floor_accumulate(sts, dG.p, ncol);
      std::vector<int> fsl;
      for (auto& s : sts) fsl.push_back(s.slot);
      release_slots(fsl);
      sts.clear();
      eptr.assign(1, 0);
      eg.clear();
      ed.clear();
    };
    for (auto& kv : cols[c].by_pole) {
      const SeedBucket& bk = kv.second;
      for (size_t i = 0; i < bk.size(); ++i) {
        Live s;
        s.col = c;
        s.u = Expo(nv);
        for (int j = 0; j < nv; ++j) s.u[j] = bk.u[i * nv + j];
        s.pole = kv.first;
        sts.push_back(s);
        eg.push_back(bk.g[i]);
        ed.insert(ed.end(), bk.dig.begin() + i * Ld, bk.dig.begin() + (i + 1) * Ld);
        eptr.push_back((int)eg.size());
        if (pol == Policy::depth_first && sts.size() >= wave) run_wave();
      }
    }
    run_wave();
  }
  std::vector<long long> hG(dG.n);
  DRZG_CUDA(cudaMemcpyAsync(hG.data(), dG.p, dG.n * sizeof(long long), cudaMemcpyDeviceToHost, st_));
  g_traffic.d2h += (long long)(dG.n * sizeof(long long));
  DRZG_CUDA(cudaEventRecord(run1, st_));
  DRZG_CUDA(cudaStreamSynchronize(st_));
  float ms = 0;
  DRZG_CUDA(cudaEventElapsedTime(&ms, run0, run1));
  clock.device_ms += ms;
  cudaEventDestroy(run0);
  cudaEventDestroy(run1);
  G.assign(ncol, {});
  for (int c = 0; c < ncol; ++c)
    G[c].assign(hG.begin() + (size_t)c * Ld * gsize_, hG.begin() + (size_t)(c + 1) * Ld * gsize_);
}


std::vector<i8> ReductionEngine::solve_units(const std::vector<int>& rows) {
  const RuvTables& T = *T_;
  const int Ld = T.dp.Ld, B = (int)rows.size();
  std::vector<i8> out((size_t)B * Ld * T.nL, 0);
  if (!B) return out;
  std::lock_guard<std::mutex> tmp_lock(tmp_mu_);
  ensure_batch(std::min(B, 1 << 14));
  std::vector<int8_t> hY;
  for (int b0 = 0; b0 < B; b0 += bcap_) {
    const int nb = std::min(bcap_, B - b0);
    // b = e_j: digit 0 is 1 at the system-order position of row j
    DRZG_CUDA(cudaMemsetAsync(Bg_.p, 0, Bg_.n, st_));
    std::vector<int> pos(nb);
    for (int s = 0; s < nb; ++s) {
      DRZG_REQUIRE(rows[b0 + s] >= 0 && rows[b0 + s] < T.nL, "solve_units: row out of range");
      pos[s] = pos_m_[rows[b0 + s]];
    }
    std::vector<int8_t> one(1, 1);
    for (int s = 0; s < nb; ++s)
      DRZG_CUDA(cudaMemcpyAsync(Bg_.p + (size_t)pos[s] * bcap_ + s, one.data(), 1, cudaMemcpyHostToDevice, st_));
    dev::StepArgs a = make_args(0, nb, 0);
    a.B = nb;
    chunk_steps_ = (double)nb;
    dixon(a);
    chunk_steps_ = 0;
    DRZG_CUDA(cudaGetLastError());
    hY.resize((size_t)Ld * nLp_ * bcap_);
    DRZG_CUDA(cudaMemcpyAsync(hY.data(), Y_.p, hY.size(), cudaMemcpyDeviceToHost, st_));
    DRZG_CUDA(cudaStreamSynchronize(st_));
    for (int s = 0; s < nb; ++s)
      for (int k = 0; k < Ld; ++k)
        for (int r = 0; r < T.nL; ++r)
          out[((size_t)(b0 + s) * Ld + k) * T.nL + r] = hY[((size_t)k * nLp_ + pos_r_[r]) * bcap_ + s];
  }
  return out;
}

}  // namespace drzg
