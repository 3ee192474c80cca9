// Device-resident reduction engine: state vectors live in an HBM slot pool,
// the host-side reduction policy (reference run_policy, reduction.hpp:464-533)
// chooses every move from (u, pole) alone, and each pole drop of a whole
// sweep runs as one batched Dixon step on the device.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "host/final.hpp"
#include "kernels/step_args.cuh"

namespace drzg {

#define DRZG_CUDA(x)                                                                          \
  do {                                                                                        \
    cudaError_t err_ = (x);                                                                   \
    if (err_ != cudaSuccess)                                                                  \
      throw ::drzg::contract_error(std::string("CUDA: ") + cudaGetErrorString(err_), __FILE__, \
                                   __LINE__);                                                 \
  } while (0)

// cudaMemGetInfo, timed: DRZG_VERBOSE reports calls slower than 5 ms (tail hunting)
inline void mem_info(size_t* fr, size_t* tot, const char* where) {
  const auto t0 = std::chrono::steady_clock::now();
  DRZG_CUDA(cudaMemGetInfo(fr, tot));
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  static const bool verbose = std::getenv("DRZG_VERBOSE") != nullptr;
  if (verbose && s > 0.005) std::fprintf(stderr, "[drzg] slow cudaMemGetInfo (%s): %.3f s\n", where, s);
}

// total memory of the current device (cached): small requests skip
// cudaMemGetInfo, which can take tens of milliseconds while the device is busy
inline size_t device_total_memory() {
  static size_t tot[64] = {0};
  int d = 0;
  cudaGetDevice(&d);
  if (d < 0 || d >= 64) return 0;
  if (!tot[d]) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d) == cudaSuccess) tot[d] = prop.totalGlobalMem;
  }
  return tot[d];
}

// host<->device traffic and kernel launches of the current call (reported
// with every result: the e2e byte counts and the launch count of the bench)
struct Traffic {
  std::atomic<long long> h2d{0}, d2h{0}, launches{0};
  void reset() { h2d = 0; d2h = 0; launches = 0; }
};
// per host thread: a call's launches and copies are issued on the calling thread,
// so concurrent calls (a batch on several threads) count their own
inline thread_local Traffic g_traffic;
// DRZG_TIMELINE diagnostics: host seconds spent in host-side allocation and
// staging waits (pinned growth, ring waits, stream-ordered allocations)
struct HostWaits {
  std::atomic<long long> pinned_ns{0}, ring_ns{0}, malloc_ns{0}, copy_ns{0};
  void reset() { pinned_ns = 0; ring_ns = 0; malloc_ns = 0; copy_ns = 0; }
};
inline HostWaits g_waits;
inline long long now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

enum class Policy { p_chunk = 0, depth_first = 1, var_by_var = 2 };

struct Ledger {
  i64 matvecs = 0, startups = 0, combines = 0;
};

// kernel-time accounting for the roofline report
struct KernelClock {
  bool on = false;
  double gemm_ms = 0, carry_ms = 0, gather_ms = 0, epi_ms = 0, other_ms = 0;
  double flush_ms = 0;  // of epi_ms: the chunk-end W -> slot transposes
  i64 gemm_launches = 0;
  double device_ms = 0;  // CUDA-event time of the whole device-resident run
  i64 peak_live = 0;     // most state slots live at once
  double gemm_macs = 0;  // digit GEMMs: int8 MACs issued (nL x nL per state-digit)
  i64 carry_launches = 0;
  double carry_macs = 0; // carry GEMMs (Jp . y_k)
};

// pinned staging ring: host-side inputs of a sweep are copied through
// page-locked buffers, so cudaMemcpyAsync really is asynchronous and the host
// policy runs ahead of the device (bounded by the ring: a buffer is reused
// only after the copy that read it has completed)
class Stager {
 public:
  ~Stager() {
    for (std::vector<Buf>* ring : {&small_, &large_})
      for (auto& b : *ring) {
        if (b.h && !b.carved) cudaFreeHost(b.h);
        if (b.ev) cudaEventDestroy(b.ev);
      }
    if (arena_) cudaFreeHost(arena_);
    for (void* h : retired_) cudaFreeHost(h);
  }
  // one pinned ring per size class and host thread (engines stage from the
  // thread that launches their kernels, so a ring only ever waits on its own
  // stream's copies; the mutex guards misuse).  Small requests use fixed
  // slots carved from one arena;
  // large ones a short ring whose slots grow to the high-water mark, so that
  // after the first sweeps no copy pins memory (cudaMallocHost costs up to
  // tens of ms, on the launcher's critical path)
  void copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    std::lock_guard<std::mutex> lk(mu_);
    const bool small = bytes <= kSmall;
    if (small && !arena_) {
      DRZG_CUDA(cudaMallocHost(&arena_, kSmall * small_.size()));
      for (size_t i = 0; i < small_.size(); ++i) {
        small_[i].h = static_cast<char*>(arena_) + i * kSmall;
        small_[i].cap = kSmall;
        small_[i].carved = true;
      }
    }
    std::vector<Buf>& ring = small ? small_ : large_;
    int& next = small ? next_small_ : next_large_;
    Buf& b = ring[next];
    next = (next + 1) % (int)ring.size();
    if (!b.ev) DRZG_CUDA(cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming));
    const long long t0 = now_ns();
    if (b.used) DRZG_CUDA(cudaEventSynchronize(b.ev));
    const long long t1 = now_ns();
    if (b.cap < bytes) {
      // the old buffer is retired, not freed: cudaFreeHost synchronises the
      // whole device, which would stall the launcher behind queued work
      if (b.h) retired_.push_back(b.h);
      hwm_ = std::max(hwm_, bytes);
      b.cap = std::max<size_t>({2 * bytes, 2 * hwm_, (size_t)2 << 20});
      DRZG_CUDA(cudaMallocHost(&b.h, b.cap));
    }
    const long long t2 = now_ns();
    std::memcpy(b.h, src, bytes);
    DRZG_CUDA(cudaMemcpyAsync(dst, b.h, bytes, cudaMemcpyHostToDevice, st));
    const long long t3 = now_ns();
    g_waits.ring_ns += t1 - t0;
    g_waits.pinned_ns += t2 - t1;
    g_waits.copy_ns += t3 - t2;
    DRZG_CUDA(cudaEventRecord(b.ev, st));
    b.used = true;
  }

 private:
  static constexpr size_t kSmall = 64 << 10;
  struct Buf {
    void* h = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool used = false;
    bool carved = false;  // part of the small-slot arena
  };
  std::vector<Buf> small_ = std::vector<Buf>(64);
  std::vector<Buf> large_ = std::vector<Buf>(8);
  int next_small_ = 0, next_large_ = 0;
  void* arena_ = nullptr;
  size_t hwm_ = 0;
  std::mutex mu_;
  std::vector<void*> retired_;
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  // stream-ordered buffers (the engine's) come from the device's retained
  // mempool and go back to it without synchronising the device; the stream
  // outlives the engine that owns the buffer
  ~DevBuf() { release(); }
  void alloc(size_t count, cudaStream_t st = nullptr) {
    if (count <= n) return;
    release();
    if (st) {
      const long long t0 = now_ns();
      DRZG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T), st));
      g_waits.malloc_ns += now_ns() - t0;
      async_ = true;
      ast_ = st;
    } else {
      DRZG_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    }
    n = count;
  }
  void release() {
    if (p) {
      if (async_)
        cudaFreeAsync(p, ast_);
      else
        cudaFree(p);
    }
    p = nullptr;
    n = 0;
    async_ = false;
  }
  void upload(const std::vector<T>& v, cudaStream_t st) {
    alloc(v.size(), st);
    if (!v.empty()) DRZG_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    g_traffic.h2d += (long long)(v.size() * sizeof(T));
  }
  // stream-ordered growth and a pinned-staged copy: never blocks the host on
  // earlier device work
  void stage(const std::vector<T>& v, Stager& sg, cudaStream_t st) {
    if (v.size() > n) alloc(std::max<size_t>(v.size() + v.size() / 2, 1024), st);
    sg.copy(p, v.data(), v.size() * sizeof(T), st);
    g_traffic.h2d += (long long)(v.size() * sizeof(T));
  }
  bool async_ = false;
  cudaStream_t ast_ = nullptr;
};

// state-pool memory a finished engine left mapped on `dev` for the next one
// (it counts as used in the driver's free figure, yet is available)
size_t cached_pool_bytes(int dev);

class ReductionEngine {
 public:
  ReductionEngine(const RuvTables& T, int n, u64 p, cudaStream_t st);
  ~ReductionEngine();

  // p-chunk policy over a group of columns; returns per column the floor
  // numerator as Ld digit-sum planes over Homog_{dn-n-1}
  void run_pchunk(std::vector<ColumnSeeds>& cols, std::vector<std::vector<i64>>& G, Ledger& led);

  // one chunk (k pole drops along v) for a batch of states supplied as
  // digit planes (reference reduce_chunk, reduction.hpp:394-423)
  void chunk_batch(const std::vector<Expo>& u, const std::vector<int>& vdir, const std::vector<i64>& k,
                   std::vector<i8>& w_digits, Ledger& led);

  // ---- state-level primitives: the C ABI's states API (drzg_states_*,
  // drzg_step_batch, drzg_run_policy) and the round-based policies ----
  struct Live {
    int col = 0;   // column (frobenius) or 0 (states API)
    Expo u;
    int pole = 0;
    int slot = -1;
  };
  // new states, one per entry list (CSR over (side row g, Ld balanced digits))
  std::vector<int> seed_states(const std::vector<int>& eptr, const std::vector<int>& eg, const std::vector<i8>& edig);
  // reduce_chunk (reduction.hpp:394-423) for every listed state at once: k
  // pole drops along its v (rank in Homog_d); u, pole updated
  void step_states(const std::vector<Live*>& sts, const std::vector<int>& vdir, const std::vector<i64>& k,
                   Ledger& led);
  // combine_states (reduction.hpp:426-451) over the listed states, keyed by
  // (col, u, pole): the first of each key keeps its slot and receives the
  // sum, the others are freed and dropped from the list
  void combine_live(std::vector<Live>& sts, Ledger& led);
  // run_policy (reduction.hpp:464-533) on device-resident states: every state
  // is driven to pole n with the policy's moves and combines; the floor states
  // are left in `sts`
  void run_policy_live(std::vector<Live>& sts, Policy pol, Ledger& led);
  // floor_to_numerator (reduction.hpp:566-581) of floor states into per-column
  // digit-sum accumulators (ncols x Ld x |Homog_{dn-n-1}|, int64)
  void floor_accumulate(const std::vector<Live>& sts, long long* dG, int ncols);
  // residues of states as Ld x side balanced digits (host)
  std::vector<i8> read_states(const std::vector<int>& slots);
  void write_state(int slot, const std::vector<i8>& digits);  // Ld x side
  void release_slots(const std::vector<int>& slots);
  // frobenius_matrix's per-column loop for the depth-first and var-by-var
  // policies (p-chunk has its own pipelined path, run_pchunk)
  void run_rounds(std::vector<ColumnSeeds>& cols, std::vector<std::vector<i64>>& G, Ledger& led, Policy pol);
  const std::vector<Expo>& dirs() const { return dirs_host_; }
  // y = Jp^{-1} e_j mod q^Ld for every listed Homog_L row j (the unit-echelon
  // solves RuvContext::solve_column hands build_ruv, reduction.hpp:200-215):
  // Ld balanced digits per solution index, [state][digit][r] (r in RuvTables order)
  std::vector<i8> solve_units(const std::vector<int>& rows);

  KernelClock clock;
  bool tensor_cores() const { return use_tc_; }
  int floor_size() const { return gsize_; }
  i64 peak_live() const { return peak_live_; }
  const RuvTables& tables() const { return *T_; }

 private:
  struct HS {
    int col;
    Expo u;
    int pole;
    int slot;
  };
  int alloc_slot();
  void free_slot(int s) { free_.push_back(s); }
  void grow_pool(int need);
  void ensure_batch(int B);
  // all chunk steps of the uploaded sweep (states sorted by k desc, then v):
  // per sub-batch, gather once from the pool, keep the state in W between
  // steps, flush to the pool where each chunk ends; returns matvecs
  i64 run_sweep(const std::vector<i64>& k_sorted);
  int chunk_max_states() const;
  dev::StepArgs make_args(int b0, int nb, int y);
  void dixon(dev::StepArgs& a);
  void timed(double* acc, const std::function<void()>& f);

  const RuvTables* T_;
  int n_;
  u64 p_;
  cudaStream_t st_;
  int nLp_ = 0, sidep_ = 0, gsize_ = 0;
  long long slot_stride_ = 0;
  // tables
  DevBuf<int8_t> C_;
  DevBuf<int8_t> Jd_;   // Jp dense (u8), nLp x nLp, for the tensor-core carry
  bool use_tc_ = false; // tcgen05 GEMMs (else the dp4a CUDA-core kernels)
  bool fast_ = false;   // fp32-reciprocal residues (host-checked operand bound)
  bool sparse_carry_ = false;  // carry GEMM over the nonzero K blocks of Jp only
  bool fused_ = false;         // whole solve in one launch (nLp <= 256; DRZG_FUSED=0 disables)
  bool chunk_ = false;         // ... every step of a chunk in that launch, T_x in-kernel (DRZG_CHUNK=0 disables)
  bool chunk_now_ = false;     // the current dixon() call is a whole-chunk launch
  double chunk_steps_ = 0;     // state-steps of the current dixon() call (accounting)
  bool flow_ = false;          // whole solve as one dataflow launch (larger systems; DRZG_FLOW=0 disables)
  bool flow2_ = false;         // ... on CTA pairs, M = 256 tiles (DRZG_FLOW2=0 keeps single-CTA tiles)
  DevBuf<int> kb2_ptr_, kb2_idx_;  // per 256-row tile: union of its 128-row tiles' nonzero K blocks
  long long kblocks2_ = 0;
  DevBuf<int> flow_ctr_;       // its per-column phase counters
  long long kblocks_ = 0;      // nonzero 128 x 128 blocks of Jp (system order)
  DevBuf<int> kb_ptr_, kb_idx_;
  DevBuf<int> ginv_;
  DevBuf<int> jp_ptr_, jp_col_, jp_val_, gidx_, dirs_, t_ptr_, t_src_, sol_i_, sol_mu_, mon_;
  DevBuf<unsigned long long> btab_;
  // pool
  int8_t* pool_ = nullptr;
  size_t vmm_reserved_ = 0, vmm_mapped_ = 0;
  int pool_dev_ = 0;
  struct VmmChunk {
    size_t off, bytes;
    unsigned long long handle;
  };
  std::vector<VmmChunk> vmm_chunks_;
  void release_pool();
  void trim_mempool(int dev);
  int cap_ = 0;
  i64 peak_live_ = 0;
  std::vector<int> free_;
  // sweep arrays
  DevBuf<int> d_slot_, d_vdir_, d_u0_;
  DevBuf<i64> d_k_;
  // temporaries.  The launcher thread owns them; the policy thread may give
  // them back (grow_pool, when the state pool needs their memory), so both
  // hold tmp_mu_ while they touch bcap_ or the buffers
  std::mutex tmp_mu_;
  int bcap_ = 0;
  int sms_ = 148;  // SM count of the engine device (set at construction)
  DevBuf<int8_t> Bg_, IN_, Y_;
  DevBuf<int8_t> H_;
  DevBuf<int8_t> W_;
  cudaEvent_t ev0_, ev1_;
  // pinned staging ring shared by every engine of the process: pinning and
  // unpinning host memory costs milliseconds per megabyte, so it is paid once
  // (never freed; the process exit releases it)
  // per host thread (concurrent calls never wait on each other's rings); the
  // engine shares ownership, so it may outlive the thread that built it
  static std::shared_ptr<Stager> thread_stager() {
    thread_local std::shared_ptr<Stager> s = std::make_shared<Stager>();
    return s;
  }
  std::shared_ptr<Stager> stager_owner_ = thread_stager();
  Stager& stager_ = *stager_owner_;
  double host_t_[5] = {0, 0, 0, 0, 0};  // host phases of run_pchunk (s)
  double prep_wait_s_ = 0;              // ... of which the policy waited for seed preparers
  double moves_only_s_ = 0;             // ... the move choices themselves (pchunk_move)
  double policy_wall_s_ = 0;            // the policy thread's whole run
  unsigned host_threads_ = call_cores();
  std::vector<Expo> dirs_host_;
  std::vector<int> pos_m_, pos_r_;  // system order of Homog_L rows / solution indices
};

}  // namespace drzg
