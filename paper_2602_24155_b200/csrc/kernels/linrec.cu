// Reference-shaped recurrence kernels (drop-in for linrec_eval and
// detail::sparse_steps, reference linalg.hpp:257-410).
//
// w <- M(0) M(1) ... M(tmax) w,  M(t) = t A + B, on the reference's own
// residue layout (limbs planes of base-beta u64 digits).  One launch per
// factor; a warp owns one output row and streams A and B once per factor
// (the HBM roofline for side >= ~700, 16 B per (i, j) per limb).  Products
// are accumulated exactly in 192-bit per digit-plane sum (t1 + t2 < limbs;
// higher planes vanish because p^M | beta^limbs), then normalised to base-beta
// digits, the top digit reduced mod p^(M - e(limbs-1)), so the output is the
// canonical residue the reference produces.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../host/common.hpp"
#include "linrec.cuh"

namespace cg = cooperative_groups;

namespace drzg {
namespace dev {

constexpr int kMaxLimbs = 4;

struct U192 {
  unsigned long long w0, w1, w2;
};

__device__ __forceinline__ void add_prod(U192& acc, unsigned long long a, unsigned long long b) {
  unsigned long long lo = a * b, hi = __umul64hi(a, b);
  asm("add.cc.u64 %0, %0, %3;\n\t"
      "addc.cc.u64 %1, %1, %4;\n\t"
      "addc.u64 %2, %2, 0;"
      : "+l"(acc.w0), "+l"(acc.w1), "+l"(acc.w2)
      : "l"(lo), "l"(hi));
}

__device__ __forceinline__ void add192(U192& a, const U192& b) {
  asm("add.cc.u64 %0, %0, %3;\n\t"
      "addc.cc.u64 %1, %1, %4;\n\t"
      "addc.u64 %2, %2, %5;"
      : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
      : "l"(b.w0), "l"(b.w1), "l"(b.w2));
}

__device__ __forceinline__ U192 shfl_down192(const U192& v, int off) {
  U192 r;
  r.w0 = __shfl_down_sync(0xffffffffu, v.w0, off);
  r.w1 = __shfl_down_sync(0xffffffffu, v.w1, off);
  r.w2 = __shfl_down_sync(0xffffffffu, v.w2, off);
  return r;
}

// v / beta and v % beta for a 192-bit v and 64-bit beta
__device__ __forceinline__ unsigned long long divmod192(U192& v, unsigned long long beta) {
  unsigned __int128 cur = v.w2;
  unsigned long long q2 = (unsigned long long)(cur / beta);
  cur = ((cur % beta) << 64) | v.w1;
  unsigned long long q1 = (unsigned long long)(cur / beta);
  cur = ((cur % beta) << 64) | v.w0;
  unsigned long long q0 = (unsigned long long)(cur / beta);
  unsigned long long r = (unsigned long long)(cur % beta);
  v.w2 = q2;
  v.w1 = q1;
  v.w0 = q0;
  return r;
}

// canonical base-beta digits of sum_s beta^s acc[s] mod p^M
__device__ __forceinline__ void normalise(U192* acc, int limbs, unsigned long long beta, unsigned long long top_mod,
                                          unsigned long long* out) {
  U192 carry{0, 0, 0};
  for (int s = 0; s < limbs; ++s) {
    U192 v = acc[s];
    add192(v, carry);
    out[s] = divmod192(v, beta);
    carry = v;
  }
  out[limbs - 1] %= top_mod;
}

struct LinrecArgs {
  const unsigned long long* A;  // limbs x side x side
  const unsigned long long* B;
  const unsigned long long* w;  // limbs x side (input of this factor)
  unsigned long long* y;        // limbs x side (output)
  int side, limbs;
  unsigned long long beta, top_mod;
  unsigned long long t;         // factor index
  // CSR variant
  const int* a_ptr;
  const int* a_col;
  const unsigned long long* a_val;  // nnz x limbs entry-major
  const int* b_ptr;
  const int* b_col;
  const unsigned long long* b_val;
};

template <int L>
__device__ __forceinline__ void normalise_t(U192 (&acc)[L], unsigned long long beta, unsigned long long top_mod,
                                            unsigned long long (&out)[L]) {
  U192 carry{0, 0, 0};
#pragma unroll
  for (int s = 0; s < L; ++s) {
    U192 v = acc[s];
    add192(v, carry);
    out[s] = divmod192(v, beta);
    carry = v;
  }
  out[L - 1] %= top_mod;
}
template <int L>
__device__ __forceinline__ void finish_row_t(const LinrecArgs& a, int i, U192 (&accA)[L], U192 (&accB)[L]) {
  unsigned long long da[L], db[L];
  normalise_t<L>(accA, a.beta, a.top_mod, da);
  normalise_t<L>(accB, a.beta, a.top_mod, db);
  U192 comb[L];
#pragma unroll
  for (int s = 0; s < L; ++s) {
    comb[s] = U192{db[s], 0, 0};
    add_prod(comb[s], a.t, da[s]);
  }
  unsigned long long out[L];
  normalise_t<L>(comb, a.beta, a.top_mod, out);
#pragma unroll
  for (int s = 0; s < L; ++s) a.y[(size_t)s * a.side + i] = out[s];
}

__device__ __forceinline__ void finish_row(const LinrecArgs& a, int i, U192* accA, U192* accB) {
  unsigned long long da[kMaxLimbs], db[kMaxLimbs];
  normalise(accA, a.limbs, a.beta, a.top_mod, da);
  normalise(accB, a.limbs, a.beta, a.top_mod, db);
  U192 comb[kMaxLimbs];
  for (int s = 0; s < a.limbs; ++s) {
    comb[s] = U192{db[s], 0, 0};
    add_prod(comb[s], a.t, da[s]);
  }
  unsigned long long out[kMaxLimbs];
  normalise(comb, a.limbs, a.beta, a.top_mod, out);
  for (int s = 0; s < a.limbs; ++s) a.y[(size_t)s * a.side + i] = out[s];
}


// One factor: a warp owns one output row, A and B stream once (the HBM bound
// for large sides).  L (the limb count) is a template parameter so the 192-bit
// accumulators and the staged loads live in registers; planes t1 + t2 < L only
// (higher planes vanish mod p^M).  Per iteration each lane has U columns of
// every plane of A and B in flight before any product: a row is otherwise a
// latency-bound stream of one 256-byte warp load per matrix.
template <int L>
__global__ void __launch_bounds__(256) linrec_dense_kernel(LinrecArgs a) {
  constexpr int U = L == 1 ? 4 : 2;
  extern __shared__ unsigned long long ws[];  // L x side
  for (int k = threadIdx.x; k < L * a.side; k += blockDim.x) ws[k] = a.w[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= a.side) return;
  U192 accA[L], accB[L];
#pragma unroll
  for (int s = 0; s < L; ++s) accA[s] = accB[s] = U192{0, 0, 0};
  const size_t nn = (size_t)a.side * a.side;
  const unsigned long long* Ar = a.A + (size_t)i * a.side;
  const unsigned long long* Br = a.B + (size_t)i * a.side;
  int j = lane;
  for (; j + 32 * (U - 1) < a.side; j += 32 * U) {
    unsigned long long av[L][U], bv[L][U];
#pragma unroll
    for (int t1 = 0; t1 < L; ++t1)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        av[t1][u] = __ldg(Ar + t1 * nn + j + 32 * u);
        bv[t1][u] = __ldg(Br + t1 * nn + j + 32 * u);
      }
#pragma unroll
    for (int t1 = 0; t1 < L; ++t1)
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t2 = 0; t1 + t2 < L; ++t2) {
          const unsigned long long x = ws[t2 * a.side + j + 32 * u];
          add_prod(accA[t1 + t2], av[t1][u], x);
          add_prod(accB[t1 + t2], bv[t1][u], x);
        }
  }
  for (; j < a.side; j += 32) {
#pragma unroll
    for (int t1 = 0; t1 < L; ++t1) {
      const unsigned long long av = __ldg(Ar + t1 * nn + j), bv = __ldg(Br + t1 * nn + j);
#pragma unroll
      for (int t2 = 0; t1 + t2 < L; ++t2) {
        const unsigned long long x = ws[t2 * a.side + j];
        add_prod(accA[t1 + t2], av, x);
        add_prod(accB[t1 + t2], bv, x);
      }
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1)
#pragma unroll
    for (int s = 0; s < L; ++s) {
      add192(accA[s], shfl_down192(accA[s], off));
      add192(accB[s], shfl_down192(accB[s], off));
    }
  if (lane == 0) finish_row_t<L>(a, i, accA, accB);
}

__global__ void linrec_csr_kernel(LinrecArgs a) {
  extern __shared__ unsigned long long ws[];
  for (int k = threadIdx.x; k < a.limbs * a.side; k += blockDim.x) ws[k] = a.w[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= a.side) return;
  U192 accA[kMaxLimbs], accB[kMaxLimbs];
  for (int s = 0; s < kMaxLimbs; ++s) accA[s] = accB[s] = U192{0, 0, 0};
  for (int e = a.a_ptr[i] + lane; e < a.a_ptr[i + 1]; e += 32) {
    int j = a.a_col[e];
    for (int t1 = 0; t1 < a.limbs; ++t1)
      for (int t2 = 0; t1 + t2 < a.limbs; ++t2) add_prod(accA[t1 + t2], a.a_val[(size_t)e * a.limbs + t1], ws[t2 * a.side + j]);
  }
  for (int e = a.b_ptr[i] + lane; e < a.b_ptr[i + 1]; e += 32) {
    int j = a.b_col[e];
    for (int t1 = 0; t1 < a.limbs; ++t1)
      for (int t2 = 0; t1 + t2 < a.limbs; ++t2) add_prod(accB[t1 + t2], a.b_val[(size_t)e * a.limbs + t1], ws[t2 * a.side + j]);
  }
  for (int off = 16; off; off >>= 1)
    for (int s = 0; s < a.limbs; ++s) {
      add192(accA[s], shfl_down192(accA[s], off));
      add192(accB[s], shfl_down192(accB[s], off));
    }
  if (lane == 0) finish_row(a, i, accA, accB);
}


// All factors of a dense linrec_eval in ONE cooperative launch: every warp owns
// rows i = warp_global, + total warps, ...; the grid synchronises between
// factors (each factor needs the whole previous vector).  A and B stream with
// 128-bit loads (two columns per lane per load, two loads in flight per matrix
// and limb), the vector sits in shared memory, reloaded after every grid sync.
// Same exact 192-bit accumulation and canonical normalisation as
// linrec_dense_kernel, so the output is bit-identical.
__global__ void __launch_bounds__(256) linrec_dense_persistent(LinrecArgs a, unsigned long long* buf0,
                                                                 unsigned long long* buf1, long long tmax) {
  extern __shared__ unsigned long long ws[];  // limbs x side
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + (threadIdx.x >> 5), nw = gridDim.x * wpb;
  const size_t nn = (size_t)a.side * a.side;
  const int side = a.side, L = a.limbs;
  const bool even = (side & 1) == 0;
  for (long long t = tmax; t >= 0; --t) {
    const unsigned long long* w = ((tmax - t) & 1) ? buf1 : buf0;
    unsigned long long* y = ((tmax - t) & 1) ? buf0 : buf1;
    for (int k = threadIdx.x; k < L * side; k += blockDim.x) ws[k] = w[k];
    __syncthreads();
    LinrecArgs b = a;
    b.y = y;
    b.t = (unsigned long long)t;
    for (int i = gw; i < side; i += nw) {
      U192 accA[kMaxLimbs], accB[kMaxLimbs];
      for (int s2 = 0; s2 < kMaxLimbs; ++s2) accA[s2] = accB[s2] = U192{0, 0, 0};
      for (int t1 = 0; t1 < L; ++t1) {
        const unsigned long long* ar = a.A + t1 * nn + (size_t)i * side;
        const unsigned long long* br = a.B + t1 * nn + (size_t)i * side;
        // rows start 16-byte aligned when side is even: two columns per load
        if (even) {
          for (int j = 2 * lane; j < side; j += 64) {
            const ulonglong2 av = __ldg(reinterpret_cast<const ulonglong2*>(ar + j));
            const ulonglong2 bv = __ldg(reinterpret_cast<const ulonglong2*>(br + j));
            for (int t2 = 0; t1 + t2 < L; ++t2) {
              const unsigned long long x0 = ws[t2 * side + j], x1 = ws[t2 * side + j + 1];
              add_prod(accA[t1 + t2], av.x, x0);
              add_prod(accA[t1 + t2], av.y, x1);
              add_prod(accB[t1 + t2], bv.x, x0);
              add_prod(accB[t1 + t2], bv.y, x1);
            }
          }
        } else {
          for (int j = lane; j < side; j += 32) {
            const unsigned long long av = __ldg(ar + j), bv = __ldg(br + j);
            for (int t2 = 0; t1 + t2 < L; ++t2) {
              const unsigned long long x = ws[t2 * side + j];
              add_prod(accA[t1 + t2], av, x);
              add_prod(accB[t1 + t2], bv, x);
            }
          }
        }
      }
      for (int off = 16; off; off >>= 1)
        for (int s2 = 0; s2 < L; ++s2) {
          add192(accA[s2], shfl_down192(accA[s2], off));
          add192(accB[s2], shfl_down192(accB[s2], off));
        }
      if (lane == 0) finish_row(b, i, accA, accB);
    }
    __threadfence();
    grid.sync();
  }
}

}  // namespace dev

namespace {
void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw contract_error(std::string(what) + ": " + cudaGetErrorString(e), __FILE__, __LINE__);
}
// the dynamic shared-memory opt-in of a kernel on the current device only
// ever rises: it is process-wide, and a concurrent call with a smaller system
// must not lower it under another thread's launch
template <class K>
void raise_smem_limit(K* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> have;
  int dev = 0;
  check(cudaGetDevice(&dev), "device");
  std::lock_guard<std::mutex> lk(mu);
  size_t& h = have[{reinterpret_cast<const void*>(kernel), dev}];
  if (h >= bytes) return;
  check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), "smem attr");
  h = bytes;
}
}  // namespace

void linrec_device(const LinrecPlan& pl, int side, const uint64_t* dA, const uint64_t* dB, int64_t tmax,
                   uint64_t* dw, cudaStream_t st, float* kernel_ms, const CsrPair* csr) {
  DRZG_REQUIRE(pl.limbs >= 1 && pl.limbs <= dev::kMaxLimbs, "linrec: unsupported limb count");
  DRZG_REQUIRE(tmax >= 0, "linrec_eval: negative range");
  size_t vec = (size_t)pl.limbs * side;
  DRZG_REQUIRE(vec * 8 <= 200 * 1024, "linrec: vector exceeds shared memory");
  uint64_t* tmp = nullptr;
  check(cudaMallocAsync(&tmp, vec * 8, st), "cudaMallocAsync");
  dev::LinrecArgs a{};
  a.A = (const unsigned long long*)dA;
  a.B = (const unsigned long long*)dB;
  a.side = side;
  a.limbs = pl.limbs;
  a.beta = pl.beta;
  a.top_mod = pl.top_mod;
  if (csr) {
    a.a_ptr = csr->a_ptr;
    a.a_col = csr->a_col;
    a.a_val = (const unsigned long long*)csr->a_val;
    a.b_ptr = csr->b_ptr;
    a.b_col = csr->b_col;
    a.b_val = (const unsigned long long*)csr->b_val;
  }
  const int warps = 8;
  dim3 grid((side + warps - 1) / warps);
  size_t smem = vec * 8;
  if (smem > 48 * 1024) {
    raise_smem_limit(dev::linrec_dense_kernel<1>, smem);
    raise_smem_limit(dev::linrec_dense_kernel<2>, smem);
    raise_smem_limit(dev::linrec_dense_kernel<3>, smem);
    raise_smem_limit(dev::linrec_dense_kernel<4>, smem);
    raise_smem_limit(dev::linrec_csr_kernel, smem);
  }
  cudaEvent_t e0, e1;
  if (kernel_ms) {
    check(cudaEventCreate(&e0), "event");
    check(cudaEventCreate(&e1), "event");
    check(cudaEventRecord(e0, st), "event");
  }
  static const bool persistent = [] {
    // opt-in: one cooperative launch for all factors measured slower than a
    // launch per factor (side 3003: 115 vs 60 us per factor; side 220-495 equal)
    const char* e = std::getenv("DRZG_LINREC_PERSISTENT");
    return e && std::string(e) == "1";
  }();
  if (!csr && persistent) {
    // one cooperative launch for every factor (grid-wide sync between factors)
    int dev = 0, sms = 0, per_sm = 0;
    check(cudaGetDevice(&dev), "device");
    check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
    raise_smem_limit(dev::linrec_dense_persistent, smem);
    check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::linrec_dense_persistent, 256, smem), "occupancy");
    DRZG_REQUIRE(per_sm >= 1, "linrec: persistent kernel does not fit an SM");
    const int rows_per_block = 8;
    const int blocks = std::max(1, std::min(sms * per_sm, (side + rows_per_block - 1) / rows_per_block));
    unsigned long long* b0 = (unsigned long long*)dw;
    unsigned long long* b1 = (unsigned long long*)tmp;
    long long tm = (long long)tmax;
    void* args[] = {&a, &b0, &b1, &tm};
    check(cudaLaunchCooperativeKernel((const void*)dev::linrec_dense_persistent, dim3(blocks), dim3(256), args, smem, st),
          "linrec cooperative launch");
    // the result is in buf0 after an odd number of factors... (tmax + 1 factors:
    // factor f (0-based) writes buf1 when f is even)
    if (((tmax + 1) & 1) == 1) check(cudaMemcpyAsync(dw, tmp, vec * 8, cudaMemcpyDeviceToDevice, st), "copy back");
    if (kernel_ms) {
      check(cudaEventRecord(e1, st), "event");
      check(cudaEventSynchronize(e1), "event");
      check(cudaEventElapsedTime(kernel_ms, e0, e1), "event");
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    check(cudaGetLastError(), "linrec launch");
    check(cudaFreeAsync(tmp, st), "cudaFreeAsync");
    return;
  }
  uint64_t* cur = dw;
  uint64_t* nxt = tmp;
  for (int64_t t = tmax; t >= 0; --t) {
    a.w = (const unsigned long long*)cur;
    a.y = (unsigned long long*)nxt;
    a.t = (unsigned long long)t;
    if (csr)
      dev::linrec_csr_kernel<<<grid, warps * 32, smem, st>>>(a);
    else
      switch (pl.limbs) {
        case 1: dev::linrec_dense_kernel<1><<<grid, warps * 32, smem, st>>>(a); break;
        case 2: dev::linrec_dense_kernel<2><<<grid, warps * 32, smem, st>>>(a); break;
        case 3: dev::linrec_dense_kernel<3><<<grid, warps * 32, smem, st>>>(a); break;
        default: dev::linrec_dense_kernel<4><<<grid, warps * 32, smem, st>>>(a); break;
      }
    std::swap(cur, nxt);
  }
  check(cudaGetLastError(), "linrec launch");
  if (kernel_ms) {
    check(cudaEventRecord(e1, st), "event");
    check(cudaEventSynchronize(e1), "event");
    check(cudaEventElapsedTime(kernel_ms, e0, e1), "event");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (cur != dw) check(cudaMemcpyAsync(dw, cur, vec * 8, cudaMemcpyDeviceToDevice, st), "copy back");
  check(cudaFreeAsync(tmp, st), "cudaFreeAsync");
}

}  // namespace drzg
