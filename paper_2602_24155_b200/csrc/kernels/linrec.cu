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
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../host/common.hpp"
#include "linrec.cuh"

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

__global__ void linrec_dense_kernel(LinrecArgs a) {
  extern __shared__ unsigned long long ws[];  // limbs x side
  for (int k = threadIdx.x; k < a.limbs * a.side; k += blockDim.x) ws[k] = a.w[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= a.side) return;
  U192 accA[kMaxLimbs], accB[kMaxLimbs];
  for (int s = 0; s < kMaxLimbs; ++s) accA[s] = accB[s] = U192{0, 0, 0};
  const size_t nn = (size_t)a.side * a.side;
  if (a.limbs == 1) {
    const unsigned long long* ar = a.A + (size_t)i * a.side;
    const unsigned long long* br = a.B + (size_t)i * a.side;
    for (int j = lane; j < a.side; j += 32) {
      unsigned long long x = ws[j];
      add_prod(accA[0], __ldg(ar + j), x);
      add_prod(accB[0], __ldg(br + j), x);
    }
  } else {
    for (int j = lane; j < a.side; j += 32) {
      for (int t1 = 0; t1 < a.limbs; ++t1) {
        unsigned long long av = __ldg(a.A + t1 * nn + (size_t)i * a.side + j);
        unsigned long long bv = __ldg(a.B + t1 * nn + (size_t)i * a.side + j);
        for (int t2 = 0; t1 + t2 < a.limbs; ++t2) {
          unsigned long long x = ws[t2 * a.side + j];
          add_prod(accA[t1 + t2], av, x);
          add_prod(accB[t1 + t2], bv, x);
        }
      }
    }
  }
  for (int off = 16; off; off >>= 1)
    for (int s = 0; s < a.limbs; ++s) {
      add192(accA[s], shfl_down192(accA[s], off));
      add192(accB[s], shfl_down192(accB[s], off));
    }
  if (lane == 0) finish_row(a, i, accA, accB);
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

}  // namespace dev

namespace {
void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw contract_error(std::string(what) + ": " + cudaGetErrorString(e), __FILE__, __LINE__);
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
    check(cudaFuncSetAttribute(dev::linrec_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
          "smem attr");
    check(cudaFuncSetAttribute(dev::linrec_csr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
          "smem attr");
  }
  cudaEvent_t e0, e1;
  if (kernel_ms) {
    check(cudaEventCreate(&e0), "event");
    check(cudaEventCreate(&e1), "event");
    check(cudaEventRecord(e0, st), "event");
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
      dev::linrec_dense_kernel<<<grid, warps * 32, smem, st>>>(a);
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
