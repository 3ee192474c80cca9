// Reference-shaped recurrence kernels (drop-in for linrec_eval and
// detail::sparse_steps, reference linalg.hpp:257-410).
//
// w <- M(0) M(1) ... M(tmax) w,  M(t) = t A + B, on the reference's own
// residue layout (limbs planes of base-beta u64 digits).  Three dense kernels:
// linrec_flat_kernel for sides whose matrices stream from HBM (a flat,
// balanced partition of the index space, a launch per factor),
// linrec_resident_kernel for smaller sides (all factors in one cooperative
// launch, the matrices in shared memory), linrec_dense_kernel (a warp per row)
// as the fallback.  Products are accumulated exactly in 192-bit per
// digit-plane sum (t1 + t2 < limbs; higher planes vanish because
// p^M | beta^limbs), then normalised to base-beta digits with preinverted
// divisions, the top digit reduced mod p^(M - e(limbs-1)), so the output is
// the canonical residue the reference produces.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
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

// two-word accumulator, for plans whose row sums stay below 2^128
// (limbs * side * (beta - 1)^2 < 2^127: both fourfold plans)
struct U128 {
  unsigned long long w0, w1;
};
__device__ __forceinline__ void add_prod(U128& acc, unsigned long long a, unsigned long long b) {
  unsigned long long lo = a * b, hi = __umul64hi(a, b);
  asm("add.cc.u64 %0, %0, %2;\n\t"
      "addc.u64 %1, %1, %3;"
      : "+l"(acc.w0), "+l"(acc.w1)
      : "l"(lo), "l"(hi));
}
__device__ __forceinline__ U192 widen(const U128& v) { return U192{v.w0, v.w1, 0}; }
__device__ __forceinline__ U192 widen(const U192& v) { return v; }

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

// Division by a per-call constant with a precomputed reciprocal (Moller and
// Granlund's 2-by-1 division, "Improved division by invariant integers",
// 2011): the divisor normalised to dn = d << s (top bit set) and
// v = floor((2^128 - 1) / dn) - 2^64, computed once on the host.  A 128-by-64
// step is two multiplies and two corrections instead of a software 128-bit
// division; the per-row digit normalisation is a serial chain of these.
struct Div64 {
  unsigned long long dn, v;
  int s;
};

inline Div64 make_div64(unsigned long long d) {
  Div64 D{};
  D.s = __builtin_clzll(d);
  D.dn = d << D.s;
  const unsigned __int128 all = ~(unsigned __int128)0;
  D.v = (unsigned long long)(all / D.dn - ((unsigned __int128)1 << 64));
  return D;
}

// (u1, u0) = q dn + r for u1 < dn; returns q, r through rr
__device__ __forceinline__ unsigned long long div2by1(unsigned long long u1, unsigned long long u0, const Div64& D,
                                                      unsigned long long& rr) {
  unsigned long long q0 = D.v * u1, q1 = __umul64hi(D.v, u1);
  q0 += u0;
  q1 += u1 + (q0 < u0 ? 1ull : 0ull);
  q1 += 1;
  unsigned long long r = u0 - q1 * D.dn;
  if (r > q0) {
    q1 -= 1;
    r += D.dn;
  }
  if (r >= D.dn) {
    q1 += 1;
    r -= D.dn;
  }
  rr = r;
  return q1;
}

// v / d and v % d for a 192-bit v (v <- quotient; the remainder returned)
__device__ __forceinline__ unsigned long long divmod192(U192& v, const Div64& D) {
  const int s = D.s;
  const unsigned long long n3 = s ? v.w2 >> (64 - s) : 0ull;
  const unsigned long long n2 = s ? (v.w2 << s) | (v.w1 >> (64 - s)) : v.w2;
  const unsigned long long n1 = s ? (v.w1 << s) | (v.w0 >> (64 - s)) : v.w1;
  const unsigned long long n0 = v.w0 << s;
  unsigned long long r = n3;
  v.w2 = div2by1(r, n2, D, r);
  v.w1 = div2by1(r, n1, D, r);
  v.w0 = div2by1(r, n0, D, r);
  return r >> s;
}

// x mod d for a 64-bit x
__device__ __forceinline__ unsigned long long mod64(unsigned long long x, const Div64& D) {
  const int s = D.s;
  unsigned long long r;
  div2by1(s ? x >> (64 - s) : 0ull, x << s, D, r);
  return r >> s;
}

// canonical base-beta digits of sum_s beta^s acc[s] mod p^M
__device__ __forceinline__ void normalise(U192* acc, int limbs, const Div64& beta, const Div64& top_mod,
                                          unsigned long long* out) {
  U192 carry{0, 0, 0};
  for (int s = 0; s < limbs; ++s) {
    U192 v = acc[s];
    add192(v, carry);
    out[s] = divmod192(v, beta);
    carry = v;
  }
  out[limbs - 1] = mod64(out[limbs - 1], top_mod);
}

struct LinrecArgs {
  const unsigned long long* A;  // limbs x side x side
  const unsigned long long* B;
  const unsigned long long* w;  // limbs x side (input of this factor)
  unsigned long long* y;        // limbs x side (output)
  int side, limbs;
  Div64 beta, top_mod;          // base and top-digit modulus, preinverted
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
__device__ __forceinline__ void normalise_t(U192 (&acc)[L], const Div64& beta, const Div64& top_mod,
                                            unsigned long long (&out)[L]) {
  U192 carry{0, 0, 0};
#pragma unroll
  for (int s = 0; s < L; ++s) {
    U192 v = acc[s];
    add192(v, carry);
    out[s] = divmod192(v, beta);
    carry = v;
  }
  out[L - 1] = mod64(out[L - 1], top_mod);
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

// One factor over a FLAT partition of the side x side index space: warp w of W
// streams the contiguous elements [E w / W, E (w+1) / W) of every plane of A
// and B (E = side^2), one resident wave, so every warp moves the same bytes
// and the reads are long sequential runs.  The vector is read through L1 (the
// same columns for every warp).  A warp's range crosses at most a few row
// boundaries; per row segment it shuffle-reduces its exact 192-bit partials,
// and a row split between warps is finished by the last of them to arrive
// (partials in `scratch`, an arrival counter per row, reset by the finisher).
struct LinrecFlat {
  U192* scratch;      // side x cmax x 2L partial sums
  unsigned* cnt;      // side arrival counters (zero between launches)
  int cmax;           // max warps sharing a row
  float keep;         // fraction of A and B loads marked L2 evict_last
};

// a load of the matrix stream under an L2 policy: the fraction f.keep of the
// lines (as many as the 126 MB L2 holds) stays resident across factors, the
// rest streams evict_first, so consecutive factors re-read the kept part from
// L2 rather than HBM
__device__ __forceinline__ unsigned long long ld_policy(const unsigned long long* p, unsigned long long pol) {
  unsigned long long v;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}

template <int L, int U, bool PF, bool N2 = false>
__global__ void __launch_bounds__(256, L == 1 ? 3 : 2) linrec_flat_kernel(LinrecArgs a, LinrecFlat f) {
  using Acc = typename std::conditional<N2, U128, U192>::type;
  const int lane = threadIdx.x & 31;
  const long long W = (long long)gridDim.x * (blockDim.x >> 5);
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long side = a.side, E = side * side;
  long long e = E * w / W;
  const long long e1 = E * (w + 1) / W;
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(pol) : "f"(f.keep));
  while (e < e1) {
    const long long r = e / side;
    const long long rend = min(e1, (r + 1) * side);
    const int c1 = (int)(rend - r * side);
    Acc pA[L], pB[L];
#pragma unroll
    for (int s = 0; s < L; ++s) pA[s] = pB[s] = Acc{};
    const unsigned long long* Ar = a.A + r * side;
    const unsigned long long* Br = a.B + r * side;
    // batches of 32 U columns, the last one predicated (zeros past the end):
    // every batch has all its loads in flight at once; with PF the next
    // batch's loads are issued before this batch's products
    unsigned long long av[L][U], bv[L][U], xv[L][U];
    auto load = [&](int j, unsigned long long (&ra)[L][U], unsigned long long (&rb)[L][U],
                    unsigned long long (&rx)[L][U]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool in = j + 32 * u < c1;
#pragma unroll
        for (int t = 0; t < L; ++t) {
          ra[t][u] = in ? ld_policy(Ar + t * E + j + 32 * u, pol) : 0ull;
          rb[t][u] = in ? ld_policy(Br + t * E + j + 32 * u, pol) : 0ull;
          rx[t][u] = in ? __ldg(a.w + t * side + j + 32 * u) : 0ull;
        }
      }
    };
    int j = (int)(e - r * side) + lane;
    if (PF) load(j, av, bv, xv);
    for (; j - lane < c1; j += 32 * U) {
      unsigned long long na[L][U], nb[L][U], nx[L][U];
      if (PF) {
        load(j + 32 * U, na, nb, nx);
      } else {
        load(j, av, bv, xv);
      }
#pragma unroll
      for (int t1 = 0; t1 < L; ++t1)
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int t2 = 0; t1 + t2 < L; ++t2) {
            add_prod(pA[t1 + t2], av[t1][u], xv[t2][u]);
            add_prod(pB[t1 + t2], bv[t1][u], xv[t2][u]);
          }
      if (PF) {
#pragma unroll
        for (int t = 0; t < L; ++t)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            av[t][u] = na[t][u];
            bv[t][u] = nb[t][u];
            xv[t][u] = nx[t][u];
          }
      }
    }
    U192 accA[L], accB[L];
#pragma unroll
    for (int s = 0; s < L; ++s) {
      accA[s] = widen(pA[s]);
      accB[s] = widen(pB[s]);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1)
#pragma unroll
      for (int s = 0; s < L; ++s) {
        add192(accA[s], shfl_down192(accA[s], off));
        add192(accB[s], shfl_down192(accB[s], off));
      }
    if (lane == 0) {
      // warps holding the row's first and last elements
      const long long wlo = ((r * side + 1) * W - 1) / E, whi = ((r + 1) * side * W - 1) / E;
      if (wlo == whi) {
        finish_row_t<L>(a, (int)r, accA, accB);
      } else {
        U192* base = f.scratch + (size_t)r * f.cmax * 2 * L;
        U192* mine = base + (size_t)(w - wlo) * 2 * L;
#pragma unroll
        for (int s = 0; s < L; ++s) {
          mine[s] = accA[s];
          mine[L + s] = accB[s];
        }
        __threadfence();
        const unsigned n = (unsigned)(whi - wlo + 1);
        if (atomicAdd(f.cnt + r, 1u) == n - 1) {
          __threadfence();
#pragma unroll
          for (int s = 0; s < L; ++s) accA[s] = accB[s] = U192{0, 0, 0};
          for (unsigned k = 0; k < n; ++k) {
            const unsigned long long* q = reinterpret_cast<const unsigned long long*>(base + (size_t)k * 2 * L);
#pragma unroll
            for (int s = 0; s < L; ++s) {
              add192(accA[s], U192{__ldcg(q + 3 * s), __ldcg(q + 3 * s + 1), __ldcg(q + 3 * s + 2)});
              add192(accB[s], U192{__ldcg(q + 3 * (L + s)), __ldcg(q + 3 * (L + s) + 1), __ldcg(q + 3 * (L + s) + 2)});
            }
          }
          finish_row_t<L>(a, (int)r, accA, accB);
          f.cnt[r] = 0;
        }
      }
    }
    e = rend;
  }
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


// Small sides, all factors in ONE cooperative launch with the matrices
// resident in shared memory: CTA c owns rows [c R, c R + R) (a warp per row)
// and loads its rows of A and B into shared memory once; each factor then
// reads only the vector (L side words, from L2) and synchronises the grid, so
// a factor costs a grid barrier instead of a launch plus an L2 pass over the
// matrices.  Same exact accumulation and normalisation as the other kernels.
template <int L>
__global__ void __launch_bounds__(256) linrec_resident_kernel(LinrecArgs a, unsigned long long* buf0,
                                                               unsigned long long* buf1, long long tmax, int R) {
  extern __shared__ unsigned long long sm[];  // [R][L][side] A, [R][L][side] B, [L][side] w
  cg::grid_group grid = cg::this_grid();
  const int side = a.side;
  const size_t nn = (size_t)side * side;
  const int r0 = blockIdx.x * R;
  const int rows = max(0, min(R, side - r0));
  unsigned long long* sA = sm;
  unsigned long long* sB = sm + (size_t)R * L * side;
  unsigned long long* sw = sB + (size_t)R * L * side;
  for (int k = threadIdx.x; k < rows * L * side; k += blockDim.x) {
    const int rr = k / (L * side), rem = k % (L * side), t = rem / side, j = rem % side;
    sA[k] = a.A[t * nn + (size_t)(r0 + rr) * side + j];
    sB[k] = a.B[t * nn + (size_t)(r0 + rr) * side + j];
  }
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  for (long long t = tmax; t >= 0; --t) {
    const unsigned long long* w = ((tmax - t) & 1) ? buf1 : buf0;
    unsigned long long* y = ((tmax - t) & 1) ? buf0 : buf1;
    for (int k = threadIdx.x; k < L * side; k += blockDim.x) sw[k] = __ldcg(w + k);
    __syncthreads();
    if (wi < rows) {
      U192 accA[L], accB[L];
#pragma unroll
      for (int s = 0; s < L; ++s) accA[s] = accB[s] = U192{0, 0, 0};
      const unsigned long long* ra = sA + (size_t)wi * L * side;
      const unsigned long long* rb = sB + (size_t)wi * L * side;
      for (int j = lane; j < side; j += 32) {
#pragma unroll
        for (int t1 = 0; t1 < L; ++t1) {
          const unsigned long long av = ra[t1 * side + j], bv = rb[t1 * side + j];
#pragma unroll
          for (int t2 = 0; t1 + t2 < L; ++t2) {
            const unsigned long long x = sw[t2 * side + j];
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
      if (lane == 0) {
        LinrecArgs b = a;
        b.y = y;
        b.t = (unsigned long long)t;
        finish_row_t<L>(b, r0 + wi, accA, accB);
      }
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
  a.beta = dev::make_div64(pl.beta);
  a.top_mod = dev::make_div64(pl.top_mod);
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
  // matrices resident in shared memory for sides whose rows spread over the
  // SMs fit (DRZG_LINREC_RESIDENT=0 disables)
  const bool resident_ok = [] {
    const char* e = std::getenv("DRZG_LINREC_RESIDENT");
    return !(e && std::string(e) == "0");
  }();
  if (!csr && resident_ok && (long long)side * side < (1LL << 20)) {
    const int L = pl.limbs;
    using KR = void (*)(dev::LinrecArgs, unsigned long long*, unsigned long long*, long long, int);
    KR kr = L == 1 ? dev::linrec_resident_kernel<1>
            : L == 2 ? dev::linrec_resident_kernel<2>
            : L == 3 ? dev::linrec_resident_kernel<3> : dev::linrec_resident_kernel<4>;
    int dev = 0, sms = 0, optin = 0;
    check(cudaGetDevice(&dev), "device");
    check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
    check(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "smem optin");
    const int R = std::min(8, (side + sms - 1) / sms);  // rows a CTA (a warp each)
    const int blocks = (side + R - 1) / R;
    const size_t rsmem = ((size_t)2 * R * L * side + (size_t)L * side) * 8;
    int per_sm = 0;
    if (rsmem <= (size_t)optin) {
      raise_smem_limit(kr, rsmem);
      check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kr, 32 * R, rsmem), "occupancy");
    }
    if (per_sm >= 1 && blocks <= sms * per_sm) {
      unsigned long long* b0 = (unsigned long long*)dw;
      unsigned long long* b1 = (unsigned long long*)tmp;
      long long tm = (long long)tmax;
      int rr = R;
      void* args[] = {&a, &b0, &b1, &tm, &rr};
      const cudaError_t le =
          cudaLaunchCooperativeKernel((const void*)kr, dim3(blocks), dim3(32 * R), args, rsmem, st);
      if (le == cudaErrorCooperativeLaunchTooLarge) {
        // the SMs are not all available to this context (MPS limits): the
        // per-factor kernels below do the same work
        (void)cudaGetLastError();
        goto per_factor;
      }
      check(le, "linrec resident launch");
      check(cudaGetLastError(), "linrec launch");
      // factor f (0-based) writes buf1 when f is even: tmax + 1 factors
      if (((tmax + 1) & 1) == 1) check(cudaMemcpyAsync(dw, tmp, vec * 8, cudaMemcpyDeviceToDevice, st), "copy back");
      if (kernel_ms) {
        check(cudaEventRecord(e1, st), "event");
        check(cudaEventSynchronize(e1), "event");
        check(cudaEventElapsedTime(kernel_ms, e0, e1), "event");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
      }
      check(cudaFreeAsync(tmp, st), "cudaFreeAsync");
      return;
    }
  }
per_factor:
  // DRZG_LINREC_FLAT: 0 = a warp per row, 1 = flat partition for large
  // sides (default), 2 = flat at every side, 3 = flat with the next batch's
  // loads in flight during the products (slower: 52 vs 44 us at side 3003)
  const int flat_mode = [] {
    const char* e = std::getenv("DRZG_LINREC_FLAT");
    return e ? std::atoi(e) : 1;
  }();
  // the flat partition wins once the matrices stream from HBM (side 3003:
  // 37 vs 47 us a factor, 1 limb); below that a warp per row finishes the
  // rows' serial digit normalisation in parallel (side 220: 6 vs 12 us)
  const bool flat = flat_mode == 2 || (flat_mode == 1 && (long long)side * side >= (1LL << 20));
  uint64_t* cur = dw;
  uint64_t* nxt = tmp;
  if (!csr && flat) {
    // one resident wave of warps over the flat index space, at least 512
    // elements a warp (the per-segment reduction amortised)
    const int L = pl.limbs;
    const bool pf = flat_mode == 3;
    using KF = void (*)(dev::LinrecArgs, dev::LinrecFlat);
    // row sums below 2^128: two-word accumulators (DRZG_LINREC_N2=0 keeps three)
    const bool n2 = [&] {
      const char* e = std::getenv("DRZG_LINREC_N2");
      if (e && std::string(e) == "0") return false;
      const unsigned __int128 sq = (unsigned __int128)(pl.beta - 1) * (pl.beta - 1);
      return sq < ((unsigned __int128)1 << 127) / ((unsigned __int128)L * (unsigned)side);
    }();
    KF kfn = L == 1 ? (pf ? dev::linrec_flat_kernel<1, 4, true>
                       : n2 ? dev::linrec_flat_kernel<1, 8, false, true> : dev::linrec_flat_kernel<1, 8, false>)
             : L == 2 ? (pf ? dev::linrec_flat_kernel<2, 2, true>
                         : n2 ? dev::linrec_flat_kernel<2, 4, false, true> : dev::linrec_flat_kernel<2, 4, false>)
             : L == 3 ? (pf ? dev::linrec_flat_kernel<3, 1, true> : dev::linrec_flat_kernel<3, 2, false>)
                      : (pf ? dev::linrec_flat_kernel<4, 1, true> : dev::linrec_flat_kernel<4, 2, false>);
    int dev = 0, sms = 0, per_sm = 0;
    check(cudaGetDevice(&dev), "device");
    check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
    check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kfn, 256, 0), "occupancy");
    DRZG_REQUIRE(per_sm >= 1, "linrec: flat kernel does not fit an SM");
    const long long E = (long long)side * side;
    const long long blocks = std::max(1LL, std::min((long long)sms * per_sm, E / (512LL * 8)));
    const long long W = blocks * 8;
    // most warps sharing one row: a warp holds at least floor(E / W) elements
    const long long per_warp = E / W;
    const int cmax = per_warp == 0 ? (int)W : (int)std::min<long long>(W, (side + per_warp - 1) / per_warp + 1);
    dev::LinrecFlat f{};
    const size_t scratch_bytes = (size_t)side * cmax * 2 * L * sizeof(dev::U192);
    check(cudaMallocAsync(&f.scratch, scratch_bytes, st), "cudaMallocAsync");
    check(cudaMallocAsync(&f.cnt, (size_t)side * sizeof(unsigned), st), "cudaMallocAsync");
    check(cudaMemsetAsync(f.cnt, 0, (size_t)side * sizeof(unsigned), st), "memset");
    f.cmax = cmax;
    {
      int l2 = 0;
      check(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev), "l2");
      const double mat = 2.0 * L * (double)E * 8;
      const double keep_scale = [] {
        const char* e = std::getenv("DRZG_LINREC_KEEP");
        return e ? std::atof(e) : 0.6;
      }();
      f.keep = (float)std::max(0.01, std::min(1.0, keep_scale * l2 / mat));
    }
    for (int64_t t = tmax; t >= 0; --t) {
      a.w = (const unsigned long long*)cur;
      a.y = (unsigned long long*)nxt;
      a.t = (unsigned long long)t;
      kfn<<<(unsigned)blocks, 256, 0, st>>>(a, f);
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
    check(cudaFreeAsync(f.scratch, st), "cudaFreeAsync");
    check(cudaFreeAsync(f.cnt, st), "cudaFreeAsync");
    check(cudaFreeAsync(tmp, st), "cudaFreeAsync");
    return;
  }
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
