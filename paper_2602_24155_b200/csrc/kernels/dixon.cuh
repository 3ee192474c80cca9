// Device kernels of the controlled-reduction step (sm_100a).
//
// One pole drop of a batch of game states, each with its own move vector v
// and exponent x (reference reduce_chunk -> linrec_eval, one factor
// R_{x,v}; reduction.hpp:394-423, linalg.hpp:366-397), is computed as
//     w'  =  T_x ( Jp^{-1} P_v w )    mod p^M
// with all residues held as Ld balanced base-q int8 digit planes:
//   gather_kernel     b = P_v w                      (per-v index table)
//   dixon_gemm_kernel y_k = bal( Cq . in_k )         (int8 dot products)
//   dixon_carry_kernel c_{k+1} = (b_k + c_k - Jp y_k) / q,  in_{k+1}
//   epilogue_kernel   w'[g] = carry-normalise( sum (x_i + mu_i) y[r] )
// Setup/bookkeeping kernels: seed materialisation, state merge
// (combine_states, reduction.hpp:426-451) and floor accumulation
// (floor_to_numerator, reduction.hpp:566-581).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fastq.cuh"

namespace drzg {
namespace dev {

constexpr int kLdMaxK = 32;
static_assert(kLdMaxK == kLdMax, "digit plane bound");

__device__ __forceinline__ int balmod(int x, int q) {
  int r = x % q;
  if (r < 0) r += q;
  if (r > (q >> 1)) r -= q;
  return r;
}

struct StepArgs {
  // tables
  const int8_t* C;        // nLp x nLp (row-major), Jp^{-1} mod q
  const int* jp_ptr;      // nL + 1
  const int* jp_col;
  const int* jp_val;
  const int* gidx;        // ndir x nL
  const int* dirs;        // ndir x nv exponents of each v
  const int* t_ptr;       // side + 1
  const int* t_src;       // solution index feeding each side row
  const int* sol_i;       // per solution index: variable i of its generator
  const int* sol_mu;      // ... and mu_i
  int nv, nL, nLp, side, sidep, Ld, q;
  FastQ fq;
  // state pool
  int8_t* pool;           // slots x (Ld * sidep)
  long long slot_stride;  // Ld * sidep
  // batch
  const int* slot;        // B
  const int* vdir;        // B
  const int* u0;          // B x nv (exponent at sweep start)
  int y;                  // step index within the chunk: x = u0 - y v
  int B;
  // temporaries
  int8_t* Bg;             // B x Ld x nLp
  int8_t* IN;             // B x nLp
  int* Cy;                // B x nL
  int8_t* Y;              // B x Ld x nLp
};

__global__ void gather_kernel(StepArgs a) {
  const int nrb = (a.nL + blockDim.x - 1) / blockDim.x;  // flattened (state, row block)
  int s = blockIdx.x / nrb;
  int r = (blockIdx.x % nrb) * blockDim.x + threadIdx.x;
  if (r >= a.nL || s >= a.B) return;
  int g = a.gidx[(size_t)a.vdir[s] * a.nL + r];
  const int8_t* src = a.pool + (size_t)a.slot[s] * a.slot_stride;
  int8_t* dst = a.Bg + (size_t)s * a.Ld * a.nLp;
  for (int t = 0; t < a.Ld; ++t) dst[(size_t)t * a.nLp + r] = g >= 0 ? src[(size_t)t * a.sidep + g] : 0;
  a.IN[(size_t)s * a.nLp + r] = (int8_t)a.fq.bal(g >= 0 ? src[g] : 0);
  a.Cy[(size_t)s * a.nL + r] = 0;
}

// Y[s][k][r] = bal( sum_j C[r][j] * IN[s][j] ), 64x64 tile, K step 64 bytes,
// 256 threads each owning a 4x4 block, int8 dot products via dp4a
__global__ void __launch_bounds__(256) dixon_gemm_kernel(StepArgs a, int k) {
  __shared__ int Cs[64][17];
  __shared__ int Is[64][17];
  const int r0 = blockIdx.y * 64, s0 = blockIdx.x * 64;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  int acc[4][4] = {};
  const int words = a.nLp >> 2;
  for (int kw = 0; kw < words; kw += 16) {
    // load 64 rows x 16 words of each operand: 1024 words, 4 per thread
    for (int l = tid; l < 1024; l += 256) {
      int row = l >> 4, w = l & 15;
      Cs[row][w] = reinterpret_cast<const int*>(a.C + (size_t)(r0 + row) * a.nLp)[kw + w];
      int s = s0 + row;
      Is[row][w] = s < a.B ? reinterpret_cast<const int*>(a.IN + (size_t)s * a.nLp)[kw + w] : 0;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 16; ++w) {
      int ca[4], ib[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) ca[i] = Cs[ty * 4 + i][w];
#pragma unroll
      for (int j = 0; j < 4; ++j) ib[j] = Is[tx * 4 + j][w];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dp4a(ca[i], ib[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int s = s0 + tx * 4 + j;
    if (s >= a.B) continue;
    int8_t* yrow = a.Y + ((size_t)s * a.Ld + k) * a.nLp;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = r0 + ty * 4 + i;
      if (r < a.nL) yrow[r] = (int8_t)balmod(acc[i][j], a.q);
    }
  }
}

__global__ void dixon_carry_kernel(StepArgs a, int k) {
  const int nrb = (a.nL + blockDim.x - 1) / blockDim.x;  // flattened (state, row block)
  int s = blockIdx.x / nrb;
  int r = (blockIdx.x % nrb) * blockDim.x + threadIdx.x;
  if (r >= a.nL || s >= a.B) return;
  const int8_t* y = a.Y + ((size_t)s * a.Ld + k) * a.nLp;
  int sum = 0;
  for (int e = a.jp_ptr[r]; e < a.jp_ptr[r + 1]; ++e) sum += a.jp_val[e] * (int)y[a.jp_col[e]];
  const int8_t* bg = a.Bg + (size_t)s * a.Ld * a.nLp;
  int num = (int)bg[(size_t)k * a.nLp + r] + a.Cy[(size_t)s * a.nL + r] - sum;
  int c = num / a.q;  // exact
  a.Cy[(size_t)s * a.nL + r] = c;
  if (k + 1 < a.Ld) a.IN[(size_t)s * a.nLp + r] = (int8_t)balmod((int)bg[(size_t)(k + 1) * a.nLp + r] + c, a.q);
}

__global__ void epilogue_kernel(StepArgs a) {
  const int nrb = (a.side + blockDim.x - 1) / blockDim.x;
  int s = blockIdx.x / nrb;
  int g = (blockIdx.x % nrb) * blockDim.x + threadIdx.x;
  if (g >= a.side || s >= a.B) return;
  int x[6];
  const int* v = a.dirs + (size_t)a.vdir[s] * a.nv;
  for (int i = 0; i < a.nv; ++i) x[i] = a.u0[(size_t)s * a.nv + i] - a.y * v[i];
  int acc[kLdMax];
  for (int t = 0; t < a.Ld; ++t) acc[t] = 0;
  const int8_t* ys = a.Y + (size_t)s * a.Ld * a.nLp;
  for (int e = a.t_ptr[g]; e < a.t_ptr[g + 1]; ++e) {
    int r = a.t_src[e];
    int wgt = x[a.sol_i[r]] + a.sol_mu[r];
    for (int t = 0; t < a.Ld; ++t) acc[t] += wgt * (int)ys[(size_t)t * a.nLp + r];
  }
  int8_t* out = a.pool + (size_t)a.slot[s] * a.slot_stride;
  int carry = 0;
  for (int t = 0; t < a.Ld; ++t) {
    int r;
    int qt = a.fq.divfloor(acc[t] + carry, r);
    if (r > (a.q >> 1)) r -= a.q, ++qt;
    carry = qt;
    out[(size_t)t * a.sidep + g] = (int8_t)r;
  }
}

// one block per seed: zero its slot, then write the one-hot digits
__global__ void seed_kernel(int8_t* pool, long long slot_stride, int sidep, int Ld, const int* slot, const int* g,
                            const int8_t* dig, int nseeds) {
  int i = blockIdx.x;
  if (i >= nseeds) return;
  int8_t* w = pool + (size_t)slot[i] * slot_stride;
  int4* w4 = reinterpret_cast<int4*>(w);
  for (long long j = threadIdx.x; j < slot_stride / 16; j += blockDim.x) w4[j] = make_int4(0, 0, 0, 0);
  __syncthreads();
  if (threadIdx.x < Ld) w[(size_t)threadIdx.x * sidep + g[i]] = dig[(size_t)i * Ld + threadIdx.x];
}

// groups (CSR over member slots, first member receives the sum)
__global__ void merge_kernel(int8_t* pool, long long slot_stride, int side, int sidep, int Ld, int q,
                             const int* gptr, const int* members) {
  const int nrb = (side + blockDim.x - 1) / blockDim.x;
  int grp = blockIdx.x / nrb;
  int g = (blockIdx.x % nrb) * blockDim.x + threadIdx.x;
  if (g >= side) return;
  int acc[kLdMax];
  for (int t = 0; t < Ld; ++t) acc[t] = 0;
  for (int m = gptr[grp]; m < gptr[grp + 1]; ++m) {
    const int8_t* w = pool + (size_t)members[m] * slot_stride;
    for (int t = 0; t < Ld; ++t) acc[t] += w[(size_t)t * sidep + g];
  }
  int8_t* out = pool + (size_t)members[gptr[grp]] * slot_stride;
  int carry = 0;
  for (int t = 0; t < Ld; ++t) {
    int v2 = acc[t] + carry;
    int dgt = balmod(v2, q);
    carry = (v2 - dgt) / q;
    out[(size_t)t * sidep + g] = (int8_t)dgt;
  }
}

// floor: G[col][t][rank(mon_g + u - 1)] += w[t][g]; mon table is side x nv
__global__ void floor_kernel(const int8_t* pool, long long slot_stride, int side, int sidep, int Ld, int nv,
                             const int* slot, const int* col, const int* u, const int* mon, const unsigned long long* btab,
                             long long* G, int gsize, int* err) {
  const int nrb = (side + blockDim.x - 1) / blockDim.x;
  int s = blockIdx.x / nrb;
  int g = (blockIdx.x % nrb) * blockDim.x + threadIdx.x;
  if (g >= side) return;
  const int8_t* w = pool + (size_t)slot[s] * slot_stride;
  int e[6];
  int deg = 0;
  bool neg = false;
  for (int i = 0; i < nv; ++i) {
    e[i] = mon[(size_t)g * nv + i] + u[(size_t)s * nv + i] - 1;
    deg += e[i];
    neg |= e[i] < 0;
  }
  // reference: "floor_to_numerator: dishonest state" unless w[g] == 0 mod p^M;
  // honest states carry 0 there (digits may hold a multiple of p^M when
  // e*Ld > M), so the entry contributes nothing
  if (neg) return;
  (void)err;
  // grevlex rank (mono.hpp)
  long long rank = 0;
  int rem = deg;
  for (int j = nv - 1; j >= 1; --j) {
    auto C = [&](int aa, int bb) -> long long {
      if (aa < 0 || bb < 0 || bb > aa) return 0;
      return (long long)btab[(size_t)aa * 7 + bb];
    };
    rank += C(rem + j, j) - C(rem - e[j] + j, j);
    rem -= e[j];
  }
  long long* Gc = G + (size_t)col[s] * Ld * gsize;
  for (int t = 0; t < Ld; ++t) {
    int dv = w[(size_t)t * sidep + g];
    if (dv) atomicAdd(reinterpret_cast<unsigned long long*>(Gc + (size_t)t * gsize + rank), (unsigned long long)(long long)dv);
  }
}

}  // namespace dev
}  // namespace drzg
