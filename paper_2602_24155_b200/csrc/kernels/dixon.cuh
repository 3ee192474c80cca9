// Device kernels of the controlled-reduction step (sm_100a).
//
// One pole drop of a batch of game states, each with its own move vector v
// and exponent x (reference reduce_chunk -> linrec_eval, one factor
// R_{x,v}; reduction.hpp:394-423, linalg.hpp:366-397), is computed as
//     w'  =  T_x ( Jp^{-1} P_v w )    mod p^M
// with all residues held as Ld balanced base-q int8 digit planes:
//   gather_kernel     b = P_v w                      (per-v index table)
//   dixon_gemm_kernel y_k = bal( Cq . in_k )         (int8 dot products)
//   dixon_carry_kernel c = (r_k - Jp y_k) / q, r_{k+1} = b_{k+1} + c = in_{k+1} + q h_{k+1}
//   epilogue_kernel   w'[g] = carry-normalise( sum (x_i + mu_i) y[r] )
// Setup/bookkeeping kernels: seed materialisation, state merge
// (combine_states, reduction.hpp:426-451) and floor accumulation
// (floor_to_numerator, reduction.hpp:566-581).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>

#include "fastq.cuh"
#include "step_args.cuh"

namespace drzg {
namespace dev {

__device__ __forceinline__ int balmod(int x, int q) {
  int r = x % q;
  if (r < 0) r += q;
  if (r > (q >> 1)) r -= q;
  return r;
}

#ifndef DRZG_EPILOGUE_ONLY
// b = P_v w at the first step of a chunk, from the slot pool into the
// state-contiguous operand Bg.  A block owns 32 states: for each digit plane
// it stages the 32 states' plane (32 x sidep bytes, coalesced 16-byte loads
// of each slot) in shared memory, then every thread assembles rows r: 32
// bytes b[t][r][s0..s0+31] = w_s[t][gidx[v_s][r]] as two 16-byte stores.
// (Digit 0 of a pool state is balanced, so b_0 is the first digit GEMM's
// operand as it stands and the first carry's residual r_0.)
constexpr int kGatherStates = 32, kGatherThreads = 512;
// shared memory holds the block's plane transposed, [g][32 states], rows
// padded to 36 bytes so the transposing stores and the row reads are free of
// bank conflicts
constexpr int kGatherPitch = 36;
inline size_t gather_smem_bytes(int sidep) { return (size_t)sidep * kGatherPitch; }
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(StepArgs a) {
  extern __shared__ __align__(16) int8_t planes[];  // sidep x kGatherPitch: [g][state]
  __shared__ int vd[kGatherStates];
  __shared__ long long base[kGatherStates];
  __shared__ int uniform_v;
  const int s0 = blockIdx.x * kGatherStates, tid = threadIdx.x;
  const int sidep = a.sidep, nL = a.nL;
  if (tid < kGatherStates) {
    const int s = s0 + tid;
    vd[tid] = s < a.B ? a.vdir[s] : -1;
    base[tid] = s < a.B ? (long long)a.slot[s] * a.slot_stride : -1;
  }
  __syncthreads();
  if (tid == 0) {
    int u = vd[0];
    for (int i = 1; i < kGatherStates; ++i)
      if (vd[i] != u && vd[i] >= 0) u = -2;
    uniform_v = u;
  }
  const size_t P = (size_t)a.P, plane = (size_t)a.nLp * P;
  const int words = sidep / 4;          // 4-row groups g4 of a slot plane
  const int groups = (words + 7) / 8;   // 8 g4 x 4 state quads per warp-wide work unit
  for (int t = 0; t < a.Ld; ++t) {
    __syncthreads();  // the previous plane is consumed (and uniform_v is set)
    // transposing load: a lane takes rows 4 g4 .. 4 g4 + 3 of four states
    // (one quad), 4 x 4 bytes, and stores them as four words of [g][state];
    // a warp reads 32 contiguous bytes of each of its 4 quads' 16 states
    // (kGU work items per thread per pass: their 4 kGU loads are all in
    // flight before any is used -- the phase is latency-bound otherwise)
    constexpr int kGU = 4;
    const int nitems = groups * 32 * 2;
    for (int e0 = tid; e0 < nitems; e0 += kGatherThreads * kGU) {
      uint32_t w[kGU][4];
      int g4s[kGU], qs[kGU];
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        const int e = e0 + u * kGatherThreads;
        const int qh = e / (groups * 32), rest = e - qh * groups * 32;
        const int gq = rest >> 5, lane = rest & 31;
        g4s[u] = e < nitems ? gq * 8 + (lane >> 2) : words;
        qs[u] = (lane & 3) + 4 * qh;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const long long bs = g4s[u] < words ? base[qs[u] * 4 + k] : -1;
          w[u][k] = bs >= 0 ? __ldg(reinterpret_cast<const uint32_t*>(a.pool + bs + (size_t)t * sidep) + g4s[u]) : 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < kGU; ++u) {
        if (g4s[u] >= words) continue;
        const uint32_t lo01 = __byte_perm(w[u][0], w[u][1], 0x5140), hi01 = __byte_perm(w[u][0], w[u][1], 0x7362);
        const uint32_t lo23 = __byte_perm(w[u][2], w[u][3], 0x5140), hi23 = __byte_perm(w[u][2], w[u][3], 0x7362);
        int8_t* dst = planes + (size_t)(4 * g4s[u]) * kGatherPitch + 4 * qs[u];
        *reinterpret_cast<uint32_t*>(dst) = __byte_perm(lo01, lo23, 0x5410);
        *reinterpret_cast<uint32_t*>(dst + kGatherPitch) = __byte_perm(lo01, lo23, 0x7632);
        *reinterpret_cast<uint32_t*>(dst + 2 * kGatherPitch) = __byte_perm(hi01, hi23, 0x5410);
        *reinterpret_cast<uint32_t*>(dst + 3 * kGatherPitch) = __byte_perm(hi01, hi23, 0x7632);
      }
    }
    __syncthreads();
    const int uv = uniform_v;
    for (int r = tid; r < nL; r += kGatherThreads) {
      uint32_t wd[8];
      if (uv >= 0) {
        // one state direction: the row's 32 bytes are one padded row of the
        // transposed plane
        const int g = __ldg(a.gidx + (size_t)uv * nL + r);
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8)
          wd[q8] = g >= 0 ? *reinterpret_cast<const uint32_t*>(planes + (size_t)g * kGatherPitch + 4 * q8) : 0u;
      } else {
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8) {
          uint32_t word = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int i = q8 * 4 + b;
            const int g = vd[i] >= 0 ? __ldg(a.gidx + (size_t)vd[i] * nL + r) : -1;
            word |= (uint32_t)(uint8_t)(g >= 0 ? planes[(size_t)g * kGatherPitch + i] : 0) << (8 * b);
          }
          wd[q8] = word;
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(a.Bg + (size_t)t * plane + (size_t)r * P + s0);
      dst[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
      dst[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
    }
  }
}

// CUDA-core fallback (DRZG_GEMM=dp4a, or Jp entries >= 256):
// Y[k][r][s] = bal( sum_j C[r][j] * IN[j][s] ), 64 x 64 tiles
__global__ void __launch_bounds__(256) dixon_gemm_kernel(StepArgs a, int k) {
  __shared__ int8_t Cs[64][68];
  __shared__ int8_t Is[64][68];  // [j][s]
  const int r0 = blockIdx.y * 64, s0 = blockIdx.x * 64;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  int acc[4][4] = {};
  for (int j0 = 0; j0 < a.nLp; j0 += 64) {
    for (int l = tid; l < 64 * 64; l += 256) {
      int rr = l >> 6, cc = l & 63;
      Cs[rr][cc] = a.C[(size_t)(r0 + rr) * a.nLp + j0 + cc];
      // digit 0 reads b_0 itself (balanced digits, c_0 = 0)
      const int8_t* src = k ? a.IN : a.Bg;
      Is[rr][cc] = s0 + cc < a.P ? src[(size_t)(j0 + rr) * a.P + s0 + cc] : (int8_t)0;
    }
    __syncthreads();
    for (int j = 0; j < 64; ++j) {
      int cv[4], iv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) cv[i] = Cs[ty * 4 + i][j];
#pragma unroll
      for (int i = 0; i < 4; ++i) iv[i] = Is[j][tx * 4 + i];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] += cv[i] * iv[jj];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = r0 + ty * 4 + i;
    if (r >= a.nL) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      int s = s0 + tx * 4 + jj;
      if (s < a.B) a.Y[((size_t)k * a.nLp + r) * a.P + s] = (int8_t)a.fq.bal(acc[i][jj]);
    }
  }
}

// c = (r_k - Jp y_k) / q with r_0 = b_0, r_k = in_k + q h_k; in_{k+1}, h_{k+1}
__global__ void dixon_carry_kernel(StepArgs a, int k) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (s >= a.B || r >= a.nL) return;
  const int8_t* y = a.Y + (size_t)k * a.nLp * a.P;
  int sum = 0;
  for (int e = a.jp_ptr[r]; e < a.jp_ptr[r + 1]; ++e) sum += a.jp_val[e] * (int)y[(size_t)a.jp_col[e] * a.P + s];
  size_t off = (size_t)r * a.P + s;
  const int rk = k ? (int)a.IN[off] + a.q * (int)a.H[off] : (int)a.Bg[off];
  int rem;
  const int c = a.fq.divfloor(rk - sum, rem);  // exact
  int hq = a.fq.divfloor((int)a.Bg[(size_t)(k + 1) * a.nLp * a.P + off] + c, rem);
  if (rem > (a.q >> 1)) rem -= a.q, ++hq;
  a.IN[off] = (int8_t)rem;
  a.H[off] = (int8_t)hq;
}

#endif  // DRZG_EPILOGUE_ONLY

// w' = T_x y into W (Ld x sidep x P) or the next step's gathered operand Bg,
// carry-normalised digits.  A block owns 128 states (each lane 4 consecutive
// states, so every global access is a 32-bit word of one digit plane) and
// kEpiRows side rows, one warp per row at a time.  The per-state data (x =
// u - y v, the direction, whether the state continues) and the block's T_x
// terms are staged in shared memory once.  A side row is fed by NT solution
// indices (0..5 for every shape in BASELINE.json; 1742 of the fourfold's 3003
// rows by none): rows are dispatched to a body specialised on NT, whose term
// weights (x_i + mu_i per state) live in registers across the digit loop, so
// the work per digit and state is NT byte-extract + multiply-adds and one
// balanced division by q (multiply-high, bias folded into the running carry).
constexpr int kEpiRows = 64, kEpiRowsMax = 512, kEpiTermCap = 1024, kEpiMaxNT = 6;
static_assert(kEpiRows == StepArgs{}.epi_rows, "StepArgs::epi_rows defaults to kEpiRows");
// rows per block for a batch of B states: kEpiRows when the batch fills the
// GPU, else halved (down to one row per warp) until there are >= 8 blocks per
// SM -- small batches are latency-bound, one warp per row in flight at once
inline int epi_rows_for(int B, int side, int sms) {
  static const int fixed = [] {
    const char* e = std::getenv("DRZG_EPI_ROWS");  // A/B override: 8 ... 512
    const int r = e ? std::atoi(e) : 0;
    return (r == 8 || r == 16 || r == 32 || r == 64 || r == 128 || r == 256 || r == 512) ? r : 0;
  }();
  if (fixed) return fixed;
  const int bx = (B + 127) / 128;
  int rows = kEpiRows;
  while (rows > 8 && bx * ((side + rows - 1) / rows) < 8 * sms) rows >>= 1;
  return rows;
}

// sign-extended byte j of w (one PRMT)
// (PTX prmt default mode: a selector nibble with bit 3 set replicates the
// sign of the selected byte; the __byte_perm intrinsic does not promise that)
__device__ __forceinline__ int sbyte(uint32_t w, int j) {
  const unsigned sel = (unsigned)(j | ((8 | j) << 4) | ((8 | j) << 8) | ((8 | j) << 12));
  unsigned r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(sel));
  return (int)r;
}

struct EpiCtx {
  const int8_t* Y;
  int8_t* W;
  int8_t* Bg;
  size_t plane, wplane, P;
  int s4;
  // division by q: xp = acc + tqb, tq = umulhi(xp, m32), digit = xp - q tq - h,
  // next tqb = tq + bias (bias = h + (q - 1) K folds the offset K = k22)
  unsigned m32;
  int q, h, bias, tq0;
};

template <int LD, int NT>
__device__ __forceinline__ void epi_row(const EpiCtx& c, const long long (&roff)[kEpiMaxNT], const int (&wg)[kEpiMaxNT][4],
                                        uint32_t (&out)[LD]) {
  int tqb[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) tqb[j] = c.tq0;
  auto digit = [&](int t, const uint32_t* cur) {
    int dg[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // wg[e][j] is the 16-bit weight packed into the half that meets byte j
      // of the word: one dp2a per product, no byte extraction
      int xp = tqb[j];
#pragma unroll
      for (int e = 0; e < NT; ++e) xp = j < 2 ? __dp2a_lo(wg[e][j], (int)cur[e], xp) : __dp2a_hi(wg[e][j], (int)cur[e], xp);
      const int tq = (int)__umulhi((unsigned)xp, c.m32);
      dg[j] = xp - tq * c.q - c.h;
      tqb[j] = tq + c.bias;
    }
    out[t] = __byte_perm(__byte_perm((uint32_t)dg[0], (uint32_t)dg[1], 0x0040),
                         __byte_perm((uint32_t)dg[2], (uint32_t)dg[3], 0x0040), 0x5410);
  };
  if constexpr (NT * LD <= 48) {
    // every plane's words in flight at once: the row is latency-bound, and
    // LD x NT independent 128-byte warp loads keep enough bytes in flight
    uint32_t w[LD][NT > 0 ? NT : 1];
#pragma unroll
    for (int t = 0; t < LD; ++t)
#pragma unroll
      for (int e = 0; e < NT; ++e) w[t][e] = __ldg(reinterpret_cast<const uint32_t*>(c.Y + (size_t)t * c.plane + roff[e]));
#pragma unroll
    for (int t = 0; t < LD; ++t) digit(t, w[t]);
  } else {
    uint32_t nxt[NT > 0 ? NT : 1];
#pragma unroll
    for (int e = 0; e < NT; ++e) nxt[e] = __ldg(reinterpret_cast<const uint32_t*>(c.Y + roff[e]));
#pragma unroll
    for (int t = 0; t < LD; ++t) {
      uint32_t cur[NT > 0 ? NT : 1];
#pragma unroll
      for (int e = 0; e < NT; ++e) cur[e] = nxt[e];
      if (t + 1 < LD) {
#pragma unroll
        for (int e = 0; e < NT; ++e)
          nxt[e] = __ldg(reinterpret_cast<const uint32_t*>(c.Y + (size_t)(t + 1) * c.plane + roff[e]));
      }
      digit(t, cur);
    }
  }
}

template <int LD>
__global__ void __launch_bounds__(256, 2) epilogue_kernel(StepArgs a) {
  __shared__ int xs_s[6][128];
  __shared__ int vd_s[128];
  __shared__ int ct_s[128];  // bit 0 valid, bit 1 continues
  __shared__ int tp_s[kEpiRowsMax + 1];
  __shared__ int2 tm_s[kEpiTermCap];  // {r, i | mu << 8}
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sb = blockIdx.x * 128;
  const int side = a.side;
  const int g0 = blockIdx.y * a.epi_rows, g1 = min(side, g0 + a.epi_rows);
  if (tid < 128) {
    const int s = sb + tid;
    const bool valid = s < a.B;
    const int sv = valid ? s : sb;
    const int vd = a.vdir[sv];
    vd_s[tid] = vd;
    ct_s[tid] = (valid ? 1 : 0) | ((valid && a.y < a.ks[sv]) ? 2 : 0);
    for (int i = 0; i < a.nv; ++i) xs_s[i][tid] = a.u0[(size_t)sv * a.nv + i] - a.y * a.dirs[(size_t)vd * a.nv + i];
  }
  for (int j = tid; j <= g1 - g0; j += 256) tp_s[j] = a.t_ptr[g0 + j];
  __syncthreads();
  const int e0 = tp_s[0], ne = tp_s[g1 - g0] - e0;
  const bool staged = ne <= kEpiTermCap;
  if (staged)
    for (int j = tid; j < ne; j += 256) {
      const int r = a.t_src[e0 + j];
      tm_s[j] = make_int2(r, a.sol_i[r] | (a.sol_mu[r] << 8));
    }
  __syncthreads();
  const int s4 = sb + lane * 4;
  if (s4 >= a.B) return;
  int vds[4];
  bool conts[4], valid[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    vds[j] = vd_s[lane * 4 + j];
    valid[j] = ct_s[lane * 4 + j] & 1;
    conts[j] = ct_s[lane * 4 + j] & 2;
  }
  const bool same_v = vds[0] == vds[1] && vds[0] == vds[2] && vds[0] == vds[3];
  const bool all_cont = conts[0] && conts[1] && conts[2] && conts[3];
  const bool none_cont = !conts[0] && !conts[1] && !conts[2] && !conts[3] && valid[3];
  EpiCtx c;
  c.Y = a.Y;
  c.W = a.W;
  c.Bg = a.Bg;
  c.P = (size_t)a.P;
  c.plane = (size_t)a.nLp * c.P;
  c.wplane = (size_t)a.sidep * c.P;
  c.s4 = s4;
  c.q = a.q;
  c.h = a.q >> 1;
  c.m32 = a.fq.m32;
  c.bias = c.h + (a.q - 1) * a.fq.k22;
  c.tq0 = c.h + a.q * a.fq.k22;
  const int* ginv = a.ginv;
  for (int g = g0 + warp; g < g1; g += 8) {
    const int eb = tp_s[g - g0], nt = tp_s[g - g0 + 1] - eb;
    // a row no solution index feeds (1742 of the fourfold's 3003) is zero in
    // every step's output: the step-1 epilogue zeroed its next-step operand
    // row, and no one writes that row of Bg again during the chunk
    if (a.y >= 2 && nt == 0 && all_cont) continue;
    // the write target of whole-lane words, fixed per row: W at chunk end, or
    // the next step's operand row of g under the lane's (shared) v
    const bool lane_word = none_cont || (all_cont && same_v);
    int8_t* dst = nullptr;
    if (none_cont) {
      dst = c.W + (size_t)g * c.P + s4;
    } else if (lane_word) {
      const int r0 = __ldg(ginv + (size_t)vds[0] * side + g);
      dst = r0 >= 0 ? c.Bg + (size_t)r0 * c.P + s4 : nullptr;
    }
    const size_t dstride = none_cont ? c.wplane : c.plane;
    // mixed lanes: per-state rows (rare: states are sorted by (k, v))
    int rn[4] = {-1, -1, -1, -1};
    if (!lane_word) {
#pragma unroll
      for (int j = 0; j < 4; ++j) rn[j] = conts[j] ? __ldg(ginv + (size_t)vds[j] * side + g) : -1;
    }
    auto put = [&](int t, uint32_t word) {
      if (lane_word) {
        if (dst) *reinterpret_cast<uint32_t*>(dst + (size_t)t * dstride) = word;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!valid[j]) continue;
          const int8_t b = (int8_t)(word >> (8 * j));
          if (!conts[j])
            c.W[(size_t)t * c.wplane + (size_t)g * c.P + s4 + j] = b;
          else if (rn[j] >= 0)
            c.Bg[(size_t)t * c.plane + (size_t)rn[j] * c.P + s4 + j] = b;
        }
      }
    };
    if (a.fast && nt <= kEpiMaxNT) {
      long long roff[kEpiMaxNT] = {0, 0, 0, 0, 0, 0};
      int wg[kEpiMaxNT][4];
#pragma unroll
      for (int e = 0; e < kEpiMaxNT; ++e) {
        if (e >= nt) {
#pragma unroll
          for (int j = 0; j < 4; ++j) wg[e][j] = 0;
          continue;
        }
        const int2 tm = staged ? tm_s[eb + e - e0]
                               : make_int2(a.t_src[eb + e], a.sol_i[a.t_src[eb + e]] | (a.sol_mu[a.t_src[eb + e]] << 8));
        const int ii = tm.y & 0xFF, mu = tm.y >> 8;
        roff[e] = (long long)tm.x * a.P + s4;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // |x_i + mu| < 2^15 on the multiply-high path (exponents < 4096):
          // states 0, 2 in the low half, 1, 3 in the high half (dp2a lo/hi)
          const int w = xs_s[ii][lane * 4 + j] + mu;
          wg[e][j] = (j & 1) ? (int)((unsigned)w << 16) : (w & 0xFFFF);
        }
      }
      uint32_t out[LD];
      switch (nt) {
        case 0:
#pragma unroll
          for (int t = 0; t < LD; ++t) out[t] = 0;
          break;
        case 1: epi_row<LD, 1>(c, roff, wg, out); break;
        case 2: epi_row<LD, 2>(c, roff, wg, out); break;
        case 3: epi_row<LD, 3>(c, roff, wg, out); break;
        case 4: epi_row<LD, 4>(c, roff, wg, out); break;
        case 5: epi_row<LD, 5>(c, roff, wg, out); break;
        default: epi_row<LD, 6>(c, roff, wg, out); break;
      }
      if (lane_word) {
        if (dst) {
#pragma unroll
          for (int t = 0; t < LD; ++t) *reinterpret_cast<uint32_t*>(dst + (size_t)t * dstride) = out[t];
        }
      } else {
#pragma unroll
        for (int t = 0; t < LD; ++t) put(t, out[t]);
      }
    } else {
      // wide rows (none in the BASELINE shapes) or operands beyond the
      // multiply-high range: plane loop over the terms, exact 64-bit division
      int carry[4] = {0, 0, 0, 0};
      for (int t = 0; t < LD; ++t) {
        int acc[4] = {carry[0], carry[1], carry[2], carry[3]};
        for (int e = eb; e < eb + nt; ++e) {
          const int2 tm = staged ? tm_s[e - e0] : make_int2(a.t_src[e], a.sol_i[a.t_src[e]] | (a.sol_mu[a.t_src[e]] << 8));
          const int ii = tm.y & 0xFF, mu = tm.y >> 8;
          const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(c.Y + (size_t)t * c.plane + (size_t)tm.x * c.P + s4));
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j] += (xs_s[ii][lane * 4 + j] + mu) * sbyte(w, j);
        }
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int rr;
          int qt = a.fq.divfloor(acc[j], rr);
          if (rr > c.h) rr -= c.q, ++qt;
          word |= (uint32_t)(uint8_t)(int8_t)rr << (8 * j);
          carry[j] = qt;
        }
        put(t, word);
      }
    }
  }
}
// host dispatch over the digit-plane count; the instantiations live in four
// translation units (kernels/epilogue_*.cu) so they compile in parallel
void launch_epilogue_1_8(const StepArgs& a, dim3 grid, cudaStream_t st);
void launch_epilogue_9_16(const StepArgs& a, dim3 grid, cudaStream_t st);
void launch_epilogue_17_24(const StepArgs& a, dim3 grid, cudaStream_t st);
void launch_epilogue_25_32(const StepArgs& a, dim3 grid, cudaStream_t st);
inline void launch_epilogue(const StepArgs& a, dim3 grid, cudaStream_t st) {
  if (a.Ld <= 8)
    launch_epilogue_1_8(a, grid, st);
  else if (a.Ld <= 16)
    launch_epilogue_9_16(a, grid, st);
  else if (a.Ld <= 24)
    launch_epilogue_17_24(a, grid, st);
  else
    launch_epilogue_25_32(a, grid, st);
}
#define DRZG_EPI_CASE(L)                           \
  case L:                                          \
    epilogue_kernel<L><<<grid, 256, 0, st>>>(a);   \
    break;

#ifndef DRZG_EPILOGUE_ONLY
// W -> slot pool for the batch columns [s_lo, s_hi) whose chunk ends here:
// 32 states x 64 side rows per block, transposed through shared memory
__global__ void __launch_bounds__(256) flush_kernel(StepArgs a, int s_lo, int s_hi) {
  // the block's 32 states start at a multiple of 4 at or below s_lo (word
  // loads); states below s_lo continue their chunk and are not written
  extern __shared__ __align__(16) int8_t ft[];  // Ld x kFlushRows x kFlushStates: [t][g][state]
  const int g0 = blockIdx.y * kFlushRows, s0 = (s_lo & ~3) + blockIdx.x * kFlushStates;
  const size_t wplane = (size_t)a.sidep * a.P;
  // W -> shared: one 4-state word per load (a warp reads 4 rows of 32 states)
  for (int e = threadIdx.x; e < a.Ld * kFlushRows * (kFlushStates / 4); e += 256) {
    const int sq = e % (kFlushStates / 4), gl = (e / (kFlushStates / 4)) % kFlushRows,
              t = e / ((kFlushStates / 4) * kFlushRows);
    const int g = g0 + gl, s = s0 + 4 * sq;
    uint32_t wd = 0;
    if (g < a.side && s < a.P) wd = *reinterpret_cast<const uint32_t*>(a.W + (size_t)t * wplane + (size_t)g * a.P + s);
    reinterpret_cast<uint32_t*>(ft)[e] = wd;
  }
  __syncthreads();
  // shared -> slots: a thread takes 4 side rows x 4 states, transposes them
  // (4 x 4 bytes) and writes each state's 4 rows as one word; a warp writes 16
  // consecutive words (64 bytes) of a slot row per state
  for (int e = threadIdx.x; e < a.Ld * (kFlushRows / 4) * (kFlushStates / 4); e += 256) {
    const int g4 = e % (kFlushRows / 4), sq = (e / (kFlushRows / 4)) % (kFlushStates / 4),
              t = e / ((kFlushRows / 4) * (kFlushStates / 4));
    const int g = g0 + 4 * g4;
    if (g >= a.side) continue;
    const uint32_t* rows = reinterpret_cast<const uint32_t*>(ft) + ((size_t)t * kFlushRows + 4 * g4) * (kFlushStates / 4) + sq;
    const uint32_t w0 = rows[0], w1 = rows[kFlushStates / 4], w2 = rows[2 * (kFlushStates / 4)],
                   w3 = rows[3 * (kFlushStates / 4)];
    const uint32_t lo01 = __byte_perm(w0, w1, 0x5140), hi01 = __byte_perm(w0, w1, 0x7362);
    const uint32_t lo23 = __byte_perm(w2, w3, 0x5140), hi23 = __byte_perm(w2, w3, 0x7362);
    const uint32_t st4[4] = {__byte_perm(lo01, lo23, 0x5410), __byte_perm(lo01, lo23, 0x7632),
                             __byte_perm(hi01, hi23, 0x5410), __byte_perm(hi01, hi23, 0x7632)};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int s = s0 + 4 * sq + j;
      if (s < s_lo || s >= s_hi) continue;
      *reinterpret_cast<uint32_t*>(a.pool + (size_t)a.slot[s] * a.slot_stride + (size_t)t * a.sidep + g) = st4[j];
    }
  }
}

// one block per new state: zero its slot, then write its entries (distinct
// side rows g, Ld balanced digits each)
__global__ void seed_kernel(int8_t* pool, long long slot_stride, int sidep, int Ld, const int* slot, const int* eptr,
                            const int* eg, const int8_t* edig, int nstates) {
  int i = blockIdx.x;
  if (i >= nstates) return;
  int8_t* w = pool + (size_t)slot[i] * slot_stride;
  int4* w4 = reinterpret_cast<int4*>(w);
  for (long long j = threadIdx.x; j < slot_stride / 16; j += blockDim.x) w4[j] = make_int4(0, 0, 0, 0);
  __syncthreads();
  for (int e = eptr[i] + (int)threadIdx.x / Ld; e < eptr[i + 1]; e += (int)blockDim.x / Ld) {
    int t = (int)threadIdx.x % Ld;
    if ((int)threadIdx.x < (int)(blockDim.x / Ld) * Ld) w[(size_t)t * sidep + eg[e]] = edig[(size_t)e * Ld + t];
  }
}

// seeds absorbed by a state already at their pole: w[t][g] += digits, with
// the carry normalised along t for each touched g
__global__ void add_entries_kernel(int8_t* pool, long long slot_stride, int sidep, int Ld, int q, const int* slot,
                                   const int* eptr, const int* eg, const int8_t* edig, int nstates) {
  int i = blockIdx.x;
  if (i >= nstates) return;
  int8_t* w = pool + (size_t)slot[i] * slot_stride;
  for (int e = eptr[i] + (int)threadIdx.x; e < eptr[i + 1]; e += blockDim.x) {
    const int g = eg[e];
    int carry = 0;
    for (int t = 0; t < Ld; ++t) {
      int v = (int)w[(size_t)t * sidep + g] + (int)edig[(size_t)e * Ld + t] + carry;
      int r = balmod(v, q);
      carry = (v - r) / q;
      w[(size_t)t * sidep + g] = (int8_t)r;
    }
  }
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

// the same merge with four side rows per thread (one 32-bit word of each
// member's plane per load: 128-byte warp accesses) and the digit planes in
// registers (LD a compile-time count); the multiply-high balanced division
// applies while |sum| < 2^22, i.e. up to 2^14 members a group (more: exact
// 64-bit division)
template <int LD>
__global__ void __launch_bounds__(128) merge4_kernel(int8_t* pool, long long slot_stride, int side, int sidep, FastQ fq,
                                                     const int* gptr, const int* members) {
  const int words = (side + 3) / 4;
  const int nrb = (words + blockDim.x - 1) / blockDim.x;
  const int grp = blockIdx.x / nrb;
  const int wi = (blockIdx.x % nrb) * blockDim.x + threadIdx.x;
  if (wi >= words) return;
  const int m0 = gptr[grp], m1 = gptr[grp + 1];
  int acc[LD][4];
#pragma unroll
  for (int t = 0; t < LD; ++t)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[t][j] = 0;
  for (int m = m0; m < m1; ++m) {
    const int8_t* w = pool + (size_t)members[m] * slot_stride + 4 * (size_t)wi;
    uint32_t wd[LD];
#pragma unroll
    for (int t = 0; t < LD; ++t) wd[t] = *reinterpret_cast<const uint32_t*>(w + (size_t)t * sidep);
#pragma unroll
    for (int t = 0; t < LD; ++t)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[t][j] += sbyte(wd[t], j);
  }
  int8_t* out = pool + (size_t)members[m0] * slot_stride + 4 * (size_t)wi;
  const bool fast = m1 - m0 <= (1 << 14);
  int carry[4] = {0, 0, 0, 0};
#pragma unroll
  for (int t = 0; t < LD; ++t) {
    int dg[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int v2 = acc[t][j] + carry[j];
      if (fast) {
        dg[j] = fq.balq(v2, carry[j]);
      } else {
        int r;
        int qt = fq.divfloor(v2, r);
        if (r > (fq.q >> 1)) r -= fq.q, ++qt;
        dg[j] = r;
        carry[j] = qt;
      }
    }
    *reinterpret_cast<uint32_t*>(out + (size_t)t * sidep) =
        __byte_perm(__byte_perm((uint32_t)dg[0], (uint32_t)dg[1], 0x0040), __byte_perm((uint32_t)dg[2], (uint32_t)dg[3], 0x0040),
                    0x5410);
  }
}
// combine_states over `ngroups` groups of slots (CSR gptr/members): the
// register version for Ld <= 16, else the plane loop
inline void launch_merge(int8_t* pool, long long slot_stride, int side, int sidep, int Ld, const FastQ& fq,
                         const int* gptr, const int* members, int ngroups, cudaStream_t st) {
  const int words = (side + 3) / 4;
  const dim3 g4((unsigned)((words + 127) / 128) * ngroups);
  switch (Ld) {
#define DRZG_MERGE_CASE(L) \
  case L:                  \
    merge4_kernel<L><<<g4, 128, 0, st>>>(pool, slot_stride, side, sidep, fq, gptr, members); \
    return;
    DRZG_MERGE_CASE(1) DRZG_MERGE_CASE(2) DRZG_MERGE_CASE(3) DRZG_MERGE_CASE(4) DRZG_MERGE_CASE(5) DRZG_MERGE_CASE(6)
    DRZG_MERGE_CASE(7) DRZG_MERGE_CASE(8) DRZG_MERGE_CASE(9) DRZG_MERGE_CASE(10) DRZG_MERGE_CASE(11) DRZG_MERGE_CASE(12)
    DRZG_MERGE_CASE(13) DRZG_MERGE_CASE(14) DRZG_MERGE_CASE(15) DRZG_MERGE_CASE(16)
#undef DRZG_MERGE_CASE
    default:
      break;
  }
  const dim3 gm((unsigned)((side + 127) / 128) * ngroups);
  merge_kernel<<<gm, 128, 0, st>>>(pool, slot_stride, side, sidep, Ld, fq.q, gptr, members);
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

#endif  // DRZG_EPILOGUE_ONLY

}  // namespace dev
}  // namespace drzg
