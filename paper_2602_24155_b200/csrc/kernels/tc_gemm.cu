// int8 tcgen05 GEMM with Dixon epilogues (see tc_gemm.cuh).
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <cstdlib>
#include <mutex>
#include <string>

#include "../host/common.hpp"
#include "tc_gemm.cuh"

namespace drzg {
namespace tc {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 128;  // bytes of K per stage (one 128B swizzle row)
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;
constexpr int B_BYTES = BN * BK;
constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// bounded wait: a pipeline bug traps (launch error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  for (uint32_t spin = 0;; ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    if (spin > (1u << 24)) __trap();
  }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO (ignored for swizzled K-major), canonical 1
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;            // descriptor version (sm100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
// MN-major 128B-swizzled operand: rows of 128 B along N, 8-row K groups 1 KB
// apart (SBO), 128-wide N atoms 16 KB apart (LBO); one MMA (K = 32) spans
// four K groups
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((BN / 2 * BK) >> 4) << 16;  // LBO: next N atom
  d |= (uint64_t)(1024 >> 4) << 32;           // SBO: next 8-row K group
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 16 columns (the first 16 entries of v)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ int balmod(int x, int q) {
  int r = x % q;
  if (r < 0) r += q;
  if (r > (q >> 1)) r -= q;
  return r;
}

// Persistent, warp-specialised: CTA c processes tiles c, c+grid, ... (M-tile
// fastest so concurrently running CTAs share the B tile in L2).
//   warp 0: TMA producer (4-stage smem ring)      warp 1: MMA issuer
//   warp 2: TMEM allocator                        warps 4..11: epilogue
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile i overlap
// the mainloop of tile i+1.
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + 32 * EPI_WARPS;

// M tile of persistent tile t: the M tiles of one N column are a
// contiguous run of t (so concurrently running CTAs share the B tile in L2),
// rotated by the column index so that a CTA, which sees t = c + grid * i,
// meets every M tile over its rounds (with block-sparse K the M tiles differ
// in cost; a fixed t % mt would pin each CTA to one cost class)
__device__ __forceinline__ int tile_m(int t, int mt) { return (t + t / mt) % mt; }

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// 32-byte (256-bit) per-lane global accesses: an epilogue lane owns one row
// and 32 consecutive states, so every access of a warp touches 32 different
// lines; one 256-bit instruction per line instead of two 128-bit ones halves
// the L1 wavefronts, which bound the epilogues
__device__ __forceinline__ void ld256_cg(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void ld256_nc(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void st256(void* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w),
               "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

// Dixon carry epilogue of one tile row segment: c = (r_k - Jp y_k) / q
// (exact), r_{k+1} = b_{k+1} + c, stored as in_{k+1} = bal(r_{k+1}) (the
// next digit product's operand, in place over in_k) and its quotient h_{k+1}
// (|h| <= 4), with r_k = b_0 (k = 0) or in_k + q h_k.  Software-pipelined:
// the 16-byte loads of chunk c+16 are in flight while chunk c is computed.
// COHERENT: in_k / h_k were written by other CTAs of the same launch (the
// dataflow kernel), so they are read through L2 (ld.global.cg), not the
// non-coherent read-only path.
__device__ __forceinline__ void epi_carry_prefetch(const TcEpiArgs& epi, int k, int m, bool mok, int nb) {
  if (!mok || nb >= epi.N) return;
  const size_t P = (size_t)epi.P;
  const int8_t* rlo = (k ? epi.IN : epi.Bg) + (size_t)m * P;
  asm volatile("prefetch.global.L2 [%0];" ::"l"(rlo + nb));
  asm volatile("prefetch.global.L2 [%0];" ::"l"(epi.Bg + ((size_t)(k + 1) * epi.nLp + m) * P + nb));
  if (k) asm volatile("prefetch.global.L2 [%0];" ::"l"(epi.H + (size_t)m * P + nb));
}

// sign-extended byte j of w (one PRMT: a selector nibble with bit 3 set
// replicates the sign of the selected byte)
__device__ __forceinline__ int sbyte_prmt(uint32_t w, int j) {
  const unsigned sel = (unsigned)(j | ((8 | j) << 4) | ((8 | j) << 8) | ((8 | j) << 12));
  unsigned r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(sel));
  return (int)r;
}
// the low bytes of four ints as one word (three byte permutes)
__device__ __forceinline__ uint32_t pack4_lo(int a, int b, int c, int d) {
  return __byte_perm(__byte_perm((uint32_t)a, (uint32_t)b, 0x0040), __byte_perm((uint32_t)c, (uint32_t)d, 0x0040),
                     0x5410);
}

// balanced digits of 16 int32 accumulators as four words
__device__ __forceinline__ void digits16(const FastQ& fq, bool fast, const int* v, uint32_t (&w4)[4]) {
  if (fast) {
    const unsigned hqk = fq.hqk256();
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      int raw[4], tq;
#pragma unroll
      for (int b = 0; b < 4; ++b) raw[b] = fq.split_raw(v[q4 * 4 + b], hqk, tq);
      w4[q4] = fq.unbias4(pack4_lo(raw[0], raw[1], raw[2], raw[3]));
    }
  } else {
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) word |= (uint32_t)(uint8_t)(int8_t)fq.bal(v[q4 * 4 + b]) << (8 * b);
      w4[q4] = word;
    }
  }
}
// the Dixon carry of 16 elements: c = (r - acc) / q with r = in + q h (h = 0
// when !has_h), r' = b + c stored as in' = bal(r') and h' = (r' - in') / q
__device__ __forceinline__ void carry16(const FastQ& fq, bool fast, bool has_h, const uint32_t (&low)[4],
                                        const uint32_t (&hiw)[4], const uint32_t (&b1w)[4], const int* v,
                                        uint32_t (&in4)[4], uint32_t (&h4)[4]) {
  if (fast) {
    const unsigned hqk = fq.hqk256();
#pragma unroll
    for (int w4 = 0; w4 < 4; ++w4) {
      int raw[4], tq[4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int c = fq.div_exact_inv(sbyte_prmt(low[w4], jj) - v[4 * w4 + jj]) + (has_h ? sbyte_prmt(hiw[w4], jj) : 0);
        raw[jj] = fq.split_raw(sbyte_prmt(b1w[w4], jj) + c, hqk, tq[jj]);
      }
      in4[w4] = fq.unbias4(pack4_lo(raw[0], raw[1], raw[2], raw[3]));
      h4[w4] = pack4_lo(tq[0], tq[1], tq[2], tq[3]);
    }
    return;
  }
#pragma unroll
  for (int w4 = 0; w4 < 4; ++w4) {
    in4[w4] = h4[w4] = 0;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int r = sbyte_prmt(low[w4], jj) + (has_h ? fq.q * sbyte_prmt(hiw[w4], jj) : 0);
      int rem, inb;
      const int cnew = fq.divfloor(r - v[4 * w4 + jj], rem);  // exact
      int hq = fq.divfloor(sbyte_prmt(b1w[w4], jj) + cnew, inb);
      if (inb > (fq.q >> 1)) inb -= fq.q, ++hq;
      in4[w4] |= (uint32_t)(uint8_t)(int8_t)inb << (8 * jj);
      h4[w4] |= (uint32_t)(uint8_t)(int8_t)hq << (8 * jj);
    }
  }
}

template <bool COHERENT>
__device__ __forceinline__ void epi_carry_tile(const TcEpiArgs& epi, int k, int m, bool mok, int n0, int cbeg,
                                               int cend, uint32_t tb, int cstep = 32) {
  // 32 states per step: every global access is a whole 32-byte sector
  const size_t P = (size_t)epi.P;
  const int8_t* rlo = (k ? epi.IN : epi.Bg) + (size_t)m * P;  // in_k, or b_0
  const int8_t* rhi = epi.H + (size_t)m * P;                    // h_k (k > 0)
  const int8_t* bk1p = epi.Bg + ((size_t)(k + 1) * epi.nLp + m) * P;
  const bool wh = k + 2 < epi.Ld;  // a later carry reads h_{k+1}
  auto ld = [&](const int8_t* p, uint4 (&v)[2]) {
    if (COHERENT)
      ld256_cg(p, v[0], v[1]);
    else
      ld256_nc(p, v[0], v[1]);
  };
  uint4 nlo[2], nhi[2], nb1[2];
#pragma unroll
  for (int x = 0; x < 2; ++x) nlo[x] = nhi[x] = nb1[x] = make_uint4(0, 0, 0, 0);
  auto fetch = [&](int c) {
    const int nb = n0 + c;
    if (!mok || nb >= epi.N) return;
    ld(rlo + nb, nlo);
    ld256_nc(bk1p + nb, nb1[0], nb1[1]);
    if (k) ld(rhi + nb, nhi);
  };
  fetch(cbeg);
  for (int c = cbeg; c < cend; c += cstep) {
    uint4 lo[2], hi[2], b1[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) lo[x] = nlo[x], hi[x] = nhi[x], b1[x] = nb1[x];
    if (c + cstep < cend) fetch(c + cstep);
    int v[32];
    tmem_ld32(tb + (uint32_t)c, v);
    const int nb = n0 + c;
    if (!mok || nb >= epi.N) continue;
    uint4 o_in[2], o_h[2];
    if (epi.fast) {
      // r - acc = (in - acc) + q h with q | (in - acc): c = (in - acc) q^-1 + h
      // (mod 2^32, exact), x = b_{k+1} + c; in_{k+1} = bal(x) and its
      // quotient from one multiply-high, packed four at a time
      const unsigned hqk = epi.fq.hqk256();
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const uint32_t low[4] = {lo[x].x, lo[x].y, lo[x].z, lo[x].w};
        const uint32_t hiw[4] = {hi[x].x, hi[x].y, hi[x].z, hi[x].w};
        const uint32_t b1w[4] = {b1[x].x, b1[x].y, b1[x].z, b1[x].w};
        uint32_t in4[4], h4[4];
#pragma unroll
        for (int w4 = 0; w4 < 4; ++w4) {
          int raw[4], tq[4];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int inb = sbyte_prmt(low[w4], jj);
            const int hb = k ? sbyte_prmt(hiw[w4], jj) : 0;
            const int b1j = sbyte_prmt(b1w[w4], jj);
            const int c = epi.fq.div_exact_inv(inb - v[16 * x + 4 * w4 + jj]) + hb;
            raw[jj] = epi.fq.split_raw(b1j + c, hqk, tq[jj]);
          }
          in4[w4] = epi.fq.unbias4(pack4_lo(raw[0], raw[1], raw[2], raw[3]));
          h4[w4] = pack4_lo(tq[0], tq[1], tq[2], tq[3]);
        }
        o_in[x] = make_uint4(in4[0], in4[1], in4[2], in4[3]);
        o_h[x] = make_uint4(h4[0], h4[1], h4[2], h4[3]);
      }
      st256(epi.IN + (size_t)m * P + nb, o_in[0], o_in[1]);
      if (wh) st256(epi.H + (size_t)m * P + nb, o_h[0], o_h[1]);
      continue;
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const uint32_t low[4] = {lo[x].x, lo[x].y, lo[x].z, lo[x].w};
      const uint32_t hiw[4] = {hi[x].x, hi[x].y, hi[x].z, hi[x].w};
      const uint32_t b1w[4] = {b1[x].x, b1[x].y, b1[x].z, b1[x].w};
      uint32_t in4[4] = {0, 0, 0, 0}, h4[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int sh = 8 * (j & 3);
        const int r = (int)(int8_t)(low[j >> 2] >> sh) + (k ? epi.q * (int)(int8_t)(hiw[j >> 2] >> sh) : 0);
        const int b1j = (int)(int8_t)(b1w[j >> 2] >> sh);
        const int acc = v[16 * x + j];
        int cnew, inb, hq;
        if (epi.fast) {
          cnew = epi.fq.div_exact_inv(r - acc);
          inb = epi.fq.bal_split(b1j + cnew, hq);
        } else {
          int rem;
          cnew = epi.fq.divfloor(r - acc, rem);  // exact
          hq = epi.fq.divfloor(b1j + cnew, inb);
          if (inb > (epi.q >> 1)) inb -= epi.q, ++hq;
        }
        in4[j >> 2] |= (uint32_t)(uint8_t)(int8_t)inb << sh;
        h4[j >> 2] |= (uint32_t)(uint8_t)(int8_t)hq << sh;
      }
      o_in[x] = make_uint4(in4[0], in4[1], in4[2], in4[3]);
      o_h[x] = make_uint4(h4[0], h4[1], h4[2], h4[3]);
    }
    st256(epi.IN + (size_t)m * P + nb, o_in[0], o_in[1]);
    if (wh) st256(epi.H + (size_t)m * P + nb, o_h[0], o_h[1]);
  }
}

// Dixon digit epilogue: Y[k][m][n0 + c ..] = bal(D), 32 states (one sector) per step
__device__ __forceinline__ void epi_digit_tile(const TcEpiArgs& epi, int k, int m, bool mok, int n0, int cbeg,
                                               int cend, uint32_t tb, int cstep = 32) {
  for (int c = cbeg; c < cend; c += cstep) {
    int v[32];
    tmem_ld32(tb + (uint32_t)c, v);
    const int nb = n0 + c;
    if (!mok || nb >= epi.N) continue;
    uint32_t w8[8];
    if (epi.fast) {
      const unsigned hqk = epi.fq.hqk256();
#pragma unroll
      for (int q4 = 0; q4 < 8; ++q4) {
        int raw[4], tq;
#pragma unroll
        for (int b = 0; b < 4; ++b) raw[b] = epi.fq.split_raw(v[q4 * 4 + b], hqk, tq);
        w8[q4] = epi.fq.unbias4(pack4_lo(raw[0], raw[1], raw[2], raw[3]));
      }
    } else {
#pragma unroll
      for (int q4 = 0; q4 < 8; ++q4) {
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) word |= (uint32_t)(uint8_t)(int8_t)epi.fq.bal(v[q4 * 4 + b]) << (8 * b);
        w8[q4] = word;
      }
    }
    st256(epi.Y + ((size_t)k * epi.nLp + m) * epi.P + nb, make_uint4(w8[0], w8[1], w8[2], w8[3]),
          make_uint4(w8[4], w8[5], w8[6], w8[7]));
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                uint32_t idesc, TcEpiArgs epi) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + STAGES * A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;       // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (K + BK - 1) / BK;
  const int mt = (epi.M + BM - 1) / BM, ntl = (epi.N + BN - 1) / BN;
  const int tiles = mt * ntl;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int mi = tile_m(t, mt);
        const int m0 = mi * BM, n0 = (t / mt) * BN;
        const int kb0 = epi.kb_ptr ? __ldg(epi.kb_ptr + mi) : 0;
        const int nkt = epi.kb_ptr ? __ldg(epi.kb_ptr + mi + 1) - kb0 : nk;
        for (int kb = 0; kb < nkt; ++kb, ++it) {
          const int kc = (epi.kb_ptr ? __ldg(epi.kb_idx + kb0 + kb) : kb) * BK;
          int s = it % STAGES;
          mbar_wait(smem_u32(&empty[s]), ((it / STAGES) & 1) ^ 1);
          uint32_t fb = smem_u32(&full[s]);
          mbar_expect_tx(fb, A_BYTES + B_BYTES);
          tma_load_2d(smem_u32(sA + s * A_BYTES), &tmA, fb, kc, m0);
          if (epi.b_mn) {
            // K x N operand: two 128-state-wide swizzle atoms per stage
            tma_load_2d(smem_u32(sB + s * B_BYTES), &tmB, fb, n0, kc);
            tma_load_2d(smem_u32(sB + s * B_BYTES + BN / 2 * BK), &tmB, fb, n0 + BN / 2, kc);
          } else {
            tma_load_2d(smem_u32(sB + s * B_BYTES), &tmB, fb, kc, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int acc = i & 1;
        mbar_wait(smem_u32(&tempty[acc]), ((i >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        const int mi = tile_m(t, mt);
        const int nkt = epi.kb_ptr ? __ldg(epi.kb_ptr + mi + 1) - __ldg(epi.kb_ptr + mi) : nk;
        for (int kb = 0; kb < nkt; ++kb, ++it) {
          int s = it % STAGES;
          mbar_wait(smem_u32(&full[s]), (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            mma_i8(d, sw128_desc(a0 + kk * 32),
                   epi.b_mn ? sw128_mn_desc(b0 + kk * 4096) : sw128_desc(b0 + kk * 32), idesc, (kb | kk) != 0);
          mma_commit(smem_u32(&empty[s]));
        }
        mma_commit(smem_u32(&tfull[acc]));
      }
    }
  } else if (warp >= 4) {
    // epilogue warp e: TMEM lane quarter e % 4, column half e / 4
    const int e = warp - 4;
    const int quarter = e & 3, half = e >> 2;
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int m0 = tile_m(t, mt) * BM, n0 = (t / mt) * BN;
      const int acc = i & 1;
      const int m = m0 + quarter * 32 + lane;
      const bool mok = m < epi.M;
      const bool carry = epi.b_mn && epi.mode == (int)TcEpilogue::carry;
      if (carry) epi_carry_prefetch(epi, epi.k, m, mok, n0 + half * (BN / 2));
      mbar_wait(smem_u32(&tfull[acc]), (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN);
      if (carry) {
        epi_carry_tile<false>(epi, epi.k, m, mok, n0, half * (BN / 2), (half + 1) * (BN / 2), tb);
      } else if (epi.b_mn && epi.mode == (int)TcEpilogue::digit) {
        epi_digit_tile(epi, epi.k, m, mok, n0, half * (BN / 2), (half + 1) * (BN / 2), tb);
      } else {
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 16) {
          int v[16];
          tmem_ld16(tb + (uint32_t)c, v);
          const int nb = n0 + c;
          if (!mok || nb >= epi.N) continue;
          const int cnt = min(16, epi.N - nb);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < cnt) epi.out[(size_t)(nb + j) * epi.M + m] = v[j];
        }
      }
      // all of this warp's TMEM reads of buffer `acc` are complete
      __syncwarp();
      asm volatile("tcgen05.fence::before_thread_sync;");
      if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
}

// ---------------------------------------------------------------------------
// The whole Dixon solve of a batch as ONE persistent dataflow launch (nLp >
// 256).  Tiles are (phase p, 256-state column, 128-row M tile): phase 2k is
// the digit product of digit k, phase 2k+1 the block-sparse carry of digit k.
// A tile may start when every M tile of phase p-1 of its column is done
// (global counters, acquire/release); tiles are ordered group by group
// (G columns, all phases, all M tiles) so the dependencies of a tile were
// issued ~G*mt tiles earlier and are normally complete.  Digit tiles keep
// the tensor pipe busy while carry tiles (short K loop, memory-heavy
// epilogue) interleave with them on every SM, instead of the two
// alternating as separate launches.  No deadlock: each CTA takes its tiles
// in increasing order and a tile depends only on earlier tiles.
struct FlowTile {
  int p, col, mi;
};
__device__ __forceinline__ FlowTile flow_tile(int t, int mt, int ncol, int G, int nph) {
  const int TG = nph * G * mt;
  const int gi = t / TG;
  const int r = t - gi * TG;
  const int Gc = min(G, ncol - gi * G);
  const int per = Gc * mt;
  FlowTile f;
  f.p = r / per;
  const int r2 = r - f.p * per;
  const int j = r2 / mt;
  f.col = gi * G + j;
  f.mi = (r2 - j * mt + j + f.p) % mt;  // rotate: a CTA meets every M tile
  return f;
}

__device__ __forceinline__ void flow_wait(const int* ctr, int target) {
  for (uint32_t spin = 0;; ++spin) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    __nanosleep(64);
    if (spin > (1u << 26)) __trap();
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
}

__global__ void __launch_bounds__(THREADS, 1)
    dixon_flow_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmJ,
                      const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmIn,
                      const __grid_constant__ CUtensorMap tmY, FlowArgs fa) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + STAGES * A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;       // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  const TcEpiArgs& epi = fa.epi;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = epi.nLp / BK;
  const int mt = (epi.M + BM - 1) / BM;
  const int nph = 2 * epi.Ld - 1;
  const int tiles = nph * fa.ncol * mt;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmJ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB0) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmIn) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmY) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const FlowTile f = flow_tile(t, mt, fa.ncol, fa.G, nph);
        const int k = f.p >> 1;
        const bool digit = !(f.p & 1);
        const int m0 = f.mi * BM, n0 = f.col * BN;
        if (f.p) flow_wait(fa.counters + (size_t)(f.p - 1) * fa.ncol + f.col, mt * EPI_WARPS);
        const int kb0 = digit ? 0 : __ldg(epi.kb_ptr + f.mi);
        const int nkt = digit ? nk : __ldg(epi.kb_ptr + f.mi + 1) - kb0;
        const CUtensorMap* ma = digit ? &tmC : &tmJ;
        const CUtensorMap* mb = digit ? (k ? &tmIn : &tmB0) : &tmY;
        const int rowoff = digit ? 0 : k * epi.nLp;
        for (int kb = 0; kb < nkt; ++kb, ++it) {
          const int kc = (digit ? kb : __ldg(epi.kb_idx + kb0 + kb)) * BK;
          const int s = it % STAGES;
          mbar_wait(smem_u32(&empty[s]), ((it / STAGES) & 1) ^ 1);
          const uint32_t fb = smem_u32(&full[s]);
          mbar_expect_tx(fb, A_BYTES + B_BYTES);
          tma_load_2d(smem_u32(sA + s * A_BYTES), ma, fb, kc, m0);
          tma_load_2d(smem_u32(sB + s * B_BYTES), mb, fb, n0, rowoff + kc);
          tma_load_2d(smem_u32(sB + s * B_BYTES + BN / 2 * BK), mb, fb, n0 + BN / 2, rowoff + kc);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const FlowTile f = flow_tile(t, mt, fa.ncol, fa.G, nph);
        const bool digit = !(f.p & 1);
        const int acc = i & 1;
        mbar_wait(smem_u32(&tempty[acc]), ((i >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        const int nkt = digit ? nk : __ldg(epi.kb_ptr + f.mi + 1) - __ldg(epi.kb_ptr + f.mi);
        const uint32_t idesc = digit ? fa.idesc_d : fa.idesc_c;
        for (int kb = 0; kb < nkt; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(smem_u32(&full[s]), (it / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 32; ++kk)
            mma_i8(d, sw128_desc(a0 + kk * 32), sw128_mn_desc(b0 + kk * 4096), idesc, (kb | kk) != 0);
          mma_commit(smem_u32(&empty[s]));
        }
        mma_commit(smem_u32(&tfull[acc]));
      }
    }
  } else if (warp >= 4) {
    const int e = warp - 4;
    const int quarter = e & 3, half = e >> 2;
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const FlowTile f = flow_tile(t, mt, fa.ncol, fa.G, nph);
      const int k = f.p >> 1;
      const bool digit = !(f.p & 1);
      const int m0 = f.mi * BM, n0 = f.col * BN;
      const int acc = i & 1;
      const int m = m0 + quarter * 32 + lane;
      const bool mok = m < epi.M;
      if (!digit) epi_carry_prefetch(epi, k, m, mok, n0 + half * (BN / 2));
      mbar_wait(smem_u32(&tfull[acc]), (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN);
      if (digit)
        epi_digit_tile(epi, k, m, mok, n0, half * (BN / 2), (half + 1) * (BN / 2), tb);
      else
        epi_carry_tile<true>(epi, k, m, mok, n0, half * (BN / 2), (half + 1) * (BN / 2), tb);
      __syncwarp();
      asm volatile("tcgen05.fence::before_thread_sync;");
      if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
      // publish: this warp's rows of the tile are in global memory
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(fa.counters + (size_t)f.p * fa.ncol + f.col, 1);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
}

__device__ __forceinline__ uint64_t sw128_mn_desc_1atom(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // LBO unused (one 128-wide N atom)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: next 8-row K group
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}


// ---------------------------------------------------------------------------
// The dataflow solve on CTA PAIRS (cta_group::2).  Same tiles, phases and
// counters as dixon_flow_kernel, but a tile is 256 rows of Cq / Jp x 256
// states, computed by the two CTAs of a cluster as one M = 256, N = 256
// tcgen05.mma.cta_group::2: each CTA stages its own 128 rows of A and HALF of
// B (128 states), so a K block costs each SM 32 KB of L2 -> SMEM traffic for
// 128 x 256 x 128 MACs instead of 48 KB (the single-CTA kernel was L2-bound).
// The leader CTA (rank 0) issues the MMAs; both CTAs' TMA loads complete on
// the leader's full barrier; the MMA commits multicast to both CTAs' empty /
// tfull barriers; both CTAs' epilogue warps release the accumulator on the
// leader's tempty barrier.  Each CTA drains its own TMEM lanes (its 128 rows,
// all 256 states).  Carry tiles run over the union of the two 128-row tiles'
// nonzero K blocks.
#ifndef DRZG_F2_EPI_WARPS
#define DRZG_F2_EPI_WARPS 12
#endif
namespace f2 {
// 12 epilogue warps (3 per TMEM lane quarter, each a third of the 256 state
// columns): the epilogues, not the MMAs, bound the dataflow solve, and 2
// epilogue warps per scheduler could not hide their latencies
constexpr int EPI_WARPS = DRZG_F2_EPI_WARPS;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BK;        // 16 KB: this CTA's 128 rows
constexpr int B_BYTES = (BN / 2) * BK;  // 16 KB: this CTA's 128 states
constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + 1024 + 256;
}  // namespace f2

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's shared memory, completing on an mbarrier of either CTA of the pair
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(dst),
      "l"(map), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive (once) on the barrier at this shared offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          bar)
      : "memory");
}
// The pair kernel's schedule: rounds of exactly one tile per cluster (the
// grid is G * mt2 clusters, a round is one phase of one G-column group).
// Three streams of column groups run one phase apart, round-robin, so every
// cluster alternates digit and carry tiles: the long carry epilogue of one
// tile overlaps the long digit MMA of the next (two carry tiles in a row left
// the tensor pipe waiting on TMEM).  A tile's dependency (the previous phase
// of its columns) is two rounds old.
__device__ __forceinline__ bool flow2_slot(int r, int j, const FlowArgs& fa, int mt2, int nph, FlowTile& f) {
  const int S = fa.streams;
  const int st = r % S, q = r / S;
  const int item = q - st;
  if (item < 0) return false;
  const int ph = item % nph, gs = item / nph;
  const int group = st + S * gs;
  if (group >= fa.ngroups) return false;
  const int cg = j / mt2;
  const int col = group * fa.G + cg;
  if (cg >= fa.G || col >= fa.ncol) return false;
  f.p = ph;
  f.col = col;
  f.mi = (j % mt2 + cg + ph) % mt2;
  return true;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
// the whole warp waits for a phase counter: lane 0 polls with relaxed loads
// (an acquire per poll would invalidate L1 every time), then one acquire fence
__device__ __forceinline__ void flow_wait_warp(const int* ctr, int target, int lane) {
  if (lane == 0) {
    for (uint32_t spin = 0;; ++spin) {
      int v;
      asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      __nanosleep(32);
      if (spin > (1u << 27)) __trap();
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
  }
  __syncwarp();
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__global__ void __launch_bounds__(f2::THREADS, 1)
    dixon_flow2_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmJ,
                       const __grid_constant__ CUtensorMap tmB0, const __grid_constant__ CUtensorMap tmIn,
                       const __grid_constant__ CUtensorMap tmY, FlowArgs fa) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + f2::STAGES * f2::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + f2::STAGES * f2::B_BYTES);
  uint64_t* full = bars;                           // leader's is used
  uint64_t* empty = bars + f2::STAGES;             // each CTA's own
  uint64_t* tfull = bars + 2 * f2::STAGES;         // [2], each CTA's own
  uint64_t* tempty = bars + 2 * f2::STAGES + 2;    // [2], leader's is used
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * f2::STAGES + 4);
  const TcEpiArgs& epi = fa.epi;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int nk = epi.nLp / BK;
  const int mt = (epi.M + BM - 1) / BM;  // 128-row tiles (counter targets)
  const int mt2 = (mt + 1) / 2;          // 256-row pair tiles
  const int nph = 2 * epi.Ld - 1;
  const int cid = blockIdx.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < f2::STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&tfull[b]), 1);
      mbar_init(smem_u32(&tempty[b]), 2 * f2::EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmJ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB0) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmIn) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmY) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote use
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  // producer and MMA roles run warp-uniformly (every lane walks the loop, one
  // elected lane issues): the stage / phase / descriptor arithmetic then lives
  // in uniform registers instead of being re-broadcast for every instruction
  if (warp == 0) {
    int s = 0;
    uint32_t ph = 0;
    const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);
    for (int r = 0; r < fa.rounds; ++r) {
      FlowTile f;
      if (!flow2_slot(r, cid, fa, mt2, nph, f)) continue;
      const int k = f.p >> 1;
      const bool digit = !(f.p & 1);
      const int m0 = f.mi * (2 * BM) + (int)rank * BM, n0 = f.col * BN + (int)rank * (BN / 2);
      // every CTA of every pair tile of the previous phase publishes (also
      // the half of a last pair that lies beyond the system when mt is odd)
      if (f.p) flow_wait_warp(fa.counters + (size_t)(f.p - 1) * fa.ncol + f.col, 2 * mt2 * f2::EPI_WARPS, lane);
      const int kb0 = digit ? 0 : __ldg(fa.kb2_ptr + f.mi);
      const int nkt = digit ? nk : __ldg(fa.kb2_ptr + f.mi + 1) - kb0;
      const CUtensorMap* ma = digit ? &tmC : &tmJ;
      const CUtensorMap* mb = digit ? (k ? &tmIn : &tmB0) : &tmY;
      const int rowoff = digit ? 0 : k * epi.nLp;
      for (int kb = 0; kb < nkt; ++kb) {
        const int kc = (digit ? kb : __ldg(fa.kb2_idx + kb0 + kb)) * BK;
        mbar_wait(smem_u32(&empty[s]), ph ^ 1);
        if (elect_one()) {
          if (rank == 0) mbar_expect_tx(smem_u32(&full[s]), 2 * (f2::A_BYTES + f2::B_BYTES));
          tma_load_2d_pair(smem_u32(sA + s * f2::A_BYTES), ma, full0 + 8 * s, kc, m0);
          tma_load_2d_pair(smem_u32(sB + s * f2::B_BYTES), mb, full0 + 8 * s, n0, rowoff + kc);
        }
        __syncwarp();
        if (++s == f2::STAGES) s = 0, ph ^= 1;
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      int s = 0, i = 0;
      uint32_t ph = 0;
      // descriptors: start address (>> 4) in bits 0-13; one MMA (K = 32)
      // advances A by 32 bytes and B by 32 rows of 128 bytes
      const uint64_t adesc0 = sw128_desc(smem_u32(sA)), bdesc0 = sw128_mn_desc_1atom(smem_u32(sB));
      for (int r = 0; r < fa.rounds; ++r) {
        FlowTile f;
        if (!flow2_slot(r, cid, fa, mt2, nph, f)) continue;
        const bool digit = !(f.p & 1);
        const int acc = i & 1;
        mbar_wait(smem_u32(&tempty[acc]), ((i >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + (uint32_t)(acc * BN);
        const int nkt = digit ? nk : __ldg(fa.kb2_ptr + f.mi + 1) - __ldg(fa.kb2_ptr + f.mi);
        const uint32_t idesc = digit ? fa.idesc_d : fa.idesc_c;
        for (int kb = 0; kb < nkt; ++kb) {
          mbar_wait(smem_u32(&full[s]), ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint64_t ad = adesc0 + (uint64_t)((s * f2::A_BYTES) >> 4);
          const uint64_t bd = bdesc0 + (uint64_t)((s * f2::B_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 32; ++kk)
              mma_i8_pair(d, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 256), idesc, (kb | kk) != 0);
            mma_commit_pair(smem_u32(&empty[s]));
          }
          __syncwarp();
          if (++s == f2::STAGES) s = 0, ph ^= 1;
        }
        if (elect_one()) mma_commit_pair(smem_u32(&tfull[acc]));
        __syncwarp();
        ++i;
      }
    }
  } else if (warp >= 4) {
    const int e = warp - 4;
    // TMEM lane quarter (warp % 4) and which third of the 32-column chunks
    const int quarter = e & 3, part = e >> 2;
    const int cbeg = part * 32, cstep = 32 * (f2::EPI_WARPS / 4);
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
    int i = 0;
    for (int r = 0; r < fa.rounds; ++r) {
      FlowTile f;
      if (!flow2_slot(r, cid, fa, mt2, nph, f)) continue;
      const int k = f.p >> 1;
      const bool digit = !(f.p & 1);
      const int m0 = f.mi * (2 * BM) + (int)rank * BM, n0 = f.col * BN;
      const int acc = i & 1;
      const int m = m0 + quarter * 32 + lane;
      const bool mok = m < epi.M;
      if (!digit) epi_carry_prefetch(epi, k, m, mok, n0 + cbeg);
      mbar_wait(smem_u32(&tfull[acc]), (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t tb = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN);
      if (fa.debug == 1) {
        for (int c = cbeg; c < BN; c += cstep) {
          int v[32];
          tmem_ld32(tb + (uint32_t)c, v);
          if (v[0] == 0x7fffffff) fa.counters[0] = v[1];  // keep the loads
        }
      } else if (fa.debug == 2) {
      } else if (fa.debug == 3) {
        // the epilogue arithmetic without its global memory (inputs zero,
        // results kept alive): separates the two costs
        uint32_t sink = 0;
        for (int c = cbeg; c < BN; c += cstep) {
          int v[32];
          tmem_ld32(tb + (uint32_t)c, v);
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            if (digit) {
              uint32_t w4[4];
              digits16(epi.fq, epi.fast, v + 16 * x, w4);
              sink ^= w4[0] ^ w4[1] ^ w4[2] ^ w4[3];
            } else {
              const uint32_t z[4] = {0, 0, 0, 0};
              uint32_t in4[4], h4[4];
              carry16(epi.fq, epi.fast, k != 0, z, z, z, v + 16 * x, in4, h4);
              sink ^= in4[0] ^ in4[1] ^ in4[2] ^ in4[3] ^ h4[0] ^ h4[1] ^ h4[2] ^ h4[3];
            }
          }
        }
        if (sink == 0x12345678u) fa.counters[0] = (int)sink;
      } else if (digit)
        epi_digit_tile(epi, k, m, mok, n0, cbeg, BN, tb, cstep);
      else
        epi_carry_tile<true>(epi, k, m, mok, n0, cbeg, BN, tb, cstep);
      __syncwarp();
      asm volatile("tcgen05.fence::before_thread_sync;");
      if (lane == 0) mbar_arrive_cluster(tempty0 + (uint32_t)(acc * sizeof(uint64_t)));
      // publish: the warp barrier orders every lane's stores of the tile
      // before lane 0's gpu-scope release (cumulative), which the consumer's
      // acquire fence pairs with
      __syncwarp();
      if (lane == 0)
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(fa.counters + (size_t)f.p * fa.ncol + f.col)
                     : "memory");
      ++i;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();  // the peer's MMAs and remote arrivals are over before the TMEM goes
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
}

// ---------------------------------------------------------------------------
// Whole Dixon solve of a 128-state block in one CTA, for systems with
// nLp <= 256 (the K3 surface: nL = 220).  Cq and Jp stay in shared memory
// for the kernel's lifetime; in_k, y_k and the residual high part h_k live in
// shared memory in the 128B-swizzled MN-major layout the MMA reads; each
// digit is two tcgen05 products (Cq . in_k into TMEM columns [0, 256), Jp .
// y_k into [256, 512)) separated by epilogues that write y_k (to shared memory
// and to the global Y plane for the T_x epilogue) and in_{k+1}, h_{k+1}.  One
// launch per pole drop instead of 2 Ld - 1, no intermediate HBM traffic
// except b_{k+1} in and y_k out.
//   warp 0: TMA (Cq, Jp once; b_0 per block)   warp 1: MMA issuer
//   warp 2: TMEM allocator                     warps 4..11: epilogue
namespace fz {
constexpr int TILE = 128 * 128;  // a 128 x 128 tile of Cq / Jp
constexpr int EPI_WARPS = 16;    // lane quarter x M tile x state half
constexpr int THREADS = 128 + 32 * EPI_WARPS;
// NS states per block: 128 (128B-swizzled in/y/h rows), 64 (64B-swizzled)
// or 32 (32B-swizzled): smaller blocks give small batches, whose launches
// are latency-bound, more CTAs and shorter per-digit epilogue phases
__host__ __device__ constexpr int box_bytes(int NS) { return NS * 128; }
__host__ __device__ constexpr int smem_bytes(int nt, int NS) {
  return 2 * nt * nt * TILE + 3 * nt * box_bytes(NS) + 1024 + 256;
}
}  // namespace fz

// byte offset of (K row r, state s) in a 128B-swizzled MN-major box set
// (one 16 KB box per 128 K rows; rows of 128 states)
template <int NS>
__device__ __forceinline__ uint32_t swz(int r, int s) {
  if (NS == 128)
    return (uint32_t)((r >> 7) * fz::box_bytes(NS) + (r & 127) * 128 + ((((s >> 4) ^ (r & 7)) & 7) << 4) + (s & 15));
  if (NS == 64)
    return (uint32_t)((r >> 7) * fz::box_bytes(NS) + (r & 127) * 64 + ((((s >> 4) ^ (r >> 1)) & 3) << 4) + (s & 15));
  return (uint32_t)((r >> 7) * fz::box_bytes(NS) + (r & 127) * 32 + ((((s >> 4) ^ (r >> 2)) & 1) << 4) + (s & 15));
}
// MN-major B operand descriptor for one NS-wide atom (SBO: next 8-row K group)
template <int NS>
__device__ __forceinline__ uint64_t mn_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * NS) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(NS == 128 ? 2 : NS == 64 ? 4 : 6) << 61;  // SWIZZLE_128B / 64B / 32B
  return d;
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }


// chunk mode: steps of block b (its first state's k; states are sorted by k
// descending), else one
__device__ __forceinline__ int fused_steps(const FusedArgs& fa, int b, int NS) {
  if (!fa.chunk) return 1;
  const long long k = __ldg(reinterpret_cast<const long long*>(fa.ks) + (size_t)b * NS);
  return k < 1 ? 1 : (int)k;
}

// chunk mode: w' = T_x y for the block's states at step y (the T_x
// epilogue of the reduction step, reduction.hpp:394-423 / DESIGN.md): side
// row g of state s gets sum over the solution indices r feeding g of
// (x_i + mu_i) y[r], x = u0 - y v, carry-normalised into Ld balanced digits;
// written to the next step's operand row ginv[v][g] of Bg while the chunk
// continues (y < k), to W at its last step (y == k), nothing after it.
// Thread `et` of the 16 epilogue warps: state et % NS, rows g = et / NS + j
// (512 / NS).  y comes from shared memory (the block's Ld planes, sYall).
__device__ __forceinline__ void fused_tx_phase(const FusedArgs& fa, int b, int y, int NS, int et,
                                               const int8_t* sYall) {
  constexpr int kThreads = 32 * fz::EPI_WARPS;
  const int sl = et % NS, grp = et / NS, ngrp = kThreads / NS;
  const int s = b * NS + sl;
  if (s >= fa.N) return;
  const long long ks = __ldg(reinterpret_cast<const long long*>(fa.ks) + s);
  if (y > ks) return;
  const bool cont = y < ks;
  const int vd = __ldg(fa.vdir + s);
  int x[6] = {0, 0, 0, 0, 0, 0};
  for (int i2 = 0; i2 < fa.nv; ++i2) x[i2] = __ldg(fa.u0 + (size_t)s * fa.nv + i2) - y * __ldg(fa.dirs + (size_t)vd * fa.nv + i2);
  const size_t P = (size_t)fa.P, plane = (size_t)fa.nLp * P, wplane = (size_t)fa.sidep * P;
  const int h = fa.q >> 1;
  for (int g = grp; g < fa.side; g += ngrp) {
    const int tb = __ldg(fa.t_ptr + g), te = __ldg(fa.t_ptr + g + 1);
    int rr[6], ww[6];
    const int nt = te - tb < 6 ? te - tb : 6;
    for (int e2 = 0; e2 < nt; ++e2) {
      const int r = __ldg(fa.t_src + tb + e2);
      rr[e2] = r;
      ww[e2] = x[__ldg(fa.sol_i + r)] + __ldg(fa.sol_mu + r);
    }
    const int rn = cont ? __ldg(fa.ginv + (size_t)vd * fa.side + g) : -1;
    int carry = 0;
    for (int t = 0; t < fa.Ld; ++t) {
      int acc = carry;
      const int8_t* yt = sYall + (size_t)t * fa.nLp * NS + sl;
      for (int e2 = 0; e2 < nt; ++e2) acc += ww[e2] * (int)yt[(size_t)rr[e2] * NS];
      for (int e2 = 6; e2 < te - tb; ++e2) {  // wide rows (none in the BASELINE shapes)
        const int r = __ldg(fa.t_src + tb + e2);
        acc += (x[__ldg(fa.sol_i + r)] + __ldg(fa.sol_mu + r)) * (int)yt[(size_t)r * NS];
      }
      int rem;
      int qt = fa.fq.divfloor(acc, rem);
      if (rem > h) rem -= fa.q, ++qt;
      carry = qt;
      if (cont) {
        if (rn >= 0) const_cast<int8_t*>(fa.Bg)[t * plane + (size_t)rn * P + s] = (int8_t)rem;
      } else {
        fa.W[t * wplane + (size_t)g * P + s] = (int8_t)rem;
      }
    }
  }
}

template <int NS>
__global__ void __launch_bounds__(fz::THREADS, 1)
    dixon_fused_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmJ,
                       const __grid_constant__ CUtensorMap tmB0, uint32_t idesc_c, uint32_t idesc_j, FusedArgs fa) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nt = fa.nLp / 128;
  uint8_t* sC = base;                       // nt x nt tiles (M tile mt, K box kb) at (mt * nt + kb)
  uint8_t* sJ = sC + nt * nt * fz::TILE;
  uint8_t* sIn = sJ + nt * nt * fz::TILE;   // nt boxes
  uint8_t* sY = sIn + nt * fz::box_bytes(NS);
  uint8_t* sH = sY + nt * fz::box_bytes(NS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sH + nt * fz::box_bytes(NS));
  // chunk mode: every y plane of the block, [k][row][state], for the in-CTA T_x
  int8_t* sYall = reinterpret_cast<int8_t*>(reinterpret_cast<uint8_t*>(bars) + 256);
  uint64_t* barA = bars;      // Cq, Jp loaded
  uint64_t* barB0 = bars + 1; // b_0 of the block loaded
  uint64_t* barD = bars + 2;  // digit product done
  uint64_t* barC = bars + 3;  // carry product done
  uint64_t* barY = bars + 4;  // y_k drained (every epilogue warp)
  uint64_t* barIn = bars + 5; // in_{k+1}, h_{k+1} written (every epilogue warp)
  uint64_t* barFree = bars + 6;  // a block's last digit product done: sIn may be refilled
  uint64_t* barTx = bars + 7;    // chunk mode: T_x of the block's step written (every epilogue warp)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Ld = fa.Ld;
  const int nblk = (fa.N + NS - 1) / NS;

  if (threadIdx.x == 0) {
    mbar_init(smem_u32(barA), 1);
    mbar_init(smem_u32(barB0), 1);
    mbar_init(smem_u32(barD), 1);
    mbar_init(smem_u32(barC), 1);
    mbar_init(smem_u32(barY), fz::EPI_WARPS);
    mbar_init(smem_u32(barIn), fz::EPI_WARPS);
    mbar_init(smem_u32(barFree), 1);
    mbar_init(smem_u32(barTx), fz::EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmJ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB0) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(smem_u32(barA), (uint32_t)(2 * nt * nt * fz::TILE));
      for (int mt = 0; mt < nt; ++mt)
        for (int kb = 0; kb < nt; ++kb) {
          tma_load_2d(smem_u32(sC + (mt * nt + kb) * fz::TILE), &tmC, smem_u32(barA), kb * 128, mt * 128);
          tma_load_2d(smem_u32(sJ + (mt * nt + kb) * fz::TILE), &tmJ, smem_u32(barA), kb * 128, mt * 128);
        }
      int i = 0;
      for (int b = blockIdx.x; b < nblk; b += gridDim.x)
        for (int y = 1, ny = fused_steps(fa, b, NS); y <= ny; ++y, ++i) {
          // the previous item's last digit product has consumed sIn (a
          // barrier of its own: barD runs Ld phases per item, and a parity
          // wait only tells the current phase from the one before it)
          if (i) mbar_wait(smem_u32(barFree), (uint32_t)((i - 1) & 1));
          // chunk mode, later steps: the block's T_x wrote this step's b (Bg)
          if (y > 1) mbar_wait(smem_u32(barTx), (uint32_t)((i - 1) & 1));
          mbar_expect_tx(smem_u32(barB0), (uint32_t)(nt * fz::box_bytes(NS)));
          for (int kb = 0; kb < nt; ++kb)
            tma_load_2d(smem_u32(sIn + kb * fz::box_bytes(NS)), &tmB0, smem_u32(barB0), b * NS, kb * 128);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(smem_u32(barA), 0);
      int i = 0;
      for (int b = blockIdx.x; b < nblk; b += gridDim.x)
        for (int y = 1, ny = fused_steps(fa, b, NS); y <= ny; ++y, ++i) {
        if (i) mbar_wait(smem_u32(barY), (uint32_t)((i * Ld - 1) & 1));  // last digit drained
        mbar_wait(smem_u32(barB0), (uint32_t)(i & 1));
        for (int k = 0; k < Ld; ++k) {
          const int d = i * Ld + k;
          if (k) mbar_wait(smem_u32(barIn), (uint32_t)((i * (Ld - 1) + k - 1) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;");
          for (int mt = 0; mt < nt; ++mt)
            for (int kb = 0; kb < nt; ++kb) {
              const uint32_t a0 = smem_u32(sC + (mt * nt + kb) * fz::TILE),
                             b0 = smem_u32(sIn + kb * fz::box_bytes(NS));
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_i8(tmem + (uint32_t)(mt * NS), sw128_desc(a0 + kk * 32), mn_desc<NS>(b0 + kk * 32 * NS), idesc_c,
                       (kb | kk) != 0);
            }
          mma_commit(smem_u32(barD));
          if (k + 1 == Ld) mma_commit(smem_u32(barFree));
          if (k + 1 < Ld) {
            mbar_wait(smem_u32(barY), (uint32_t)(d & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int mt = 0; mt < nt; ++mt)
              for (int kb = 0; kb < nt; ++kb) {
                const uint32_t a0 = smem_u32(sJ + (mt * nt + kb) * fz::TILE),
                               b0 = smem_u32(sY + kb * fz::box_bytes(NS));
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_i8(tmem + (uint32_t)(256 + mt * NS), sw128_desc(a0 + kk * 32), mn_desc<NS>(b0 + kk * 32 * NS),
                         idesc_j, (kb | kk) != 0);
              }
            mma_commit(smem_u32(barC));
          }
        }
      }
    }
  } else if (warp >= 4) {
    // epilogue warp e: TMEM lane quarter e % 4, M tile (e / 4) % 2, states
    // [NS/2 (e / 8), +NS/2); every phase drains NS/2 accumulators per thread
    // with 32-column TMEM loads
    const int e = warp - 4, quarter = e & 3, mt = (e >> 2) & 1, half = e >> 3;
    const int m = mt * 128 + quarter * 32 + lane;  // K row of in / y, M row of the products
    const bool active = mt < nt;
    const uint32_t lanebase = tmem + ((uint32_t)(quarter * 32) << 16);
    const size_t P = (size_t)fa.P;
    const bool tr = fa.trace && blockIdx.x == 0 && threadIdx.x == 128;
    auto stamp = [&](int slot) {
      if (tr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        fa.trace[slot] = (long long)t;
      }
    };
    stamp(0);
    int i = 0;
    for (int b = blockIdx.x; b < nblk; b += gridDim.x)
      for (int y = 1, ny = fused_steps(fa, b, NS); y <= ny; ++y, ++i) {
      const int n0 = b * NS + half * (NS / 2);
      constexpr int NCH = NS / 32;           // 16-state chunks per thread
      constexpr int PER = NCH >= 2 ? 2 : 1;  // chunks per TMEM load (32 or 16 columns)
      for (int k = 0; k < Ld; ++k) {
        const int d = i * Ld + k;
        const bool carry = k + 1 < Ld;
        // b_{k+1} for this thread's row: independent of the products, in flight early
        uint4 b1[NCH];
        if (carry && active) {
          const int8_t* src = fa.Bg + ((size_t)(k + 1) * fa.nLp + m) * P + n0;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
            b1[ch] = n0 + ch * 16 < fa.N ? __ldcg(reinterpret_cast<const uint4*>(src + ch * 16)) : make_uint4(0, 0, 0, 0);
        }
        mbar_wait(smem_u32(barD), (uint32_t)(d & 1));
        if (i == 0) stamp(1 + 4 * k);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (active) {
          int8_t* yg = fa.Y + ((size_t)k * fa.nLp + m) * P + n0;
#pragma unroll
          for (int hh = 0; hh < NCH / PER; ++hh) {
            int v[32];
            if constexpr (PER == 2)
              tmem_ld32(lanebase + (uint32_t)(mt * NS + half * (NS / 2) + hh * 32), v);
            else
              tmem_ld16(lanebase + (uint32_t)(mt * NS + half * (NS / 2) + hh * 16), v);
#pragma unroll
            for (int c2 = 0; c2 < PER; ++c2) {
              const int ch = hh * PER + c2;
              uint32_t w4[4];
              digits16(fa.fq, fa.fast, v + c2 * 16, w4);
              const uint4 y4 = make_uint4(w4[0], w4[1], w4[2], w4[3]);
              if (carry) *reinterpret_cast<uint4*>(sY + swz<NS>(m, half * (NS / 2) + ch * 16)) = y4;
              if (fa.chunk)
                *reinterpret_cast<uint4*>(sYall + ((size_t)k * fa.nLp + m) * NS + half * (NS / 2) + ch * 16) = y4;
              else if (m < fa.nL && n0 + ch * 16 < fa.N)
                *reinterpret_cast<uint4*>(yg + ch * 16) = y4;
            }
          }
        }
        fence_async_smem();
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(barY));
        if (i == 0) stamp(2 + 4 * k);
        if (!carry) continue;
        if (k == 0) mbar_wait(smem_u32(barB0), (uint32_t)(i & 1));  // b_0 (TMA) is r_0
        mbar_wait(smem_u32(barC), (uint32_t)((i * (Ld - 1) + k) & 1));
        if (i == 0) stamp(3 + 4 * k);
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (active) {
#pragma unroll
          for (int hh = 0; hh < NCH / PER; ++hh) {
            int v[32];
            if constexpr (PER == 2)
              tmem_ld32(lanebase + (uint32_t)(256 + mt * NS + half * (NS / 2) + hh * 32), v);
            else
              tmem_ld16(lanebase + (uint32_t)(256 + mt * NS + half * (NS / 2) + hh * 16), v);
#pragma unroll
            for (int c2 = 0; c2 < PER; ++c2) {
              const int ch = hh * PER + c2;
              const uint32_t off = swz<NS>(m, half * (NS / 2) + ch * 16);
              const uint4 lo = *reinterpret_cast<const uint4*>(sIn + off);
              const uint4 hi = k ? *reinterpret_cast<const uint4*>(sH + off) : make_uint4(0, 0, 0, 0);
              const uint32_t low[4] = {lo.x, lo.y, lo.z, lo.w};
              const uint32_t hiw[4] = {hi.x, hi.y, hi.z, hi.w};
              const uint32_t b1w[4] = {b1[ch].x, b1[ch].y, b1[ch].z, b1[ch].w};
              uint32_t in4[4], h4[4];
              carry16(fa.fq, fa.fast, k != 0, low, hiw, b1w, v + c2 * 16, in4, h4);
              *reinterpret_cast<uint4*>(sIn + off) = make_uint4(in4[0], in4[1], in4[2], in4[3]);
              *reinterpret_cast<uint4*>(sH + off) = make_uint4(h4[0], h4[1], h4[2], h4[3]);
            }
          }
        }
        fence_async_smem();
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(barIn));
        if (i == 0) stamp(4 + 4 * k);
      }
      if (fa.chunk) {
        // every y plane of the block is in shared memory
        asm volatile("bar.sync 1, %0;" ::"r"(32 * fz::EPI_WARPS) : "memory");
        fused_tx_phase(fa, b, y, NS, e * 32 + lane, sYall);
        // generic writes of Bg before the producer's TMA reads of the next
        // step, and before any warp's next-step reads of Bg and sYall
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(32 * fz::EPI_WARPS) : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(barTx));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// Two blocks in flight per CTA ("ping-pong"): the fused solve above, with two
// NS-state blocks (parities p = 0, 1) processed in lockstep through their
// digits.  Each has its own in/y/h shared-memory boxes and TMEM accumulators
// (digit products at columns 128 p, carry products at 256 + 128 p), so while
// the epilogue warps drain one block's phase the MMA unit computes the other
// block's: the per-digit MMA waits (~0.9 us each of a ~3.9 us digit) leave
// the critical path.  Order per digit k: D(0,k) D(1,k) | Y(0,k) -> C(0,k),
// Y(1,k) -> C(1,k) | In(0,k) -> D(0,k+1), In(1,k) -> D(1,k+1).  Barrier phase
// of pair j, digit k: j Ld + k (D, Y), j (Ld - 1) + k (C, In), j (B0, Free).
// Same products and epilogue arithmetic per block: identical results.
namespace fz {
__host__ __device__ constexpr int smem_bytes_pp(int nt, int NS) { return 2 * nt * nt * TILE + 6 * nt * box_bytes(NS) + 1024 + 256; }
}  // namespace fz

template <int NS>
__global__ void __launch_bounds__(fz::THREADS, 1)
    dixon_fused_pp_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmJ,
                          const __grid_constant__ CUtensorMap tmB0, uint32_t idesc_c, uint32_t idesc_j, FusedArgs fa) {
  static_assert(NS <= 64, "two blocks' accumulators must fit 128 TMEM columns each");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nt = fa.nLp / 128;
  uint8_t* sC = base;
  uint8_t* sJ = sC + nt * nt * fz::TILE;
  uint8_t* sIn[2];
  uint8_t* sY[2];
  uint8_t* sH[2];
  {
    uint8_t* q0 = sJ + nt * nt * fz::TILE;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      sIn[p] = q0;
      sY[p] = q0 + nt * fz::box_bytes(NS);
      sH[p] = q0 + 2 * nt * fz::box_bytes(NS);
      q0 += 3 * nt * fz::box_bytes(NS);
    }
  }
  uint64_t* bars = reinterpret_cast<uint64_t*>(sH[1] + nt * fz::box_bytes(NS));
  uint64_t* barA = bars;
  uint64_t* barB0 = bars + 1;    // [2] b_0 of the block loaded
  uint64_t* barD = bars + 3;     // [2] digit product done
  uint64_t* barC = bars + 5;     // [2] carry product done
  uint64_t* barY = bars + 7;     // [2] y_k drained
  uint64_t* barIn = bars + 9;    // [2] in_{k+1}, h_{k+1} written
  uint64_t* barFree = bars + 11; // [2] the block's last digit product done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Ld = fa.Ld;
  const int nblk = (fa.N + NS - 1) / NS;
  const int nmine = blockIdx.x < nblk ? (nblk - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int npairs = (nmine + 1) / 2;
  auto blk = [&](int j, int p) { return blockIdx.x + (2 * j + p) * gridDim.x; };
  auto has = [&](int j, int p) { return 2 * j + p < nmine; };

  if (threadIdx.x == 0) {
    mbar_init(smem_u32(barA), 1);
    for (int p = 0; p < 2; ++p) {
      mbar_init(smem_u32(barB0 + p), 1);
      mbar_init(smem_u32(barD + p), 1);
      mbar_init(smem_u32(barC + p), 1);
      mbar_init(smem_u32(barY + p), fz::EPI_WARPS);
      mbar_init(smem_u32(barIn + p), fz::EPI_WARPS);
      mbar_init(smem_u32(barFree + p), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmJ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB0) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(smem_u32(barA), (uint32_t)(2 * nt * nt * fz::TILE));
      for (int mt = 0; mt < nt; ++mt)
        for (int kb = 0; kb < nt; ++kb) {
          tma_load_2d(smem_u32(sC + (mt * nt + kb) * fz::TILE), &tmC, smem_u32(barA), kb * 128, mt * 128);
          tma_load_2d(smem_u32(sJ + (mt * nt + kb) * fz::TILE), &tmJ, smem_u32(barA), kb * 128, mt * 128);
        }
      for (int j = 0; j < npairs; ++j)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          if (!has(j, p)) continue;
          if (j) mbar_wait(smem_u32(barFree + p), (uint32_t)((j - 1) & 1));
          mbar_expect_tx(smem_u32(barB0 + p), (uint32_t)(nt * fz::box_bytes(NS)));
          for (int kb = 0; kb < nt; ++kb)
            tma_load_2d(smem_u32(sIn[p] + kb * fz::box_bytes(NS)), &tmB0, smem_u32(barB0 + p), blk(j, p) * NS,
                        kb * 128);
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(smem_u32(barA), 0);
      for (int j = 0; j < npairs; ++j)
        for (int k = 0; k < Ld; ++k) {
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            if (!has(j, p)) continue;
            if (k == 0) {
              if (j) mbar_wait(smem_u32(barY + p), (uint32_t)((j * Ld - 1) & 1));  // previous block drained
              mbar_wait(smem_u32(barB0 + p), (uint32_t)(j & 1));
            } else {
              mbar_wait(smem_u32(barIn + p), (uint32_t)((j * (Ld - 1) + k - 1) & 1));
            }
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int mt = 0; mt < nt; ++mt)
              for (int kb = 0; kb < nt; ++kb) {
                const uint32_t a0 = smem_u32(sC + (mt * nt + kb) * fz::TILE),
                               b0 = smem_u32(sIn[p] + kb * fz::box_bytes(NS));
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_i8(tmem + (uint32_t)(128 * p + mt * NS), sw128_desc(a0 + kk * 32), mn_desc<NS>(b0 + kk * 32 * NS),
                         idesc_c, (kb | kk) != 0);
              }
            mma_commit(smem_u32(barD + p));
            if (k + 1 == Ld) mma_commit(smem_u32(barFree + p));
          }
          if (k + 1 == Ld) continue;
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            if (!has(j, p)) continue;
            mbar_wait(smem_u32(barY + p), (uint32_t)((j * Ld + k) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int mt = 0; mt < nt; ++mt)
              for (int kb = 0; kb < nt; ++kb) {
                const uint32_t a0 = smem_u32(sJ + (mt * nt + kb) * fz::TILE),
                               b0 = smem_u32(sY[p] + kb * fz::box_bytes(NS));
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_i8(tmem + (uint32_t)(256 + 128 * p + mt * NS), sw128_desc(a0 + kk * 32),
                         mn_desc<NS>(b0 + kk * 32 * NS), idesc_j, (kb | kk) != 0);
              }
            mma_commit(smem_u32(barC + p));
          }
        }
    }
  } else if (warp >= 4) {
    const int e = warp - 4, quarter = e & 3, mt = (e >> 2) & 1, half = e >> 3;
    const int m = mt * 128 + quarter * 32 + lane;
    const bool active = mt < nt;
    const uint32_t lanebase = tmem + ((uint32_t)(quarter * 32) << 16);
    const size_t P = (size_t)fa.P;
    constexpr int NCH = NS / 32;
    constexpr int PER = NCH >= 2 ? 2 : 1;
    for (int j = 0; j < npairs; ++j)
      for (int k = 0; k < Ld; ++k) {
        const bool carry = k + 1 < Ld;
        uint4 b1[2][NCH];
        // y_k of both blocks
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          if (!has(j, p)) continue;
          const int n0 = blk(j, p) * NS + half * (NS / 2);
          if (carry && active) {
            const int8_t* src = fa.Bg + ((size_t)(k + 1) * fa.nLp + m) * P + n0;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
              b1[p][ch] =
                  n0 + ch * 16 < fa.N ? __ldcg(reinterpret_cast<const uint4*>(src + ch * 16)) : make_uint4(0, 0, 0, 0);
          }
          mbar_wait(smem_u32(barD + p), (uint32_t)((j * Ld + k) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (active) {
            int8_t* yg = fa.Y + ((size_t)k * fa.nLp + m) * P + n0;
#pragma unroll
            for (int hh = 0; hh < NCH / PER; ++hh) {
              int v[32];
              if constexpr (PER == 2)
                tmem_ld32(lanebase + (uint32_t)(128 * p + mt * NS + half * (NS / 2) + hh * 32), v);
              else
                tmem_ld16(lanebase + (uint32_t)(128 * p + mt * NS + half * (NS / 2) + hh * 16), v);
#pragma unroll
              for (int c2 = 0; c2 < PER; ++c2) {
                const int ch = hh * PER + c2;
                uint32_t w4[4];
                digits16(fa.fq, fa.fast, v + c2 * 16, w4);
                const uint4 y4 = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                if (carry) *reinterpret_cast<uint4*>(sY[p] + swz<NS>(m, half * (NS / 2) + ch * 16)) = y4;
                if (m < fa.nL && n0 + ch * 16 < fa.N) *reinterpret_cast<uint4*>(yg + ch * 16) = y4;
              }
            }
          }
          fence_async_smem();
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(barY + p));
        }
        if (!carry) continue;
        // in_{k+1}, h_{k+1} of both blocks
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          if (!has(j, p)) continue;
          if (k == 0) mbar_wait(smem_u32(barB0 + p), (uint32_t)(j & 1));  // b_0 (TMA) is r_0
          mbar_wait(smem_u32(barC + p), (uint32_t)((j * (Ld - 1) + k) & 1));
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (active) {
#pragma unroll
            for (int hh = 0; hh < NCH / PER; ++hh) {
              int v[32];
              if constexpr (PER == 2)
                tmem_ld32(lanebase + (uint32_t)(256 + 128 * p + mt * NS + half * (NS / 2) + hh * 32), v);
              else
                tmem_ld16(lanebase + (uint32_t)(256 + 128 * p + mt * NS + half * (NS / 2) + hh * 16), v);
#pragma unroll
              for (int c2 = 0; c2 < PER; ++c2) {
                const int ch = hh * PER + c2;
                const uint32_t off = swz<NS>(m, half * (NS / 2) + ch * 16);
                const uint4 lo = *reinterpret_cast<const uint4*>(sIn[p] + off);
                const uint4 hi = k ? *reinterpret_cast<const uint4*>(sH[p] + off) : make_uint4(0, 0, 0, 0);
                const uint32_t low[4] = {lo.x, lo.y, lo.z, lo.w};
                const uint32_t hiw[4] = {hi.x, hi.y, hi.z, hi.w};
                const uint32_t b1w[4] = {b1[p][ch].x, b1[p][ch].y, b1[p][ch].z, b1[p][ch].w};
                uint32_t in4[4], h4[4];
                carry16(fa.fq, fa.fast, k != 0, low, hiw, b1w, v + c2 * 16, in4, h4);
                *reinterpret_cast<uint4*>(sIn[p] + off) = make_uint4(in4[0], in4[1], in4[2], in4[3]);
                *reinterpret_cast<uint4*>(sH[p] + off) = make_uint4(h4[0], h4[1], h4[2], h4[3]);
              }
            }
          }
          fence_async_smem();
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(barIn + p));
        }
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace tc

namespace {
// Per-device launch facts.  The SM count and the >48 KB dynamic shared-memory
// opt-in are properties of (device, kernel): a process that launches on a
// second device must opt in there too.
constexpr int kMaxDev = 64;
int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
int sm_count() {
  static std::atomic<int> sms[kMaxDev];
  const int d = cur_device();
  DRZG_REQUIRE(d >= 0 && d < kMaxDev, "tc_gemm: device index out of range");
  int v = sms[d].load(std::memory_order_relaxed);
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    sms[d].store(v, std::memory_order_relaxed);
  }
  return v;
}
template <class K>
void smem_opt_in(K* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes opted in
  const int d = cur_device();
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{reinterpret_cast<const void*>(kernel), d}];
  if (have >= bytes) return;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  DRZG_REQUIRE(e == cudaSuccess, std::string("shared-memory opt-in: ") + cudaGetErrorString(e));
  have = bytes;
}
}  // namespace

namespace {
// The dataflow kernels spin on counters other clusters publish, so each needs
// all its clusters resident at once.  Two in flight on one device (engines on
// several host threads, each with its own stream) could each hold SMs the
// other's clusters wait for.  Their launches are therefore chained per device
// through an event: at most one dataflow kernel runs at a time, while every
// other kernel of every stream overlaps freely.  (Splitting the device
// between concurrent dataflow kernels instead, each on a quarter of the
// clusters, made the 64-threefold batch slower: 32.8 s against 16.7 s.)
template <class F>
void gated_flow_launch(cudaStream_t st, F&& launch) {
  struct Gate {
    std::mutex mu;
    cudaEvent_t last = nullptr;
  };
  static Gate gates[kMaxDev];
  const int d = cur_device();
  DRZG_REQUIRE(d >= 0 && d < kMaxDev, "dixon_flow: device index out of range");
  Gate& g = gates[d];
  std::lock_guard<std::mutex> lk(g.mu);
  cudaError_t e = cudaSuccess;
  if (!g.last)
    e = cudaEventCreateWithFlags(&g.last, cudaEventDisableTiming);
  else
    e = cudaStreamWaitEvent(st, g.last, 0);
  DRZG_REQUIRE(e == cudaSuccess, std::string("dixon_flow gate: ") + cudaGetErrorString(e));
  launch();
  e = cudaEventRecord(g.last, st);
  DRZG_REQUIRE(e == cudaSuccess, std::string("dixon_flow gate: ") + cudaGetErrorString(e));
}

// grid rounds of tiles per phase of a column group: a tile's dependencies
// (the previous phase of its column) were issued this many rounds earlier
int flow_rounds() {
  static const int r = [] {
    const char* e = std::getenv("DRZG_FLOW_ROUNDS");
    const int v = e ? std::atoi(e) : 0;
    return v >= 1 && v <= 64 ? v : 2;
  }();
  return r;
}
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  DRZG_REQUIRE(fn != nullptr, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map(const int8_t* ptr, int rows, int ld, int K, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DRZG_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}
}  // namespace

void tc_gemm_i8(const int8_t* A, int rowsA, int lda, const int8_t* B, int rowsB, int ldb, int K,
                const TcEpiArgs& epi, cudaStream_t st) {
  DRZG_REQUIRE(lda % 16 == 0 && ldb % 16 == 0, "tc_gemm: row pitch must be a multiple of 16 bytes");
  DRZG_REQUIRE(((uintptr_t)A & 15) == 0 && ((uintptr_t)B & 15) == 0, "tc_gemm: operands must be 16-byte aligned");
  CUtensorMap ma = make_map(A, rowsA, lda, K, tc::BM);
  CUtensorMap mb = epi.b_mn ? make_map(B, K, ldb, ldb, tc::BK)  // K rows x ldb states, box 128 x 128
                            : make_map(B, rowsB, ldb, K, tc::BN);
  // kind::i8 instruction descriptor: D s32, A signed (Cq) or unsigned (Jp),
  // B signed, both K-major, N = BN, M = 128
  uint32_t a_signed = epi.a_unsigned ? 0u : 1u;
  uint32_t idesc = (2u << 4) | (a_signed << 7) | (1u << 10) | ((uint32_t)(epi.b_mn ? 1u : 0u) << 16) |
                   ((uint32_t)(tc::BN >> 3) << 17) |
                   ((uint32_t)(tc::BM >> 4) << 24);
  smem_opt_in(tc::gemm_kernel, tc::SMEM_BYTES);
  const int sms = sm_count();
  int tiles = ((epi.N + tc::BN - 1) / tc::BN) * ((epi.M + tc::BM - 1) / tc::BM);
  dim3 grid(std::min(tiles, sms));
  tc::gemm_kernel<<<grid, tc::THREADS, tc::SMEM_BYTES, st>>>(ma, mb, K, idesc, epi);
  cudaError_t e = cudaGetLastError();
  DRZG_REQUIRE(e == cudaSuccess, std::string("tc_gemm launch: ") + cudaGetErrorString(e));
}




namespace {
CUtensorMap make_map_box(const int8_t* ptr, int rows, int ld, int inner, int box_inner, int box_rows,
                         CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DRZG_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// Tensor maps of the one-launch solve, kept per launching thread: a map is a
// pure function of (address, dims, pitch), and re-encoding three of them for
// every ~40 us launch put the launcher behind the device on small batches
struct MapCache {
  const void* p = nullptr;
  int a = -1, b = -1;
  CUtensorMap m;
};
template <class F>
const CUtensorMap& cached_map(MapCache& c, const void* p, int a, int b, F make) {
  if (c.p != p || c.a != a || c.b != b) {
    c.m = make();
    c.p = p;
    c.a = a;
    c.b = b;
  }
  return c.m;
}

template <int NS>
void launch_fused_pp(const CUtensorMap& mc, const CUtensorMap& mj, const FusedArgs& fa, int sms, cudaStream_t st) {
  const int nt = fa.nLp / 128;
  thread_local MapCache bcache;
  const CUtensorMap& mb = cached_map(bcache, fa.Bg, fa.nLp, fa.P, [&] {
    return make_map_box(fa.Bg, fa.nLp, fa.P, fa.P, NS, 128,
                        NS == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  });
  const uint32_t common = (2u << 4) | (1u << 10) | (1u << 16) | ((uint32_t)(NS >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t idesc_c = common | (1u << 7), idesc_j = common;
  const int smem = tc::fz::smem_bytes_pp(nt, NS);
  smem_opt_in(tc::dixon_fused_pp_kernel<NS>, smem);
  const int nblk = (fa.N + NS - 1) / NS;
  tc::dixon_fused_pp_kernel<NS><<<std::min(nblk, sms), tc::fz::THREADS, smem, st>>>(mc, mj, mb, idesc_c, idesc_j, fa);
}

template <int NS>
void launch_fused(const CUtensorMap& mc, const CUtensorMap& mj, const FusedArgs& fa, int sms, cudaStream_t st) {
  const int nt = fa.nLp / 128;
  thread_local MapCache bcache;
  const CUtensorMap& mb = cached_map(bcache, fa.Bg, fa.nLp, fa.P, [&] {
    return make_map_box(fa.Bg, fa.nLp, fa.P, fa.P, NS, 128,
                        NS == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                        : NS == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                   : CU_TENSOR_MAP_SWIZZLE_32B);
  });
  // kind::i8, D s32, B signed MN-major, N = NS, M = 128; A signed (Cq) / unsigned (Jp)
  const uint32_t common = (2u << 4) | (1u << 10) | (1u << 16) | ((uint32_t)(NS >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t idesc_c = common | (1u << 7), idesc_j = common;
  const int smem = tc::fz::smem_bytes(nt, NS) + (fa.chunk ? fa.Ld * fa.nLp * NS : 0);
  smem_opt_in(tc::dixon_fused_kernel<NS>, smem);
  const int nblk = (fa.N + NS - 1) / NS;
  static const bool one_block = std::getenv("DRZG_FUSED_ONEBLOCK") != nullptr;  // debug: one block per CTA
  tc::dixon_fused_kernel<NS><<<one_block ? nblk : std::min(nblk, sms), tc::fz::THREADS, smem, st>>>(
      mc, mj, mb, idesc_c, idesc_j, fa);
}
}  // namespace

bool dixon_fused_ok(int nLp) { return nLp % 128 == 0 && nLp <= 256; }
// whole-chunk launches keep the block's Ld y planes in shared memory too
bool dixon_chunk_ok(int nLp, int Ld) { return dixon_fused_ok(nLp) && tc::fz::smem_bytes(nLp / 128, 32) + Ld * nLp * 32 <= 227 * 1024; }

void dixon_fused(const int8_t* C, const int8_t* Jd, const FusedArgs& fa, cudaStream_t st) {
  DRZG_REQUIRE(dixon_fused_ok(fa.nLp), "dixon_fused: system order must be 128 or 256");
  DRZG_REQUIRE(fa.P % 64 == 0, "dixon_fused: state pitch must be a multiple of 64");
  thread_local MapCache ccache, jcache;
  const CUtensorMap& mc = cached_map(ccache, C, fa.nLp, 0, [&] { return make_map(C, fa.nLp, fa.nLp, fa.nLp, 128); });
  const CUtensorMap& mj = cached_map(jcache, Jd, fa.nLp, 0, [&] { return make_map(Jd, fa.nLp, fa.nLp, fa.nLp, 128); });
  const int sms = sm_count();
  // small batches (fewer 128-state blocks than SMs) run 64-state blocks
  const char* ns_env = std::getenv("DRZG_FUSED_NS");  // per launch: the path tests switch it
  // (32-state blocks when the whole batch fits one round of them: the
  // per-digit epilogue phases halve, which is what a small batch waits on)
  // (large batches: 64-state blocks beat 128 too, 82 vs 86 ms of fused time
  // per K3 zeta function -- the per-digit epilogue phase is what a block
  // waits on, and it halves; DRZG_FUSED_NS=128 keeps the 128-state variant)
  const int ns = fa.chunk ? 32 : ns_env ? std::atoi(ns_env) : (fa.N <= 32 * sms ? 32 : 64);
  // two 64-state blocks in flight per CTA once every CTA has two or more
  // (DRZG_FUSED_PP=0 keeps one block per CTA)
  const char* pp_env = std::getenv("DRZG_FUSED_PP");  // per launch: the path tests switch it
  const bool pp_on = !(pp_env && std::string(pp_env) == "0");
  if (pp_on && !fa.chunk && !ns_env && fa.N >= 2 * 64 * sms &&
      tc::fz::smem_bytes_pp(fa.nLp / 128, 64) <= 227 * 1024) {
    launch_fused_pp<64>(mc, mj, fa, sms, st);
  } else if (ns == 32)
    launch_fused<32>(mc, mj, fa, sms, st);
  else if (ns == 64)
    launch_fused<64>(mc, mj, fa, sms, st);
  else
    launch_fused<128>(mc, mj, fa, sms, st);
  cudaError_t e = cudaGetLastError();
  DRZG_REQUIRE(e == cudaSuccess, std::string("dixon_fused launch: ") + cudaGetErrorString(e));
}

void dixon_flow(const int8_t* C, const int8_t* Jd, FlowArgs fa, cudaStream_t st) {
  TcEpiArgs& e = fa.epi;
  DRZG_REQUIRE(e.kb_ptr && e.kb_idx, "dixon_flow: the carry needs its K-block lists");
  DRZG_REQUIRE(e.nLp % tc::BK == 0 && e.P % 64 == 0, "dixon_flow: system order / pitch alignment");
  e.b_mn = 1;
  fa.ncol = (e.N + tc::BN - 1) / tc::BN;
  CUtensorMap mc = make_map(C, e.nLp, e.nLp, e.nLp, tc::BM);
  CUtensorMap mj = make_map(Jd, e.nLp, e.nLp, e.nLp, tc::BM);
  // MN-major B operands: K rows x P states, box 128 states x 128 rows
  CUtensorMap mb0 = make_map(e.Bg, e.nLp, e.P, e.P, tc::BK);             // b_0 = in_0
  CUtensorMap min_ = make_map(e.IN, e.nLp, e.P, e.P, tc::BK);            // in_k
  CUtensorMap my = make_map(e.Y, e.Ld * e.nLp, e.P, e.P, tc::BK);        // y_k at row k * nLp
  const uint32_t common = (2u << 4) | (1u << 10) | (1u << 16) | ((uint32_t)(tc::BN >> 3) << 17) |
                          ((uint32_t)(tc::BM >> 4) << 24);
  fa.idesc_d = common | (1u << 7);  // Cq signed
  fa.idesc_c = common;              // Jp unsigned
  smem_opt_in(tc::dixon_flow_kernel, tc::SMEM_BYTES);
  const int sms = sm_count();
  const int mt = (e.M + tc::BM - 1) / tc::BM;
  const int nph = 2 * e.Ld - 1;
  // columns per group: enough tiles per phase (~2 rounds of the grid) that a
  // tile's dependencies were issued a round earlier
  fa.G = std::max(1, std::min(fa.ncol, (flow_rounds() * sms + mt - 1) / mt));
  {
    cudaError_t me = cudaMemsetAsync(fa.counters, 0, sizeof(int) * (size_t)nph * fa.ncol, st);
    DRZG_REQUIRE(me == cudaSuccess, std::string("dixon_flow counters: ") + cudaGetErrorString(me));
  }
  const int tiles = nph * fa.ncol * mt;
  gated_flow_launch(st, [&] {
    tc::dixon_flow_kernel<<<std::min(tiles, sms), tc::THREADS, tc::SMEM_BYTES, st>>>(mc, mj, mb0, min_, my, fa);
  });
  cudaError_t err = cudaGetLastError();
  DRZG_REQUIRE(err == cudaSuccess, std::string("dixon_flow launch: ") + cudaGetErrorString(err));
}


void dixon_flow2(const int8_t* C, const int8_t* Jd, FlowArgs fa, cudaStream_t st) {
  TcEpiArgs& e = fa.epi;
  DRZG_REQUIRE(fa.kb2_ptr && fa.kb2_idx, "dixon_flow2: the carry needs its pair K-block lists");
  DRZG_REQUIRE(e.nLp % tc::BK == 0 && e.P % 64 == 0, "dixon_flow2: system order / pitch alignment");
  e.b_mn = 1;
  fa.ncol = (e.N + tc::BN - 1) / tc::BN;
  CUtensorMap mc = make_map(C, e.nLp, e.nLp, e.nLp, tc::BM);
  CUtensorMap mj = make_map(Jd, e.nLp, e.nLp, e.nLp, tc::BM);
  CUtensorMap mb0 = make_map(e.Bg, e.nLp, e.P, e.P, tc::BK);
  CUtensorMap min_ = make_map(e.IN, e.nLp, e.P, e.P, tc::BK);
  CUtensorMap my = make_map(e.Y, e.Ld * e.nLp, e.P, e.P, tc::BK);
  // kind::i8, D s32, B signed MN-major, N = 256, M = 256 (the pair)
  const uint32_t common = (2u << 4) | (1u << 10) | (1u << 16) | ((uint32_t)(tc::BN >> 3) << 17) |
                          ((uint32_t)((2 * tc::BM) >> 4) << 24);
  fa.idesc_d = common | (1u << 7);  // Cq signed
  fa.idesc_c = common;              // Jp unsigned
  smem_opt_in(tc::dixon_flow2_kernel, tc::f2::SMEM_BYTES);
  static const int dbg = [] {
    const char* e = std::getenv("DRZG_FLOW_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  fa.debug = dbg;
  const int mt = (e.M + tc::BM - 1) / tc::BM, mt2 = (mt + 1) / 2;
  const int nph = 2 * e.Ld - 1;
  // every cluster must be resident at once (tiles wait on other clusters'
  // counters): the grid is the number of co-resident pairs
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(tc::f2::THREADS);
  cfg.dynamicSmemBytes = tc::f2::SMEM_BYTES;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static thread_local int max_clusters[64] = {0};
  const int dev = cur_device();
  if (!max_clusters[dev]) {
    cfg.gridDim = dim3(2 * (sm_count() / 2));
    int nc = 0;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&nc, tc::dixon_flow2_kernel, &cfg);
    DRZG_REQUIRE(oe == cudaSuccess && nc > 0, std::string("dixon_flow2 occupancy: ") + cudaGetErrorString(oe));
    max_clusters[dev] = nc;
  }
  // one round = one phase of a G-column group = one tile per cluster
  fa.G = std::max(1, max_clusters[dev] / mt2);
  fa.ngroups = (fa.ncol + fa.G - 1) / fa.G;
  fa.streams = std::min(3, fa.ngroups);
  {
    int rounds = 0;
    for (int st = 0; st < fa.streams; ++st) {
      const int groups = (fa.ngroups - st + fa.streams - 1) / fa.streams;
      rounds = std::max(rounds, fa.streams * (groups * nph + st));
    }
    fa.rounds = rounds;
  }
  {
    cudaError_t me = cudaMemsetAsync(fa.counters, 0, sizeof(int) * (size_t)nph * fa.ncol, st);
    DRZG_REQUIRE(me == cudaSuccess, std::string("dixon_flow2 counters: ") + cudaGetErrorString(me));
  }
  cfg.gridDim = dim3(2 * std::min(fa.G, fa.ncol) * mt2);
  cudaError_t err = cudaSuccess;
  gated_flow_launch(st, [&] { err = cudaLaunchKernelEx(&cfg, tc::dixon_flow2_kernel, mc, mj, mb0, min_, my, fa); });
  DRZG_REQUIRE(err == cudaSuccess, std::string("dixon_flow2 launch: ") + cudaGetErrorString(err));
  err = cudaGetLastError();
  DRZG_REQUIRE(err == cudaSuccess, std::string("dixon_flow2 launch: ") + cudaGetErrorString(err));
}

}  // namespace drzg
