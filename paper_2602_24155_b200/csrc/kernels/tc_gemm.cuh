// int8 tcgen05 GEMM with Dixon epilogues (sm_100a).
//
//   D[m][n] = sum_k A[m][k] * B[n][k]      (A: M x K, B: N x K, both K-major int8)
//
// 128 x BN CTA tile, K staged 128 bytes at a time through a 4-deep
// TMA -> shared-memory (128B-swizzled) ring; one elected thread issues
// tcgen05.mma.kind::i8 (M=128, N=BN, K=32) into a TMEM int32 accumulator;
// four epilogue warps drain TMEM with tcgen05.ld and apply the Dixon step's
// elementwise epilogue in registers:
//   EPI_DIGIT  y_k = bal(D mod q) -> int8 Y plane          (D = Cq . in_k)
//   EPI_CARRY  c = (r_k - D) / q, r_{k+1} = b_{k+1} + c -> in_{k+1} = bal(r_{k+1}), h_{k+1}
//              with r_k = b_0 (k = 0) or in_k + q h_k                  (D = Jp . y_k)
//   EPI_RAW    D as int32 (tests)
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastq.cuh"

namespace drzg {

enum class TcEpilogue : int { raw = 0, digit = 1, carry = 2 };

struct TcEpiArgs {
  int mode = 0;
  int a_unsigned = 0;      // A operand u8 (else s8)
  int b_mn = 0;            // B stored K x N (states contiguous, "MN-major"); else N x K
  int P = 0;               // b_mn: state pitch of every per-state array (elements)
  int M = 0, N = 0;        // valid output extent
  int q = 0, Ld = 0, k = 0;
  FastQ fq;
  int fast = 0;            // every epilogue operand is below 2^23 in magnitude (host-checked)
  int nLp = 0, nL = 0;
  // raw
  int32_t* out = nullptr;  // N x M (row n holds the M outputs of column n)
  // digit
  int8_t* Y = nullptr;     // N x Ld x nLp
  // carry
  const int8_t* Bg = nullptr;  // Ld x nLp x P gathered digits b_t
  int8_t* H = nullptr;         // nLp x P: high part of the running residual r = in + q h
  int8_t* IN = nullptr;        // nLp x P: in_k (read by carry k > 0, overwritten with in_{k+1})
  // block-sparse A (carry): M tile i runs over K blocks kb_idx[kb_ptr[i] ..
  // kb_ptr[i+1]) (128-wide) only; null = dense
  const int* kb_ptr = nullptr;
  const int* kb_idx = nullptr;
};

// host side: build tensor maps and launch; A is (rowsA x K) with row pitch
// lda bytes; B is (rowsB x K) with row pitch ldb bytes, or with epi.b_mn a
// K x ldb matrix (row pitch ldb bytes, N = epi.N valid columns)
void tc_gemm_i8(const int8_t* A, int rowsA, int lda, const int8_t* B, int rowsB, int ldb, int K,
                const TcEpiArgs& epi, cudaStream_t st);



// whole Dixon solve of every state of a batch in one launch, for systems of
// order nLp in {128, 256}: Cq, Jp resident in shared memory, one CTA per
// 128-state block (see dixon_fused_kernel)
struct FusedArgs {
  int nL = 0, nLp = 0, N = 0, P = 0, Ld = 0, q = 0;
  FastQ fq;
  int fast = 0;
  const int8_t* Bg = nullptr;  // Ld x nLp x P gathered digits (plane 0 is read through TMA)
  int8_t* Y = nullptr;         // Ld x nLp x P: y_k out
  long long* trace = nullptr;  // debug: %globaltimer stamps of CTA 0's first epilogue thread
  // chunk mode: every step of each state's chunk in this launch.  After a
  // block's Dixon solve the CTA applies T_x itself (w' = T_x y, reduction
  // step epilogue) and writes the next step's operand Bg (through ginv) or,
  // at the state's last step, W; the block's next step then reloads b_0.
  // States are sorted by k descending, so a block runs k of its first state.
  int chunk = 0;
  const int64_t* ks = nullptr;  // N: chunk length of each state
  const int* vdir = nullptr;    // N
  const int* u0 = nullptr;      // N x nv (exponent at the chunk start)
  const int* dirs = nullptr;    // ndir x nv
  const int *t_ptr = nullptr, *t_src = nullptr, *sol_i = nullptr, *sol_mu = nullptr, *ginv = nullptr;
  int8_t* W = nullptr;          // Ld x sidep x P
  int side = 0, sidep = 0, nv = 0;
};
bool dixon_fused_ok(int nLp);
bool dixon_chunk_ok(int nLp, int Ld);
void dixon_fused(const int8_t* C, const int8_t* Jd, const FusedArgs& fa, cudaStream_t st);


// whole Dixon solve of a batch in one persistent dataflow launch (nLp > 256,
// block-sparse carry): digit and carry tiles of all Ld digits, ordered by
// per-column phase counters (see dixon_flow_kernel)
struct FlowArgs {
  TcEpiArgs epi;             // M, N, P, q, fq, fast, Ld, nLp, nL, Bg, IN, H, Y, kb_ptr, kb_idx
  int ncol = 0, G = 0;       // 256-state columns, columns per group (set by dixon_flow)
  int* counters = nullptr;   // (2 Ld - 1) x ncol ints of device scratch
  uint32_t idesc_d = 0, idesc_c = 0;
  // CTA-pair variant: per 256-row tile, the union of its two 128-row tiles'
  // nonzero K blocks
  const int* kb2_ptr = nullptr;
  const int* kb2_idx = nullptr;
  int ngroups = 0, streams = 1, rounds = 0;  // the pair kernel's round schedule (set by dixon_flow2)
  int debug = 0;  // DRZG_FLOW_DEBUG (timing experiments only; results are wrong): 1 skip the
                  // epilogue arithmetic and memory, 2 also the TMEM loads
};
void dixon_flow(const int8_t* C, const int8_t* Jd, FlowArgs fa, cudaStream_t st);
// the same dataflow solve on CTA pairs (cta_group::2, M = 256 tiles)
void dixon_flow2(const int8_t* C, const int8_t* Jd, FlowArgs fa, cudaStream_t st);

}  // namespace drzg
