// Step arguments and layout constants shared by the engine and its kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "fastq.cuh"

namespace drzg {
namespace dev {

constexpr int kLdMax = 32;  // digit planes (register arrays)


struct StepArgs {
  // tables
  const int8_t* C;        // nLp x nLp (row-major), Jp^{-1} mod q
  const int* jp_ptr;      // nL + 1
  const int* jp_col;
  const int* jp_val;
  const int* gidx;        // ndir x nL
  const int* ginv;        // ndir x side (next step's row of each side row, or -1)
  const int64_t* ks;      // B: chunk length of each batch state
  const int* dirs;        // ndir x nv exponents of each v
  const int* t_ptr;       // side + 1
  const int* t_src;       // solution index feeding each side row
  const int* sol_i;       // per solution index: variable i of its generator
  const int* sol_mu;      // ... and mu_i
  int nv, nL, nLp, side, sidep, Ld, q;
  FastQ fq;
  int fast;               // fp32 reciprocal path valid (all operands < 2^23)
  // state pool
  int8_t* pool;           // slots x (Ld * sidep)
  long long slot_stride;  // Ld * sidep
  // batch
  const int* slot;        // B
  const int* vdir;        // B
  const int* u0;          // B x nv (exponent at sweep start)
  int y;                  // step index within the chunk: x = u0 - y v
  int B;
  int P;                  // state pitch of the temporaries (>= B, multiple of 64)
  int epi_rows = 64;      // side rows per T_x-epilogue block (<= kEpiRows; fewer for small batches)
  // temporaries, state-contiguous ("MN-major" GEMM operands)
  int8_t* Bg;             // Ld x nLp x P
  int8_t* IN;             // nLp x P
  int8_t* H;              // nLp x P: high part of the running residual r = in + q h
  int8_t* W;              // Ld x sidep x P: the state between steps of a chunk
  int8_t* Y;              // Ld x nLp x P
};

constexpr int kFlushRows = 64, kFlushStates = 32;

}  // namespace dev
}  // namespace drzg
