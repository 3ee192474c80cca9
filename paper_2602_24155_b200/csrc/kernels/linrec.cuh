// Reference-shaped recurrence kernels: host-side launch interface.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace drzg {

struct LinrecPlan {
  uint64_t p = 0;
  int M = 0, limbs = 1, limb_exp = 0;
  uint64_t beta = 0;     // p^limb_exp
  uint64_t top_mod = 0;  // p^(M - limb_exp*(limbs-1)): modulus of the top digit
};

struct CsrPair {
  const int* a_ptr;
  const int* a_col;
  const uint64_t* a_val;
  const int* b_ptr;
  const int* b_col;
  const uint64_t* b_val;
};

// w <- M(0)...M(tmax) w on device buffers (reference linalg.hpp:337-410);
// csr != nullptr selects the sparse kernel (reference linalg.hpp:257-331)
void linrec_device(const LinrecPlan& pl, int side, const uint64_t* dA, const uint64_t* dB, int64_t tmax,
                   uint64_t* dw, cudaStream_t st, float* kernel_ms, const CsrPair* csr);

}  // namespace drzg
