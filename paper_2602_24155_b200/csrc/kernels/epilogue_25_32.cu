// T_x epilogue instantiations for 25 <= Ld <= 32 (see dixon.cuh)
#define DRZG_EPILOGUE_ONLY
#include "dixon.cuh"

namespace drzg {
namespace dev {
void launch_epilogue_25_32(const StepArgs& a, dim3 grid, cudaStream_t st) {
  switch (a.Ld) {
    DRZG_EPI_CASE(25) DRZG_EPI_CASE(26) DRZG_EPI_CASE(27) DRZG_EPI_CASE(28) DRZG_EPI_CASE(29) DRZG_EPI_CASE(30) DRZG_EPI_CASE(31) DRZG_EPI_CASE(32)
    default:
      break;
  }
}
}  // namespace dev
}  // namespace drzg
