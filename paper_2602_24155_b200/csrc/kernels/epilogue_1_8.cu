// T_x epilogue instantiations for 1 <= Ld <= 8 (see dixon.cuh)
#define DRZG_EPILOGUE_ONLY
#include "dixon.cuh"

namespace drzg {
namespace dev {
void launch_epilogue_1_8(const StepArgs& a, dim3 grid, cudaStream_t st) {
  switch (a.Ld) {
    DRZG_EPI_CASE(1) DRZG_EPI_CASE(2) DRZG_EPI_CASE(3) DRZG_EPI_CASE(4) DRZG_EPI_CASE(5) DRZG_EPI_CASE(6) DRZG_EPI_CASE(7) DRZG_EPI_CASE(8)
    default:
      break;
  }
}
}  // namespace dev
}  // namespace drzg
