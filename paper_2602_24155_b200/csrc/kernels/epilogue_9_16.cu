// T_x epilogue instantiations for 9 <= Ld <= 16 (see dixon.cuh)
#define DRZG_EPILOGUE_ONLY
#include "dixon.cuh"

namespace drzg {
namespace dev {
void launch_epilogue_9_16(const StepArgs& a, dim3 grid, cudaStream_t st) {
  switch (a.Ld) {
    DRZG_EPI_CASE(9) DRZG_EPI_CASE(10) DRZG_EPI_CASE(11) DRZG_EPI_CASE(12) DRZG_EPI_CASE(13) DRZG_EPI_CASE(14) DRZG_EPI_CASE(15) DRZG_EPI_CASE(16)
    default:
      break;
  }
}
}  // namespace dev
}  // namespace drzg
