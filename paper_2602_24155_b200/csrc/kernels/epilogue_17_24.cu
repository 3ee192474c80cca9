// T_x epilogue instantiations for 17 <= Ld <= 24 (see dixon.cuh)
#define DRZG_EPILOGUE_ONLY
#include "dixon.cuh"

namespace drzg {
namespace dev {
void launch_epilogue_17_24(const StepArgs& a, dim3 grid, cudaStream_t st) {
  switch (a.Ld) {
    DRZG_EPI_CASE(17) DRZG_EPI_CASE(18) DRZG_EPI_CASE(19) DRZG_EPI_CASE(20) DRZG_EPI_CASE(21) DRZG_EPI_CASE(22) DRZG_EPI_CASE(23) DRZG_EPI_CASE(24)
    default:
      break;
  }
}
}  // namespace dev
}  // namespace drzg
