#include "common.cuh"
namespace svg {
int launch_attend_tc(const SvgEarShape&, const bf16*, const bf16*, const bf16*, const int32_t*,
                     const int32_t*, const int32_t*, const uint8_t*, bf16*, float*, AttendScratch&,
                     cudaStream_t) {
  return SVGEAR_EUNSUPPORTED;
}
}  // namespace svg
