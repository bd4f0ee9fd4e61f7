// K1 tensor-core path (tcgen05 / TMA / TMEM, 3xTF32) — placeholder until the kernel lands.
#include "omp_internal.cuh"

namespace ompb {
cudaError_t launch_corr_tc(const Planes&, const Planes&, int64_t, float*, int64_t, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace ompb
