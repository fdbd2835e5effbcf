// tcgen05 split-TF32 GEMMs — placeholder until the tensor-core kernels land.
#include "kernels.cuh"

namespace lpca {

bool tc_xw_supported(index_t, index_t) { return false; }
bool tc_utx_supported(index_t, index_t) { return false; }
void launch_xw_tc(cudaStream_t, const float*, index_t, index_t, index_t, const float*, const float*,
                  index_t, index_t, float*, index_t, int) {
  throw Error(kInternal, "tcgen05 path not built");
}
void launch_utx_tc(cudaStream_t, const float*, index_t, const float*, index_t, index_t, index_t,
                   index_t, index_t, double*, int) {
  throw Error(kInternal, "tcgen05 path not built");
}

}  // namespace lpca
