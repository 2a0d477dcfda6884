// K3 (tcgen05 variant) -- placeholder until the TMA/tcgen05/TMEM kernel lands.
#include "rsa_internal.cuh"

namespace rsa {

bool tc_supported(const Geometry&) { return false; }

cudaError_t launch_attn_tc(const Geometry&, const void*, const void*, const void*, void*, float*,
                           const Workspace&, bool, bool, cudaStream_t, int*) {
  return cudaErrorNotSupported;
}

}  // namespace rsa
