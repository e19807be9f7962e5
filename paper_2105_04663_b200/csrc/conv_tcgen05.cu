// Placeholder for the NHWC bf16 implicit-GEMM convolution on tcgen05; until it
// lands every convolution takes the direct kernel in contract.cu.
#include "common.cuh"

namespace spmd {

int conv_tcgen05(const spmd_tensor&, const spmd_tensor&, const spmd_tensor&,
                 const spmd_conv_dims&, int64_t, cudaStream_t) {
  return SPMD_ERR_UNSUPPORTED;
}

}  // namespace spmd
