// Kernel launch with programmatic dependent launch (PDL): the launch carries
// cudaLaunchAttributeProgrammaticStreamSerialization, so inside the iteration
// graph consecutive kernels get programmatic edges and the next kernel's CTAs
// are scheduled while the previous one drains (each kernel starts with
// griddep_wait()).
#pragma once
#include <cuda_runtime.h>
#include <stdlib.h>

#include <utility>

namespace cb {

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace cb
