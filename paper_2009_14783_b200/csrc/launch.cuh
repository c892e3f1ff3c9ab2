// Kernel launch through cudaLaunchKernelEx with an optional thread-block
// cluster dimension (the CTA-pair tcgen05 GEMM and the bulk-copy kernels
// share this one helper).
#pragma once

#include <cuda_runtime.h>

#include "hp_common.h"

namespace hp {

template <typename... KArgs, typename... Args>
inline void launch_ex(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                      int cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  unsigned n = 0;
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  HP_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}

}  // namespace hp
