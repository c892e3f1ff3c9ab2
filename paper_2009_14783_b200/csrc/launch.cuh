// Kernel launch with programmatic dependent launch (PDL).
//
// The step is a chain of ~200 dependent kernels on one stream (GEMM ->
// attention -> GEMM -> LayerNorm -> ...), most of them a few microseconds
// long, so the launch latency and prologue (barrier init, TMEM allocation,
// tensor-map prefetch) of each one is a visible share of the step.  Kernels
// launched through launch_pdl may be scheduled while their predecessor on the
// stream is still running; each such kernel executes pdl_wait() (PTX
// griddepcontrol.wait: every prerequisite grid has completed and its memory
// is visible) before it touches global memory a predecessor may write or
// read, and pdl_trigger() (griddepcontrol.launch_dependents) right after, so
// at most one kernel runs ahead of the chain.  Kernels launched without the
// attribute behave as before; pdl_wait() is a no-op for them.
// Opt-in (HP_PDL=1, or a class list "gemm,attn,ln"): on the C2 step every
// variant measured within noise or slower than plain launches (the early
// CTAs take SM slots from the concurrent weight-gradient / update streams),
// so the default is off.
#pragma once

#include <cuda_runtime.h>

#include "hp_common.h"

namespace hp {

// kernel classes for HP_PDL ("1" all, "0" none, or a list "gemm,attn,ln")
enum PdlClass { PDL_GEMM = 0, PDL_ATTN = 1, PDL_LN = 2 };
bool pdl_on(int cls);  // kernels.cu

template <typename... KArgs, typename... Args>
inline void launch_pdl(int cls, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, int cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_on(cls)) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  HP_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
#ifndef HP_PDL_NO_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

}  // namespace hp
