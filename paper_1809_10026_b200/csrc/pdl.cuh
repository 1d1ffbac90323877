// Programmatic dependent launch (PDL) helpers shared by the kernel headers.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace ls {

// Programmatic dependent launch: the kernels of the hot path are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a launch can start while the
// previous kernel of the stream drains; everything before pdl_wait() (staging the constant
// W = U^T / U and lambda into shared memory) overlaps that tail.  pdl_wait() returns once
// the previous grid has completed and its writes are visible; no global store and no load
// of the previous kernel's output happens before it.  Without the attribute it is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// process-wide switch (ls_tune LS_TUNE_PDL), default on
extern int g_ls_pdl;

template <typename... Params, typename... Args>
static inline cudaError_t launch_pdl(void (*k)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_ls_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

}  // namespace ls
