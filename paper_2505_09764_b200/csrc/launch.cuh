// launch.cuh -- kernel launches with optional programmatic dependent launch
// (PDL) and the internal (non-exported) synthesis entry used by the
// alltoallv call chain.
//
// On the per-call chain gather -> balance -> decompose [-> sort] -> plan ->
// exec every kernel triggers its dependents as soon as it starts
// (griddepcontrol.launch_dependents) and waits for its predecessor's memory
// before touching it (griddepcontrol.wait), so each launch and CTA
// rasterisation overlaps the previous kernel instead of following it.  Both
// instructions are no-ops for a kernel launched without the PDL attribute
// (the batched synthesis path).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "fastb200.h"

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// fast_synth_batch for the alltoallv chain (synth.cu): pdl = launch every
// kernel with the PDL attribute; the caller has zeroed out->status already
// (a memset node would break the programmatic chain).
int fast_synth_batch_chain(const int64_t* D, int B, int n, int m, const fast_sched_bufs* out,
                           cudaStream_t s, bool pdl);
