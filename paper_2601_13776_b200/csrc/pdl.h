// Host side of programmatic dependent launch (see umma.cuh griddep_*): launch a
// kernel with cudaLaunchAttributeProgrammaticStreamSerialization so that its CTAs
// may be scheduled while the previous kernel on the stream drains (its prologue
// -- barrier init, TMEM allocation, descriptor prefetch -- overlaps that tail).
// The kernel must call umma::griddep_wait() before touching global memory.
// ORTH_NO_PDL=1 launches without the attribute (A/B switch).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace orth {

inline bool pdl_enabled() {
  static const bool on = std::getenv("ORTH_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace orth
