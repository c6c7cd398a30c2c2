// launch_util.h -- host-side launch helpers shared by the kernel files.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace fc {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the current
// device's context: remember what was set per device (a process may drive
// several GPUs), setting it again only when a launch needs more.
inline cudaError_t set_smem_attr(const void* kern, int bytes, int* cache /* [64], zero-initialised */) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cache[dev] = bytes;
  return e;
}

// Programmatic dependent launch: kernels that call griddep_wait() before
// their first read of data an earlier kernel produced (and griddep_launch()
// once that wait has returned) are launched with the programmatic stream
// serialization attribute, so their prologue (launch, shared-memory tables,
// barriers, TMEM allocation) overlaps the tail of the previous kernel in the
// stream.  FFTCONV_PDL=0 launches them normally (A/B switch).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FFTCONV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace fc
