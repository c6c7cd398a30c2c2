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
// once that wait has returned) may be launched with the programmatic stream
// serialization attribute, so their prologue (launch, shared-memory tables,
// barriers, TMEM allocation) overlaps the tail of the previous kernel in the
// stream.  FFTCONV_PDL selects which launches use it (A/B switch):
// 0 none (default), 1 both, 2 the convolution only, 3 the k_f precompute
// only.  Measured on B200 (tools/pdl_probe.py, profiles/r02c/pdl_probe.txt):
// back-to-back convolutions gain 3 % (117.0 -> 113.2 us, cfg2 shape), but
// the k_f precompute -> convolution chain of a step loses 3-7 us at N = 1024
// with any of 1-3, so it is off.
enum PdlKernel { PDL_KF = 0, PDL_CONV = 1 };
inline bool pdl_enabled(PdlKernel k) {
  static const int mode = [] {
    const char* e = std::getenv("FFTCONV_PDL");
    return e ? std::atoi(e) : 0;
  }();
  return mode == 1 || (mode == 2 && k == PDL_CONV) || (mode == 3 && k == PDL_KF);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(PdlKernel which, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(which) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace fc
