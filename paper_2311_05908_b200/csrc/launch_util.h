// launch_util.h -- host-side launch helpers shared by the kernel files.
#pragma once
#include <cuda_runtime.h>

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

}  // namespace fc
