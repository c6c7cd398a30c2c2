// kernels_kf.cu -- k_f = FFT_L(pad(k)) on the GPU in fp32.
//
// One CTA per head: the zero-padded filter row is transformed by an
// iterative radix-2 FFT in shared memory (fp32, twiddles from sincospif of an
// exactly representable dyadic argument), multiplied by the frequency mask
// (A13) and written in the fused kernel's plan layout: complex fp32 at
// f = k2 + L2 k1 stored as [k2][k1/2] element pairs {re, re', im, im'}, 128-byte XOR-swizzled so the pointwise
// epilogue reads it bank-conflict free.  No cuFFT.
#include <cuda_runtime.h>

#include "fwd_params.h"
#include "sm100.cuh"

namespace fc {

__global__ void __launch_bounds__(512) precompute_kf_kernel(const KfParams prm) {
  extern __shared__ float2 xs[];  // L data + L/2 twiddles
  const int64_t h = blockIdx.x;
  const int64_t L = prm.L, K = prm.K;
  float2* tw = xs + L;
  const int lg = __ffsll(L) - 1;
  const float* krow = prm.k + h * K;
  // twiddle table W_L^j, j < L/2 (dyadic argument, exact in fp32)
  for (int64_t j = threadIdx.x; j < L / 2; j += blockDim.x) {
    float sn, cs;
    sincospif(-2.0f * float(j) / float(L), &sn, &cs);
    tw[j] = make_float2(cs, sn);
  }
  // bit-reversed load of the zero-padded row
  for (int64_t n = threadIdx.x; n < L; n += blockDim.x) {
    const int64_t r = __brevll(uint64_t(n)) >> (64 - lg);
    xs[r] = make_float2(n < K ? krow[n] : 0.f, 0.f);
  }
  __syncthreads();
  for (int64_t len = 2, stride = L / 2; len <= L; len <<= 1, stride >>= 1) {
    const int64_t half = len >> 1;
    for (int64_t i = threadIdx.x; i < L / 2; i += blockDim.x) {
      const int64_t j = i & (half - 1), s = (i - j) * 2;
      const float2 w = tw[j * stride];
      const float2 a = xs[s + j], b = xs[s + j + half];
      const float2 t = make_float2(b.x * w.x - b.y * w.y, b.x * w.y + b.y * w.x);
      xs[s + j] = make_float2(a.x + t.x, a.y + t.y);
      xs[s + j + half] = make_float2(a.x - t.x, a.y - t.y);
    }
    __syncthreads();
  }
  uint8_t* out = reinterpret_cast<uint8_t*>(prm.kf) + h * L * 8;
  for (int64_t f = threadIdx.x; f < L; f += blockDim.x) {
    const int k2 = int(f % prm.L2), k1 = int(f / prm.L2);
    float2 v = xs[f];
    if (prm.mask) {
      const float m = prm.mask[f];
      v.x *= m;
      v.y *= m;
    }
    // [k2][k1/2] float4 {kr(k1), kr(k1+1), ki(k1), ki(k1+1)}, row-XOR swizzled (tab_off_rt)
    const uint32_t o = tab_off_rt(uint32_t(prm.L1 / 2), uint32_t(k2), uint32_t(k1 / 2)) + (k1 & 1) * 4;
    *reinterpret_cast<float*>(out + o) = v.x;
    *reinterpret_cast<float*>(out + o + 8) = v.y;
  }
}

cudaError_t launch_precompute_kf(const KfParams& prm, cudaStream_t s) {
  if (prm.H <= 0) return cudaSuccess;
  const size_t smem = size_t(prm.L) * sizeof(float2) * 3 / 2;
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(precompute_kf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  precompute_kf_kernel<<<unsigned(prm.H), 512, smem, s>>>(prm);
  return cudaGetLastError();
}

}  // namespace fc
