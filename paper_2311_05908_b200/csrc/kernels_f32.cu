// kernels_f32.cu -- fp32 validation build of the fused order-2 convolution
// (north star: "<= 1e-5 relative L2 on an fp32 validation build").
//
// The same method as kernels_fwd.cu -- two real rows packed as one complex
// sequence z = g_b + i g_{b+1}, the order-2 Monarch decomposition
// L = L1 * 64, n = n1 + L1 n2, f = k2 + 64 k1 (Alg. 1
// P:200-220), causal skipping of the zero half in stage A and of the
// discarded half in stage A^-1, the pointwise product with k_f in
// the plan layout, gating fused on load and store -- but every stage
// is an fp32 sum on the CUDA cores instead of an fp16 tensor-core GEMM, so
// the result is limited only by fp32 rounding.  One CTA per (row pair, head);
// the working set (L complex fp32, two buffers) and the plan's W_L^e table
// live in shared memory.  It is also the inner pass of the fp32 multipass
// regime (circular, fp32 complex rows in place).  Not a performance path.
#include <cuda_runtime.h>

#include "fwd_params.h"
#include "layout.h"
#include "sm100.cuh"

namespace fc {

namespace {

FC_DEVICE float2 cmac(float2 acc, float2 a, float2 w) {
  return make_float2(fmaf(a.x, w.x, fmaf(-a.y, w.y, acc.x)), fmaf(a.x, w.y, fmaf(a.y, w.x, acc.y)));
}
FC_DEVICE float2 cmacc(float2 acc, float2 a, float2 w) {  // acc + a * conj(w)
  return make_float2(fmaf(a.x, w.x, fmaf(a.y, w.y, acc.x)), fmaf(a.y, w.x, fmaf(-a.x, w.y, acc.y)));
}
FC_DEVICE float2 cmul_(float2 a, float2 w) { return cmac(make_float2(0.f, 0.f), a, w); }
FC_DEVICE float2 cmulc_(float2 a, float2 w) { return cmacc(make_float2(0.f, 0.f), a, w); }

template <bool CAUSAL, bool GATED>
__global__ void __launch_bounds__(256) fftconv_f32_kernel(const FwdParams prm) {
  extern __shared__ float2 sm[];  // X[L] | Y[L] | W[L] (W_L^e)
  const int L1 = prm.L1, L = L1 * 64, N = int(prm.N);
  float2* X = sm;
  float2* Y = sm + L;
  float2* W = sm + 2 * L;
  const float2* wl = reinterpret_cast<const float2*>(prm.wl);
  for (int e = threadIdx.x; e < L; e += blockDim.x) W[e] = wl[e];
  const int64_t H = prm.H, B = prm.B, pairs = (B + 1) / 2;
  const float* u = reinterpret_cast<const float*>(prm.u);
  const float* w = reinterpret_cast<const float*>(prm.w);
  const float* v = reinterpret_cast<const float*>(prm.v);
  float* y = reinterpret_cast<float*>(prm.y);
  const uint32_t cpr = uint32_t(L1 / 2);
  const float inv_l = 1.0f / float(L);
  constexpr int KA = CAUSAL ? 32 : 64;  // stage A contracts only the non-zero half
  for (int64_t unit = blockIdx.x; unit < pairs * H; unit += gridDim.x) {
    const int64_t h = unit % H, p = unit / H;
    const int64_t r0 = ((2 * p) * H + h) * prm.N, r1 = r0 + H * prm.N;
    const bool has1 = 2 * p + 1 < B;
    const uint8_t* kf = reinterpret_cast<const uint8_t*>(prm.kf) + h * int64_t(64 * tab_stride(cpr));
    __syncthreads();  // W loaded / the previous unit is done with X and Y
    for (int n = threadIdx.x; n < L; n += blockDim.x) {
      float a = 0.f, c = 0.f;
      if (n < N) {
        a = u[r0 + n];
        c = has1 ? u[r1 + n] : 0.f;
        if (GATED) {
          a *= w[r0 + n];
          c *= has1 ? w[r1 + n] : 0.f;
        }
      }
      X[n] = make_float2(a, c);
    }
    __syncthreads();
    // stage A (contract n2 -> k2) and twiddle W_L^{n1 k2}: Y[k2 L1 + n1]
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      const int n1 = i % L1, k2 = i / L1;
      float2 acc = make_float2(0.f, 0.f);
      for (int n2 = 0; n2 < KA; ++n2) acc = cmac(acc, X[n1 + L1 * n2], W[((n2 * k2) & 63) * L1]);
      Y[i] = cmul_(acc, W[n1 * k2]);
    }
    __syncthreads();
    // stage B (contract n1 -> k1) and pointwise k_f: X[f], f = k2 + 64 k1
    for (int f = threadIdx.x; f < L; f += blockDim.x) {
      const int k2 = f & 63, k1 = f >> 6;
      float2 acc = make_float2(0.f, 0.f);
      for (int n1 = 0; n1 < L1; ++n1) acc = cmac(acc, Y[k2 * L1 + n1], W[((n1 * k1) % L1) * 64]);
      const float4 q = *reinterpret_cast<const float4*>(kf + tab_off_rt(cpr, uint32_t(k2), uint32_t(k1 >> 1)));
      X[f] = cmul_(acc, (k1 & 1) ? make_float2(q.y, q.w) : make_float2(q.x, q.z));
    }
    __syncthreads();
    // stage B^-1 (contract k1 -> n1) and conj twiddle: Y[k2 L1 + n1]
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      const int n1 = i % L1, k2 = i / L1;
      float2 acc = make_float2(0.f, 0.f);
      for (int k1 = 0; k1 < L1; ++k1) acc = cmacc(acc, X[k2 + 64 * k1], W[((n1 * k1) % L1) * 64]);
      Y[i] = cmulc_(acc, W[n1 * k2]);
    }
    __syncthreads();
    // stage A^-1 (contract k2 -> n2), only n < N; 1/L; demux, gate, store
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const int n1 = n % L1, n2 = n / L1;
      float2 acc = make_float2(0.f, 0.f);
      for (int k2 = 0; k2 < 64; ++k2) acc = cmacc(acc, Y[k2 * L1 + n1], W[((n2 * k2) & 63) * L1]);
      float a = acc.x * inv_l, c = acc.y * inv_l;
      if (GATED) {
        a *= v[r0 + n];
        if (has1) c *= v[r1 + n];
      }
      y[r0 + n] = a;
      if (has1) y[r1 + n] = c;
    }
  }
}

template <bool CAUSAL, bool GATED>
cudaError_t launch_f32_t(const FwdParams& prm, cudaStream_t s) {
  const int L = prm.L1 * 64;
  const size_t smem = size_t(3) * size_t(L) * sizeof(float2);
  auto kern = fftconv_f32_kernel<CAUSAL, GATED>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const int64_t units = ((prm.B + 1) / 2) * prm.H;
  const int64_t cap = int64_t(prm.num_sms) * 4;
  const unsigned grid = unsigned(units < cap ? units : cap);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, 256, smem, s>>>(prm);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fwd_f32(const FwdParams& prm, cudaStream_t s) {
  if (prm.L1 * 64 > 2048 || prm.L1 < 8) return cudaErrorInvalidValue;
  if (prm.causal) return prm.gated ? launch_f32_t<true, true>(prm, s) : launch_f32_t<true, false>(prm, s);
  return prm.gated ? launch_f32_t<false, true>(prm, s) : launch_f32_t<false, false>(prm, s);
}

}  // namespace fc
