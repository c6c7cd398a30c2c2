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
#include "launch_util.h"
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

// ---------------------------------------------------------------- backward
// The same decomposition as the forward, as block-wide device functions
// over shared buffers (256 threads; L = 64 L1, W = W_L^e).
// forward: x (time, natural, only n < nin non-zero) -> y (stage A + twiddle,
// [k2][n1]) -> X (spectrum, natural f)
FC_DEVICE void f32_forward(const float2* x, float2* y, float2* X, const float2* W, int L1, int ka) {
  const int L = 64 * L1;
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const int n1 = i % L1, k2 = i / L1;
    float2 acc = make_float2(0.f, 0.f);
    for (int n2 = 0; n2 < ka; ++n2) acc = cmac(acc, x[n1 + L1 * n2], W[((n2 * k2) & 63) * L1]);
    y[i] = cmul_(acc, W[n1 * k2]);
  }
  __syncthreads();
  for (int f = threadIdx.x; f < L; f += blockDim.x) {
    const int k2 = f & 63, k1 = f >> 6;
    float2 acc = make_float2(0.f, 0.f);
    for (int n1 = 0; n1 < L1; ++n1) acc = cmac(acc, y[k2 * L1 + n1], W[((n1 * k1) % L1) * 64]);
    X[f] = acc;
  }
  __syncthreads();
}
// inverse without scaling: X (spectrum) -> y ([k2][n1]) ; outputs n < nout
// are returned through out(n, value)
template <typename Out>
FC_DEVICE void f32_inverse(const float2* X, float2* y, const float2* W, int L1, int nout, Out&& out) {
  const int L = 64 * L1;
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const int n1 = i % L1, k2 = i / L1;
    float2 acc = make_float2(0.f, 0.f);
    for (int k1 = 0; k1 < L1; ++k1) acc = cmacc(acc, X[k2 + 64 * k1], W[((n1 * k1) % L1) * 64]);
    y[i] = cmulc_(acc, W[n1 * k2]);
  }
  __syncthreads();
  for (int n = threadIdx.x; n < nout; n += blockDim.x) {
    const int n1 = n % L1, n2 = n / L1;
    float2 acc = make_float2(0.f, 0.f);
    for (int k2 = 0; k2 < 64; ++k2) acc = cmacc(acc, y[k2 * L1 + n1], W[((n2 * k2) & 63) * L1]);
    out(n, acc);
  }
  __syncthreads();
}

// One CTA per (row pair, head): G = FFT(g), DC = FFT(dc) (two rows packed
// per complex transform, R1/R2), the pair's partial spectrum DC conj(G) / L
// for dk (summed over pairs by dk_rows in pair order: deterministic),
// c = IFFT(G k_f) / L (dv), dg = IFFT(DC conj(k_f)) / L (du, dw).
template <bool CAUSAL, bool GATE_IO, bool NEED_C>
__global__ void __launch_bounds__(256) fftconv_bwd_f32_kernel(const BwdParams prm, const float2* wl) {
  extern __shared__ float2 sm[];  // X | Y | G | D | W  (L complex each)
  const int L1 = prm.L1, L = 64 * L1, N = int(prm.N);
  float2 *X = sm, *Y = sm + L, *G = sm + 2 * L, *D = sm + 3 * L, *W = sm + 4 * L;
  for (int e = threadIdx.x; e < L; e += blockDim.x) W[e] = wl[e];
  const int64_t H = prm.H, B = prm.B, pairs = (B + 1) / 2;
  const float* gu = reinterpret_cast<const float*>(prm.u);
  const float* gw = reinterpret_cast<const float*>(prm.w);
  const float* gv = reinterpret_cast<const float*>(prm.v);
  const float* gdy = reinterpret_cast<const float*>(prm.dy);
  float* gdu = reinterpret_cast<float*>(prm.du);
  float* gdw = reinterpret_cast<float*>(prm.dw);
  float* gdv = reinterpret_cast<float*>(prm.dv);
  const uint32_t cpr = uint32_t(L1 / 2);
  const float inv_l = 1.0f / float(L);
  const int ka = CAUSAL ? 32 : 64;
  for (int64_t unit = blockIdx.x; unit < pairs * H; unit += gridDim.x) {
    const int64_t h = unit % H, p = unit / H;
    const int64_t r0 = ((2 * p) * H + h) * prm.N, r1 = r0 + H * prm.N;
    const bool has1 = 2 * p + 1 < B;
    const uint8_t* kfh = reinterpret_cast<const uint8_t*>(prm.kf) + h * int64_t(64 * tab_stride(cpr));
    auto kf_at = [&](int f) {
      const int k2 = f & 63, k1 = f >> 6;
      const float4 q = *reinterpret_cast<const float4*>(kfh + tab_off_rt(cpr, uint32_t(k2), uint32_t(k1 >> 1)));
      return (k1 & 1) ? make_float2(q.y, q.w) : make_float2(q.x, q.z);
    };
    __syncthreads();
    // g = u (* w), dc = dy (* v): rows b, b+1 packed as one complex row
    for (int n = threadIdx.x; n < L; n += blockDim.x) {
      float a = 0.f, c = 0.f;
      if (n < N) {
        a = gu[r0 + n];
        c = has1 ? gu[r1 + n] : 0.f;
        if (GATE_IO) { a *= gw[r0 + n]; c *= has1 ? gw[r1 + n] : 0.f; }
      }
      X[n] = make_float2(a, c);
    }
    __syncthreads();
    f32_forward(X, Y, G, W, L1, ka);
    for (int n = threadIdx.x; n < L; n += blockDim.x) {
      float a = 0.f, c = 0.f;
      if (n < N) {
        a = gdy[r0 + n];
        c = has1 ? gdy[r1 + n] : 0.f;
        if (GATE_IO) { a *= gv[r0 + n]; c *= has1 ? gv[r1 + n] : 0.f; }
      }
      X[n] = make_float2(a, c);
    }
    __syncthreads();
    f32_forward(X, Y, D, W, L1, ka);
    // partial spectrum of this pair (natural f order), X1 = G k_f
    float2* part = reinterpret_cast<float2*>(prm.acc) + (h * pairs + p) * int64_t(L);
    for (int f = threadIdx.x; f < L; f += blockDim.x) {
      const float2 g = G[f], d = D[f];
      part[f] = make_float2((d.x * g.x + d.y * g.y) * inv_l, (d.y * g.x - d.x * g.y) * inv_l);
      if (NEED_C) X[f] = cmul_(g, kf_at(f));
    }
    __syncthreads();
    if (NEED_C) {  // c -> dv = dy * c (gated I/O) or the c rows (inner)
      f32_inverse(X, Y, W, L1, N, [&](int n, float2 o) {
        float a = o.x * inv_l, c = o.y * inv_l;
        if (GATE_IO) {
          gdv[r0 + n] = a * gdy[r0 + n];
          if (has1) gdv[r1 + n] = c * gdy[r1 + n];
        } else {
          gdv[r0 + n] = a;
          if (has1) gdv[r1 + n] = c;
        }
      });
    }
    // X2 = DC conj(k_f) -> dg -> du = dg * w, dw = dg * u (gated I/O) or dg
    for (int f = threadIdx.x; f < L; f += blockDim.x) X[f] = cmulc_(D[f], kf_at(f));
    __syncthreads();
    f32_inverse(X, Y, W, L1, N, [&](int n, float2 o) {
      const float a = o.x * inv_l, c = o.y * inv_l;
      if (GATE_IO) {
        const float u0 = gu[r0 + n], w0 = gw[r0 + n];
        gdu[r0 + n] = a * w0;
        gdw[r0 + n] = a * u0;
        if (has1) {
          const float u1 = gu[r1 + n], w1 = gw[r1 + n];
          gdu[r1 + n] = c * w1;
          gdw[r1 + n] = c * u1;
        }
      } else {
        gdu[r0 + n] = a;
        if (has1) gdu[r1 + n] = c;
      }
    });
  }
}

template <bool CAUSAL, bool GATE_IO, bool NEED_C>
cudaError_t launch_bwd_f32_t(const BwdParams& prm, const float2* wl, cudaStream_t s) {
  const int L = prm.L1 * 64;
  const size_t smem = size_t(5) * size_t(L) * sizeof(float2);
  auto kern = fftconv_bwd_f32_kernel<CAUSAL, GATE_IO, NEED_C>;
  static int attr[64] = {0};
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(smem), attr)) return e;
  const int64_t units = ((prm.B + 1) / 2) * prm.H;
  const int64_t cap = int64_t(prm.num_sms) * 2;
  const unsigned grid = unsigned(units < cap ? units : cap);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, 256, smem, s>>>(prm, wl);
  return cudaGetLastError();
}

template <bool CAUSAL, bool GATED>
cudaError_t launch_f32_t(const FwdParams& prm, cudaStream_t s) {
  const int L = prm.L1 * 64;
  const size_t smem = size_t(3) * size_t(L) * sizeof(float2);
  auto kern = fftconv_f32_kernel<CAUSAL, GATED>;
  static int attr[64] = {0};
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(smem), attr)) return e;
  const int64_t units = ((prm.B + 1) / 2) * prm.H;
  const int64_t cap = int64_t(prm.num_sms) * 4;
  const unsigned grid = unsigned(units < cap ? units : cap);
  if (grid == 0) return cudaSuccess;
  kern<<<grid, 256, smem, s>>>(prm);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_bwd_f32(const BwdParams& prm, const void* wl, cudaStream_t s) {
  if (prm.L1 * 64 > 2048 || prm.L1 < 8) return cudaErrorInvalidValue;
  const float2* w = static_cast<const float2*>(wl);
  if (prm.gate_io) {  // fused gated: c always needed for dv
    return prm.causal ? launch_bwd_f32_t<true, true, true>(prm, w, s) : launch_bwd_f32_t<false, true, true>(prm, w, s);
  }
  if (prm.need_c)
    return prm.causal ? launch_bwd_f32_t<true, false, true>(prm, w, s) : launch_bwd_f32_t<false, false, true>(prm, w, s);
  return prm.causal ? launch_bwd_f32_t<true, false, false>(prm, w, s) : launch_bwd_f32_t<false, false, false>(prm, w, s);
}
int64_t bwd_f32_units_per_head(int64_t B) { return (B + 1) / 2; }

cudaError_t launch_fwd_f32(const FwdParams& prm, cudaStream_t s) {
  if (prm.L1 * 64 > 2048 || prm.L1 < 8) return cudaErrorInvalidValue;
  if (prm.causal) return prm.gated ? launch_f32_t<true, true>(prm, s) : launch_f32_t<true, false>(prm, s);
  return prm.gated ? launch_f32_t<false, true>(prm, s) : launch_f32_t<false, false>(prm, s);
}

}  // namespace fc
