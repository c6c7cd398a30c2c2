// kernels_mp.cu -- multipass regime for long sequences (Alg. 4).
//
// L = L0 * L' with L' = 2048 (the fused order-2 kernel's circular size) and
// L0 = L / L' in {2, 4, 8, 16}; n = n' + L' n0, f = k0 + L0 f'.
//   pass 1 (outer forward, this file): for each row pair z = g_b + i g_{b+1}
//     and column n', DFT_L0 over n0 (only n0 < L0/2 are non-zero: causal
//     padding), twiddle W_L^{n' k0}, scale 1/sqrt(L0)  ->  T,
//     stored as fp16 rows (2p + re/im, h L0 + k0, n').
//   pass 2 (inner, kernels_fwd.cu): the fused circular kernel on T with
//     H' = H L0 "heads" (h, k0); head (h, k0) uses the k_f block
//     K_f[k0 + L0 f'] ("fold N1 into H").
//   pass 3 (outer inverse, this file): conj twiddle, IDFT_L0 over k0, keep
//     n0 < L0/2 (causal output), scale 1/sqrt(L0), split re/im into rows b,
//     b+1, gate by v, store.
// The outer DFTs are small (L0 <= 16) and run in fp32 registers; the
// tensor-core work is in pass 2.  T is written in place by pass 2.
#include <cuda_runtime.h>

#include <type_traits>

#include "dft_small.cuh"
#include "fwd_params.h"
#include "sm100.cuh"

namespace fc {

namespace {

template <typename T>
FC_DEVICE float2 ld2(const T* p);
template <>
FC_DEVICE float2 ld2<__half>(const __half* p) {
  return __half22float2(*reinterpret_cast<const __half2*>(p));
}
template <>
FC_DEVICE float2 ld2<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
}
template <typename T>
FC_DEVICE void st2(T* p, float a, float b);
template <>
FC_DEVICE void st2<__half>(__half* p, float a, float b) {
  *reinterpret_cast<__half2*>(p) = __floats2half2_rn(a, b);
}
template <>
FC_DEVICE void st2<__nv_bfloat16>(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}

// Each thread owns two adjacent columns (n', n'+1) of one (pair, head).
template <int L0, bool GATED, typename T>
__global__ void __launch_bounds__(256) mp_pass1_kernel(const MpParams prm) {
  const int64_t NP = int64_t(prm.Lp) / 2;  // column pairs per (pair, head)
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t pairs = (prm.B + 1) / 2;
  if (idx >= pairs * prm.H * NP) return;
  const int cp = int(idx % NP);
  const int64_t ph = idx / NP;
  const int64_t h = ph % prm.H, p = ph / prm.H;
  const int n = 2 * cp;  // first column n'
  const int64_t b0 = 2 * p, b1 = 2 * p + 1;
  const bool has1 = b1 < prm.B;
  const T* __restrict__ u = reinterpret_cast<const T*>(prm.u);
  const T* __restrict__ w = reinterpret_cast<const T*>(prm.w);
  // element offset of sample n0 = 0 of each row; window start (may be < 0)
  int64_t r0, r1, s0 = 0, s1 = 0;
  if (prm.partial) {
    const int64_t j0 = b0 % prm.NC, j1 = b1 % prm.NC;
    s0 = (j0 - 1) * prm.C;
    s1 = (j1 - 1) * prm.C;
    r0 = ((b0 / prm.NC) * prm.H + h) * prm.N + s0 + n;
    r1 = ((b1 / prm.NC) * prm.H + h) * prm.N + s1 + n;
  } else {
    r0 = (b0 * prm.H + h) * prm.N + n;
    r1 = (b1 * prm.H + h) * prm.N + n;
  }
  float2 z0[L0], z1[L0];  // column n and n+1, complex z = g_b + i g_{b+1}
#pragma unroll
  for (int n0 = 0; n0 < L0; ++n0) {
    z0[n0] = make_float2(0.f, 0.f);
    z1[n0] = make_float2(0.f, 0.f);
  }
  // causal: the zero-padded upper half is never loaded; partial: full window
  constexpr int NL = L0;
#pragma unroll
  for (int n0 = 0; n0 < NL; ++n0) {
    if (!prm.partial && !prm.circ && n0 >= L0 / 2) break;
    const int64_t o = int64_t(n0) * prm.Lp;
    const bool ok0 = s0 + o >= 0, ok1 = has1 && s1 + o >= 0;
    float2 a = ok0 ? ld2<T>(u + r0 + o) : make_float2(0.f, 0.f);  // row b, columns n, n+1
    float2 c = ok1 ? ld2<T>(u + r1 + o) : make_float2(0.f, 0.f);
    if (GATED) {
      const float2 wa = ok0 ? ld2<T>(w + r0 + o) : make_float2(0.f, 0.f);
      const float2 wc = ok1 ? ld2<T>(w + r1 + o) : make_float2(0.f, 0.f);
      a.x *= wa.x; a.y *= wa.y;
      c.x *= wc.x; c.y *= wc.y;
    }
    z0[n0] = make_float2(a.x, c.x);
    z1[n0] = make_float2(a.y, c.y);
  }
  // DFT_L0 over n0.  Causal rows are zero for n0 >= L0/2, so the first
  // radix-2 stage reduces to X[2m] = DFT_{L0/2}(z)[m],
  // X[2m+1] = DFT_{L0/2}(z W_L0^{n0})[m].
  float2 X0[L0], X1[L0];
  if (!prm.partial && !prm.circ) {
    float2 a0[L0 / 2], b0[L0 / 2], a1[L0 / 2], b1[L0 / 2];
#pragma unroll
    for (int n0 = 0; n0 < L0 / 2; ++n0) {
      const float2 w = w_root<L0>(n0);
      a0[n0] = z0[n0];
      a1[n0] = z1[n0];
      b0[n0] = c_mul(z0[n0], w);
      b1[n0] = c_mul(z1[n0], w);
    }
    DftReg<L0 / 2, false>::run(a0);
    DftReg<L0 / 2, false>::run(b0);
    DftReg<L0 / 2, false>::run(a1);
    DftReg<L0 / 2, false>::run(b1);
#pragma unroll
    for (int m = 0; m < L0 / 2; ++m) {
      X0[2 * m] = a0[m]; X0[2 * m + 1] = b0[m];
      X1[2 * m] = a1[m]; X1[2 * m + 1] = b1[m];
    }
  } else {
#pragma unroll
    for (int i = 0; i < L0; ++i) { X0[i] = z0[i]; X1[i] = z1[i]; }
    DftReg<L0, false>::run(X0);
    DftReg<L0, false>::run(X1);
  }
  // twiddle W_L^{n' k0} from the plan table [k0][n'], scale 1/sqrt(L0)
  const float s = rsqrtf(float(L0));
  __half* __restrict__ Tre = reinterpret_cast<__half*>(prm.ws) + ((2 * p) * prm.H * L0 + h * L0) * int64_t(prm.Lp) + n;
  __half* __restrict__ Tim = Tre + prm.H * L0 * int64_t(prm.Lp);
  // on-the-fly twiddles (deep levels): W_Llev^{n k0} by recurrence from
  // W_Llev^{n} (sincospif of an exact dyadic fraction; error ~ L0 ulp)
  float2 bw0 = make_float2(1.f, 0.f), bw1 = bw0, tw0 = bw0, tw1 = bw0;
  if (!prm.wtab) {
    float sn, cs;
    sincospif(-2.0f * float(n) / float(prm.Llev), &sn, &cs);
    bw0 = make_float2(cs, sn);
    sincospif(-2.0f * float(n + 1) / float(prm.Llev), &sn, &cs);
    bw1 = make_float2(cs, sn);
  }
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    float4 tw;
    if (prm.wtab) {
      tw = *reinterpret_cast<const float4*>(prm.wtab + int64_t(k0) * prm.Lp + n);
    } else {
      tw = make_float4(tw0.x, tw0.y, tw1.x, tw1.y);
      tw0 = c_mul(tw0, bw0);
      tw1 = c_mul(tw1, bw1);
    }
    const float2 a = c_mul(X0[k0], make_float2(tw.x, tw.y)), c = c_mul(X1[k0], make_float2(tw.z, tw.w));
    if (!prm.row_keep || prm.row_keep[k0]) {  // masked rows are skipped downstream
      *reinterpret_cast<__half2*>(Tre + int64_t(k0) * prm.Lp) = __floats2half2_rn(a.x * s, c.x * s);
      *reinterpret_cast<__half2*>(Tim + int64_t(k0) * prm.Lp) = __floats2half2_rn(a.y * s, c.y * s);
    }
  }
}

template <int L0, bool GATED, typename T>
__global__ void __launch_bounds__(256) mp_pass3_kernel(const MpParams prm) {
  const int64_t NP = int64_t(prm.Lp) / 2;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t pairs = (prm.B + 1) / 2;
  if (idx >= pairs * prm.H * NP) return;
  const int cp = int(idx % NP);
  const int64_t ph = idx / NP;
  const int64_t h = ph % prm.H, p = ph / prm.H;
  const int n = 2 * cp;
  const __half* __restrict__ Tre =
      reinterpret_cast<const __half*>(prm.ws) + ((2 * p) * prm.H * L0 + h * L0) * int64_t(prm.Lp) + n;
  const __half* __restrict__ Tim = Tre + prm.H * L0 * int64_t(prm.Lp);
  float2 e0[L0 / 2], o0[L0 / 2], e1[L0 / 2], o1[L0 / 2];  // even / odd k0
  float2 bw0 = make_float2(1.f, 0.f), bw1 = bw0, tw0 = bw0, tw1 = bw0;
  if (!prm.wtab) {
    float sn, cs;
    sincospif(-2.0f * float(n) / float(prm.Llev), &sn, &cs);
    bw0 = make_float2(cs, sn);
    sincospif(-2.0f * float(n + 1) / float(prm.Llev), &sn, &cs);
    bw1 = make_float2(cs, sn);
  }
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    const bool kept = !prm.row_keep || prm.row_keep[k0];
    const float2 re = kept ? __half22float2(*reinterpret_cast<const __half2*>(Tre + int64_t(k0) * prm.Lp))
                           : make_float2(0.f, 0.f);
    const float2 im = kept ? __half22float2(*reinterpret_cast<const __half2*>(Tim + int64_t(k0) * prm.Lp))
                           : make_float2(0.f, 0.f);
    float4 tw;
    if (prm.wtab) {
      tw = *reinterpret_cast<const float4*>(prm.wtab + int64_t(k0) * prm.Lp + n);
    } else {
      tw = make_float4(tw0.x, tw0.y, tw1.x, tw1.y);
      tw0 = c_mul(tw0, bw0);
      tw1 = c_mul(tw1, bw1);
    }
    const float2 a = c_mulc(make_float2(re.x, im.x), make_float2(tw.x, tw.y));
    const float2 c = c_mulc(make_float2(re.y, im.y), make_float2(tw.z, tw.w));
    if (k0 & 1) { o0[k0 / 2] = a; o1[k0 / 2] = c; }
    else { e0[k0 / 2] = a; e1[k0 / 2] = c; }
  }
  // inverse DFT_L0 over k0, half of the outputs: y[n0] = E[n0] +- W_L0^{-n0} O[n0]
  DftReg<L0 / 2, true>::run(e0);
  DftReg<L0 / 2, true>::run(o0);
  DftReg<L0 / 2, true>::run(e1);
  DftReg<L0 / 2, true>::run(o1);
  // causal keeps n0 < L0/2 (lo), partial n0 >= L0/2 (hi), circular both
  float2 x0[L0], x1[L0];
#pragma unroll
  for (int m = 0; m < L0 / 2; ++m) {
    float2 w = w_root<L0>(m);
    w.y = -w.y;
    const float2 t0 = c_mul(o0[m], w), t1 = c_mul(o1[m], w);
    x0[m] = c_add(e0[m], t0);
    x1[m] = c_add(e1[m], t1);
    x0[m + L0 / 2] = c_sub(e0[m], t0);
    x1[m + L0 / 2] = c_sub(e1[m], t1);
  }
  const float s = rsqrtf(float(L0));
  const int64_t b0 = 2 * p, b1 = 2 * p + 1;
  const bool has1 = b1 < prm.B;
  T* __restrict__ y = reinterpret_cast<T*>(prm.y);
  const T* __restrict__ v = reinterpret_cast<const T*>(prm.v);
  int64_t r0, r1;
  if (prm.partial) {
    r0 = ((b0 / prm.NC) * prm.H + h) * prm.N + (b0 % prm.NC) * prm.C + n;
    r1 = ((b1 / prm.NC) * prm.H + h) * prm.N + (b1 % prm.NC) * prm.C + n;
  } else {
    r0 = (b0 * prm.H + h) * prm.N + n;
    r1 = (b1 * prm.H + h) * prm.N + n;
  }
  auto emit = [&](auto q0c, auto noutc) {
    constexpr int Q0 = decltype(q0c)::value, NOUT = decltype(noutc)::value;
#pragma unroll
    for (int i0 = 0; i0 < NOUT; ++i0) {
      const int n0 = i0 + Q0;
      const int64_t o = int64_t(i0) * prm.Lp;
      float a0 = x0[n0].x * s, a1 = x1[n0].x * s;  // row b
      float c0 = x0[n0].y * s, c1 = x1[n0].y * s;  // row b+1
      if (GATED) {
        const float2 va = ld2<T>(v + r0 + o);
        a0 *= va.x; a1 *= va.y;
        if (has1) {
          const float2 vc = ld2<T>(v + r1 + o);
          c0 *= vc.x; c1 *= vc.y;
        }
      }
      if (prm.y2) {  // second gated output (backward: dw = dg * u)
        const T* v2 = reinterpret_cast<const T*>(prm.v2);
        T* y2 = reinterpret_cast<T*>(prm.y2);
        const float2 vb = ld2<T>(v2 + r0 + o);
        st2<T>(y2 + r0 + o, x0[n0].x * s * vb.x, x1[n0].x * s * vb.y);
        if (has1) {
          const float2 vd = ld2<T>(v2 + r1 + o);
          st2<T>(y2 + r1 + o, x0[n0].y * s * vd.x, x1[n0].y * s * vd.y);
        }
      }
      st2<T>(y + r0 + o, a0, a1);
      if (has1) st2<T>(y + r1 + o, c0, c1);
        }
  };
  if (prm.circ) emit(std::integral_constant<int, 0>{}, std::integral_constant<int, L0>{});
  else if (prm.partial) emit(std::integral_constant<int, L0 / 2>{}, std::integral_constant<int, L0 / 2>{});
  else emit(std::integral_constant<int, 0>{}, std::integral_constant<int, L0 / 2>{});
}

// k_f, step 1: per (head, column n'): DFT_L0 of k[n' + Lrow n0] (n0 < L0/2,
// K <= L/2), twiddle W_L^{n' k0}; fp32 scratch written into the head's k_f
// blocks: element (h, k0, n') lives in 2048-element block
// (h L0 + k0) * (Lrow / 2048) + n' / 2048 at offset n' % 2048 (unpadded).
template <int L0>
__global__ void __launch_bounds__(256) mp_kf_cols_kernel(const KfParams prm, int64_t Lrow, int64_t Lfull,
                                                         size_t block_bytes) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= prm.H * Lrow) return;
  const int64_t n = idx % Lrow;
  const int64_t h = idx / Lrow;
  float2 z[L0];
#pragma unroll
  for (int n0 = 0; n0 < L0; ++n0) {
    const int64_t t = n + int64_t(n0) * Lrow;
    z[n0] = make_float2(t < prm.K ? prm.k[h * prm.K + t] : 0.f, 0.f);
  }
  DftReg<L0, false>::run(z);
  float sn, cs;
  sincospif(-2.0f * float(n) / float(Lfull), &sn, &cs);  // exact dyadic argument
  const float2 bw = make_float2(cs, sn);
  float2 tw = make_float2(1.f, 0.f);
  const int64_t nb = Lrow / 2048;
  uint8_t* kf = reinterpret_cast<uint8_t*>(prm.kf);
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    const int64_t blk = (h * L0 + k0) * nb + n / 2048;
    reinterpret_cast<float2*>(kf + blk * block_bytes)[n % 2048] = c_mul(z[k0], tw);
    tw = c_mul(tw, bw);
  }
}

// Deeper levels, in place: rows of length Lrow = L0 * Lp (2048-element blocks
// of block_bytes each); thread (row, n'') reads x[n'' + Lp m], m < L0, and
// writes DFT_L0 (INV: inverse, unscaled) twiddled by W_Lrow^{+-n'' k0} at
// k0 Lp + n'' -- the same addresses, so no other thread is touched.
// Forward applies the twiddle after the DFT, inverse before it.
template <int L0, bool INV>
__global__ void __launch_bounds__(256) mp_cols_cplx_kernel(float2* data, int64_t rows, int64_t Lrow,
                                                           size_t block_bytes) {
  const int64_t Lp = Lrow / L0;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * Lp) return;
  const int64_t n = idx % Lp, r = idx / Lp;
  const int64_t nb = Lrow / 2048;
  uint8_t* base = reinterpret_cast<uint8_t*>(data);
  auto at = [&](int64_t e) -> float2* {
    return reinterpret_cast<float2*>(base + (r * nb + e / 2048) * int64_t(block_bytes)) + (e % 2048);
  };
  float sn, cs;
  sincospif((INV ? 2.0f : -2.0f) * float(n) / float(Lrow), &sn, &cs);
  const float2 bw = make_float2(cs, sn);
  float2 v[L0];
  float2 tw = make_float2(1.f, 0.f);
#pragma unroll
  for (int m = 0; m < L0; ++m) {
    v[m] = *at(n + Lp * m);
    if (INV) {  // inverse: twiddle first (index m is k0 here)
      v[m] = c_mul(v[m], tw);
      tw = c_mul(tw, bw);
    }
  }
  DftReg<L0, INV>::run(v);
#pragma unroll
  for (int m = 0; m < L0; ++m) {
    float2 o = v[m];
    if (!INV) {
      o = c_mul(o, tw);
      tw = c_mul(tw, bw);
    }
    *at(n + Lp * m) = o;
  }
}

}  // namespace

// k_f, step 2 lives in kernels_kf.cu (row FFTs into the inner plan layout).
cudaError_t launch_mp_kf_rows(const KfParams& prm, int L0, int Lp, size_t block_bytes, cudaStream_t s);

template <int L0>
static cudaError_t launch_mp_l0(const MpParams& prm, int pass, cudaStream_t s) {
  const int64_t total = ((prm.B + 1) / 2) * prm.H * (prm.Lp / 2);
  const unsigned grid = unsigned((total + 255) / 256);
  if (total == 0) return cudaSuccess;
  const bool g = prm.gated != 0;
  if (pass == 1) {
    if (prm.dtype == 0) {
      if (g) mp_pass1_kernel<L0, true, __half><<<grid, 256, 0, s>>>(prm);
      else mp_pass1_kernel<L0, false, __half><<<grid, 256, 0, s>>>(prm);
    } else {
      if (g) mp_pass1_kernel<L0, true, __nv_bfloat16><<<grid, 256, 0, s>>>(prm);
      else mp_pass1_kernel<L0, false, __nv_bfloat16><<<grid, 256, 0, s>>>(prm);
    }
  } else {
    if (prm.dtype == 0) {
      if (g) mp_pass3_kernel<L0, true, __half><<<grid, 256, 0, s>>>(prm);
      else mp_pass3_kernel<L0, false, __half><<<grid, 256, 0, s>>>(prm);
    } else {
      if (g) mp_pass3_kernel<L0, true, __nv_bfloat16><<<grid, 256, 0, s>>>(prm);
      else mp_pass3_kernel<L0, false, __nv_bfloat16><<<grid, 256, 0, s>>>(prm);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_mp_pass(const MpParams& prm, int pass, cudaStream_t s) {
  switch (prm.L0) {
    case 2: return launch_mp_l0<2>(prm, pass, s);
    case 4: return launch_mp_l0<4>(prm, pass, s);
    case 8: return launch_mp_l0<8>(prm, pass, s);
    case 16: return launch_mp_l0<16>(prm, pass, s);
    default: return cudaErrorInvalidValue;
  }
}

template <bool INV>
static cudaError_t launch_cols_cplx(float2* data, int L0, int64_t rows, int64_t Lrow, size_t block_bytes,
                                    cudaStream_t s) {
  const unsigned grid = unsigned((rows * (Lrow / L0) + 255) / 256);
  switch (L0) {
    case 2: mp_cols_cplx_kernel<2, INV><<<grid, 256, 0, s>>>(data, rows, Lrow, block_bytes); break;
    case 4: mp_cols_cplx_kernel<4, INV><<<grid, 256, 0, s>>>(data, rows, Lrow, block_bytes); break;
    case 8: mp_cols_cplx_kernel<8, INV><<<grid, 256, 0, s>>>(data, rows, Lrow, block_bytes); break;
    case 16: mp_cols_cplx_kernel<16, INV><<<grid, 256, 0, s>>>(data, rows, Lrow, block_bytes); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_mp_cols_inverse(float2* data, int L0, int64_t rows, int64_t Lrow, cudaStream_t s) {
  return launch_cols_cplx<true>(data, L0, rows, Lrow, 2048 * sizeof(float2), s);
}

cudaError_t launch_mp_precompute_kf(const KfParams& prm, const int32_t* lev_L0, int nlev, int64_t Lfull,
                                    size_t block_bytes, cudaStream_t s) {
  if (prm.H <= 0) return cudaSuccess;
  const int L0 = lev_L0[0];
  const int64_t Lrow = Lfull / L0;
  const unsigned grid = unsigned((prm.H * Lrow + 255) / 256);
  switch (L0) {
    case 2: mp_kf_cols_kernel<2><<<grid, 256, 0, s>>>(prm, Lrow, Lfull, block_bytes); break;
    case 4: mp_kf_cols_kernel<4><<<grid, 256, 0, s>>>(prm, Lrow, Lfull, block_bytes); break;
    case 8: mp_kf_cols_kernel<8><<<grid, 256, 0, s>>>(prm, Lrow, Lfull, block_bytes); break;
    case 16: mp_kf_cols_kernel<16><<<grid, 256, 0, s>>>(prm, Lrow, Lfull, block_bytes); break;
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int64_t rows = prm.H * L0, Lr = Lrow;
  for (int l = 1; l < nlev; ++l) {
    e = launch_cols_cplx<false>(reinterpret_cast<float2*>(prm.kf), lev_L0[l], rows, Lr, block_bytes, s);
    if (e != cudaSuccess) return e;
    rows *= lev_L0[l];
    Lr /= lev_L0[l];
  }
  int64_t L0tot = 1;
  for (int l = 0; l < nlev; ++l) L0tot *= lev_L0[l];
  return launch_mp_kf_rows(prm, int(L0tot), 2048, block_bytes, s);
}

}  // namespace fc
