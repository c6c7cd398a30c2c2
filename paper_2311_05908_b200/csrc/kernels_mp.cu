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
#include "dft_vec.cuh"
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
template <>
FC_DEVICE float2 ld2<float>(const float* p) {
  return *reinterpret_cast<const float2*>(p);
}
template <typename T>
FC_DEVICE void st2(T* p, float a, float b);
template <>
FC_DEVICE void st2<float>(float* p, float a, float b) {
  *reinterpret_cast<float2*>(p) = make_float2(a, b);
}
template <>
FC_DEVICE void st2<__half>(__half* p, float a, float b) {
  *reinterpret_cast<__half2*>(p) = __floats2half2_rn(a, b);
}
template <>
FC_DEVICE void st2<__nv_bfloat16>(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}

// Outer passes.  Each thread owns COLS adjacent columns n' of one (pair,
// head); every complex value is a column vector (dft_vec.cuh), so the
// DFT_L0 over n0 runs on packed f32x2 instructions and every global access
// is a COLS-wide vector (a warp reads/writes 32 * COLS consecutive elements
// of a row).  MODE: 0 causal (inputs n0 < L0/2, outputs n0 < L0/2),
// 1 partial (overlap-save window: all inputs, outputs n0 >= L0/2), 2 circular
// (deep levels: complex rows in and out).
template <int L0>
struct PassCfg {
  static constexpr int COLS = L0 <= 8 ? 4 : 2;
  static constexpr int C2 = COLS / 2;
};

// COLS adjacent elements of type T as one vector access
template <int BYTES>
struct RawVec;
template <>
struct RawVec<4> { using type = uint32_t; };
template <>
struct RawVec<8> { using type = uint2; };
template <>
struct RawVec<16> { using type = uint4; };
template <typename T, int COLS>
using Raw = typename RawVec<int(sizeof(T)) * COLS>::type;

template <typename T, int COLS>
FC_DEVICE void unpack_cols(const Raw<T, COLS>& v, float* f) {
  const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int j = 0; j < COLS; j += 2) {
    const float2 a = ld2<T>(e + j);
    f[j] = a.x; f[j + 1] = a.y;
  }
}
template <typename T, int COLS>
FC_DEVICE void ld_cols(const T* p, float* f) {
  unpack_cols<T, COLS>(*reinterpret_cast<const Raw<T, COLS>*>(p), f);
}
template <typename T, int COLS>
FC_DEVICE void st_cols(T* p, const float* f) {
  Raw<T, COLS> v;
  T* e = reinterpret_cast<T*>(&v);
#pragma unroll
  for (int j = 0; j < COLS; j += 2) st2<T>(e + j, f[j], f[j + 1]);
  *reinterpret_cast<Raw<T, COLS>*>(p) = v;
}

// per-column twiddle base W_Llev^{n + j}: plan table (W_L^{n'}, n' < Lp) for
// one-level plans (wtab set), else sincospif of an exact dyadic fraction
template <int C2>
FC_DEVICE CV<C2> twiddle_base(const MpParams& prm, int n) {
  CV<C2> bw;
#pragma unroll
  for (int c = 0; c < C2; ++c) {
    float2 w0, w1;
    if (prm.wtab) {
      const float4 q = *reinterpret_cast<const float4*>(prm.wbase + n + 2 * c);
      w0 = make_float2(q.x, q.y);
      w1 = make_float2(q.z, q.w);
    } else {
      float sn, cs;
      sincospif(-2.0f * float(n + 2 * c) / float(prm.Llev), &sn, &cs);
      w0 = make_float2(cs, sn);
      sincospif(-2.0f * float(n + 2 * c + 1) / float(prm.Llev), &sn, &cs);
      w1 = make_float2(cs, sn);
    }
    bw.r[c] = make_float2(w0.x, w1.x);
    bw.i[c] = make_float2(w0.y, w1.y);
  }
  return bw;
}

template <int L0, int MODE, bool GATED, typename T, typename TT>
#ifndef FC_PASS_MINB
#define FC_PASS_MINB 3
#endif
__global__ void __launch_bounds__(256, FC_PASS_MINB) mp_pass1_kernel(const MpParams prm) {
  constexpr int COLS = PassCfg<L0>::COLS, C2 = PassCfg<L0>::C2;
  constexpr int NIN = MODE == 0 ? L0 / 2 : L0;
  const int64_t NCH = int64_t(prm.Lp) / COLS;  // column groups per (pair, head)
  // 32-bit index math (the launcher checks pairs * H * NCH < 2^31); NCH is a power of two
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t pairs = uint32_t((prm.B + 1) / 2);
  if (idx >= pairs * uint32_t(prm.H) * uint32_t(NCH)) return;
  const int n = int(idx & uint32_t(NCH - 1)) * COLS;
  const uint32_t ph = idx >> (31 - __clz(uint32_t(NCH)));
  const int64_t h = ph % uint32_t(prm.H), p = ph / uint32_t(prm.H);
  const int64_t b0 = 2 * p, b1 = 2 * p + 1;
  const bool has1 = b1 < prm.B;
  const T* __restrict__ u = reinterpret_cast<const T*>(prm.u);
  const T* __restrict__ w = reinterpret_cast<const T*>(prm.w);
  // element offset of sample n0 = 0 of each row; window start (may be < 0)
  const int64_t Hg = prm.Hg ? prm.Hg : prm.H, hg = h + prm.h0;  // global head
  const int64_t g0 = b0 + 2 * prm.pair0, g1 = g0 + 1;          // global rows
  int64_t r0, r1, s0 = 0, s1 = 0;
  if (MODE == 1) {  // virtual rows < 2^31 (launcher): 32-bit division
    const uint32_t nc = uint32_t(prm.NC);
    const int64_t q0 = uint32_t(g0) / nc, q1 = uint32_t(g1) / nc;
    const int64_t j0 = g0 - q0 * nc, j1 = g1 - q1 * nc;
    s0 = (j0 - 1) * prm.C;
    s1 = (j1 - 1) * prm.C;
    r0 = (q0 * Hg + hg) * prm.N + s0 + n;
    r1 = (q1 * Hg + hg) * prm.N + s1 + n;
  } else {
    r0 = (g0 * Hg + hg) * prm.N + n;
    r1 = (g1 * Hg + hg) * prm.N + n;
  }
  CV<C2> z[NIN];  // z = g_b + i g_{b+1}
#pragma unroll
  for (int n0 = 0; n0 < NIN; ++n0) {
    const int64_t o = int64_t(n0) * prm.Lp;
    // partial: the window's first half may precede the row (zeros); the
    // backward's dc windows keep only their second half (win_hi_only)
    const bool hi_only = MODE == 1 && prm.win_hi_only && n0 < L0 / 2;
    // a pair's two windows are consecutive (j, j+1) of one row: the second
    // window's first half is the first window's second half (copied below)
    const bool reused = MODE == 1 && !prm.win_hi_only && n0 < L0 / 2;
    const bool ok0 = !hi_only && (MODE != 1 || s0 + o >= 0);
    const bool ok1 = !hi_only && !reused && has1 && (MODE != 1 || s1 + o >= 0);
    float a[COLS], c[COLS];
#pragma unroll
    for (int j = 0; j < COLS; ++j) a[j] = c[j] = 0.f;
    if (ok0) ld_cols<T, COLS>(u + r0 + o, a);
    if (ok1) ld_cols<T, COLS>(u + r1 + o, c);
    if (GATED) {
      float wa[COLS], wc[COLS];
#pragma unroll
      for (int j = 0; j < COLS; ++j) wa[j] = wc[j] = 0.f;
      if (ok0) ld_cols<T, COLS>(w + r0 + o, wa);
      if (ok1) ld_cols<T, COLS>(w + r1 + o, wc);
#pragma unroll
      for (int j = 0; j < COLS; ++j) { a[j] *= wa[j]; c[j] *= wc[j]; }
    }
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      z[n0].r[cc] = make_float2(a[2 * cc], a[2 * cc + 1]);
      z[n0].i[cc] = make_float2(c[2 * cc], c[2 * cc + 1]);
    }
  }
  if (MODE == 1 && !prm.win_hi_only && has1) {
#pragma unroll
    for (int n0 = 0; n0 < L0 / 2; ++n0)
#pragma unroll
      for (int cc = 0; cc < C2; ++cc) z[n0].i[cc] = z[n0 + L0 / 2].r[cc];
  }
  // DFT_L0 over n0.  Causal rows are zero for n0 >= L0/2, so the first
  // radix-2 stage reduces to X[2m] = DFT_{L0/2}(z)[m],
  // X[2m+1] = DFT_{L0/2}(z W_L0^{n0})[m].
  CV<C2> X[L0];
  if constexpr (MODE == 0) {
    CV<C2> a[L0 / 2], b[L0 / 2];
#pragma unroll
    for (int n0 = 0; n0 < L0 / 2; ++n0) {
      a[n0] = z[n0];
      if (n0 == 0) {
        b[n0] = z[n0];
      } else if (4 * n0 == L0) {  // * (-i)
#pragma unroll
        for (int cc = 0; cc < C2; ++cc) {
          b[n0].r[cc] = z[n0].i[cc];
          b[n0].i[cc] = make_float2(-z[n0].r[cc].x, -z[n0].r[cc].y);
        }
      } else {
        const float2 wr = w_root<L0>(n0);
        b[n0] = cv_mul_s(z[n0], wr.x, wr.y);
      }
    }
    DftVec<L0 / 2, false, C2>::run(a);
    DftVec<L0 / 2, false, C2>::run(b);
#pragma unroll
    for (int m = 0; m < L0 / 2; ++m) {
      X[2 * m] = a[m];
      X[2 * m + 1] = b[m];
    }
  } else {
#pragma unroll
    for (int i = 0; i < L0; ++i) X[i] = z[i];
    DftVec<L0, false, C2>::run(X);
  }
  // twiddle W_L^{n' k0} (recurrence over k0 from W_L^{n'}), scale 1/sqrt(L0)
  const CV<C2> bw = twiddle_base<C2>(prm, n);
  const float s = ldexpf(rsqrtf(float(L0)), -prm.shift);  // (headroom pre-scale)
  CV<C2> tw;
#pragma unroll
  for (int cc = 0; cc < C2; ++cc) {
    tw.r[cc] = make_float2(s, s);
    tw.i[cc] = make_float2(0.f, 0.f);
  }
  TT* __restrict__ Tre = reinterpret_cast<TT*>(prm.ws) + ((2 * p) * prm.H * L0 + h * L0) * int64_t(prm.Lp) + n;
  TT* __restrict__ Tim = Tre + prm.H * L0 * int64_t(prm.Lp);
  uint32_t keep = ~0u;  // masked rows (sparse plans) are skipped downstream
  if (prm.row_keep) {
    keep = 0;
#pragma unroll
    for (int k0 = 0; k0 < L0; ++k0) keep |= prm.row_keep[k0] ? (1u << k0) : 0u;
  }
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    const CV<C2> o = cv_mul(X[k0], tw);
    if (k0 + 1 < L0) tw = cv_mul(tw, bw);
    if (keep & (1u << k0)) {
      float fr[COLS], fi[COLS];
#pragma unroll
      for (int cc = 0; cc < C2; ++cc) {
        fr[2 * cc] = o.r[cc].x; fr[2 * cc + 1] = o.r[cc].y;
        fi[2 * cc] = o.i[cc].x; fi[2 * cc + 1] = o.i[cc].y;
      }
      st_cols<TT, COLS>(Tre + int64_t(k0) * prm.Lp, fr);
      st_cols<TT, COLS>(Tim + int64_t(k0) * prm.Lp, fi);
    }
  }
}

template <int L0, int MODE, bool GATED, typename T, typename TT>
__global__ void __launch_bounds__(256, FC_PASS_MINB) mp_pass3_kernel(const MpParams prm) {
  constexpr int COLS = PassCfg<L0>::COLS, C2 = PassCfg<L0>::C2;
  const int64_t NCH = int64_t(prm.Lp) / COLS;
  // 32-bit index math (the launcher checks pairs * H * NCH < 2^31); NCH is a power of two
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t pairs = uint32_t((prm.B + 1) / 2);
  if (idx >= pairs * uint32_t(prm.H) * uint32_t(NCH)) return;
  const int n = int(idx & uint32_t(NCH - 1)) * COLS;
  const uint32_t ph = idx >> (31 - __clz(uint32_t(NCH)));
  const int64_t h = ph % uint32_t(prm.H), p = ph / uint32_t(prm.H);
  const TT* __restrict__ Tre =
      reinterpret_cast<const TT*>(prm.ws) + ((2 * p) * prm.H * L0 + h * L0) * int64_t(prm.Lp) + n;
  const TT* __restrict__ Tim = Tre + prm.H * L0 * int64_t(prm.Lp);
  const CV<C2> bw = twiddle_base<C2>(prm, n);
  const float s = ldexpf(rsqrtf(float(L0)), prm.shift);  // (undo the headroom pre-scale)
  CV<C2> tw;
#pragma unroll
  for (int cc = 0; cc < C2; ++cc) {
    tw.r[cc] = make_float2(s, s);
    tw.i[cc] = make_float2(0.f, 0.f);
  }
  CV<C2> e[L0 / 2], o[L0 / 2];  // even / odd k0, conj-twiddled and scaled
  // all rows are loaded up front (no load waits on another): dense plans
  // unconditionally, sparse plans only the kept rows (the others were never
  // written by pass 1)
  using RawT = Raw<TT, COLS>;
  RawT rr[L0], ri[L0];
  const bool sparse = prm.row_keep != nullptr;
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    if (!sparse || prm.row_keep[k0]) {
      rr[k0] = *reinterpret_cast<const RawT*>(Tre + int64_t(k0) * prm.Lp);
      ri[k0] = *reinterpret_cast<const RawT*>(Tim + int64_t(k0) * prm.Lp);
    } else {
      rr[k0] = RawT{};
      ri[k0] = RawT{};
    }
  }
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    float fr[COLS], fi[COLS];
    unpack_cols<TT, COLS>(rr[k0], fr);
    unpack_cols<TT, COLS>(ri[k0], fi);
    CV<C2> x;
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      x.r[cc] = make_float2(fr[2 * cc], fr[2 * cc + 1]);
      x.i[cc] = make_float2(fi[2 * cc], fi[2 * cc + 1]);
    }
    x = cv_mulc(x, tw);
    if (k0 + 1 < L0) tw = cv_mul(tw, bw);
    if (k0 & 1) o[k0 / 2] = x;
    else e[k0 / 2] = x;
  }
  // inverse DFT_L0 over k0: y[m] = E[m] + W_L0^{-m} O[m], y[m + L0/2] = E[m] - W_L0^{-m} O[m]
  DftVec<L0 / 2, true, C2>::run(e);
  DftVec<L0 / 2, true, C2>::run(o);
  CV<C2> xl[L0 / 2], xh[L0 / 2];
#pragma unroll
  for (int m = 0; m < L0 / 2; ++m) cv_bfly<L0, true>(m, e[m], o[m], xl[m], xh[m]);
  const int64_t b0 = 2 * p, b1 = 2 * p + 1;
  const bool has1 = b1 < prm.B;
  T* __restrict__ y = reinterpret_cast<T*>(prm.y);
  const T* __restrict__ v = reinterpret_cast<const T*>(prm.v);
  const int64_t Hg = prm.Hg ? prm.Hg : prm.H, hg = h + prm.h0;  // global head
  const int64_t g0 = b0 + 2 * prm.pair0, g1 = g0 + 1;          // global rows
  int64_t r0, r1;
  if (MODE == 1) {  // virtual rows < 2^31 (launcher): 32-bit division
    const uint32_t nc = uint32_t(prm.NC);
    const int64_t q0 = uint32_t(g0) / nc, q1 = uint32_t(g1) / nc;
    r0 = (q0 * Hg + hg) * prm.N + (g0 - q0 * nc) * prm.C + n;
    r1 = (q1 * Hg + hg) * prm.N + (g1 - q1 * nc) * prm.C + n;
  } else {
    r0 = (g0 * Hg + hg) * prm.N + n;
    r1 = (g1 * Hg + hg) * prm.N + n;
  }
  auto emit = [&](const CV<C2>& x, int64_t off) {
    float a[COLS], c[COLS];  // rows b (real part), b+1 (imaginary part)
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      a[2 * cc] = x.r[cc].x; a[2 * cc + 1] = x.r[cc].y;
      c[2 * cc] = x.i[cc].x; c[2 * cc + 1] = x.i[cc].y;
    }
    if (prm.y2) {  // second gated output (backward: dw = dg * u)
      const T* v2 = reinterpret_cast<const T*>(prm.v2);
      T* y2 = reinterpret_cast<T*>(prm.y2);
      float g[COLS], q[COLS];
      ld_cols<T, COLS>(v2 + r0 + off, g);
#pragma unroll
      for (int j = 0; j < COLS; ++j) q[j] = a[j] * g[j];
      st_cols<T, COLS>(y2 + r0 + off, q);
      if (has1) {
        ld_cols<T, COLS>(v2 + r1 + off, g);
#pragma unroll
        for (int j = 0; j < COLS; ++j) q[j] = c[j] * g[j];
        st_cols<T, COLS>(y2 + r1 + off, q);
      }
    }
    if (GATED) {
      float g[COLS];
      ld_cols<T, COLS>(v + r0 + off, g);
#pragma unroll
      for (int j = 0; j < COLS; ++j) a[j] *= g[j];
      if (has1) {
        ld_cols<T, COLS>(v + r1 + off, g);
#pragma unroll
        for (int j = 0; j < COLS; ++j) c[j] *= g[j];
      }
    }
    st_cols<T, COLS>(y + r0 + off, a);
    if (has1) st_cols<T, COLS>(y + r1 + off, c);
  };
  // causal keeps n0 < L0/2 (lo), partial n0 >= L0/2 (hi), circular both;
  // partial output rows start at the window's second half (offset 0 of y)
  if (MODE != 1) {
#pragma unroll
    for (int m = 0; m < L0 / 2; ++m) emit(xl[m], int64_t(m) * prm.Lp);
  }
  if (MODE != 0) {
    const int64_t q0 = MODE == 2 ? L0 / 2 : 0;
#pragma unroll
    for (int m = 0; m < L0 / 2; ++m) emit(xh[m], (q0 + m) * prm.Lp);
  }
}

// Frequency-sparse one-level plans: only the nrow kept outer rows k0 are
// produced (pass 1) and consumed (pass 3), each as a direct sum over n0 with
// W_L0^{n0 k0} from the constant root table and W_L^{n' k0} from the plan's
// [k0][n'] table -- a quarter of the work of the full DFT_L0 for cfg 5's
// 4-of-16 pattern, with 4-column vectors at every L0.
template <int NPT>
FC_DEVICE float2 w_full(int k) {  // W_NPT^k, any k
  k &= NPT - 1;
  if (k < NPT / 2) return w_root<NPT>(k);
  const float2 w = w_root<NPT>(k - NPT / 2);
  return make_float2(-w.x, -w.y);
}

template <int L0, int MODE, bool GATED, typename T, typename TT>
__global__ void __launch_bounds__(256, 2) mp_pass1_sparse_kernel(const MpParams prm) {
  constexpr int COLS = 4, C2 = 2;
  constexpr int NIN = MODE == 0 ? L0 / 2 : L0;
  const int64_t NCH = int64_t(prm.Lp) / COLS;
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t pairs = uint32_t((prm.B + 1) / 2);
  if (idx >= pairs * uint32_t(prm.H) * uint32_t(NCH)) return;
  const int n = int(idx & uint32_t(NCH - 1)) * COLS;
  const uint32_t ph = idx >> (31 - __clz(uint32_t(NCH)));
  const int64_t h = ph % uint32_t(prm.H), p = ph / uint32_t(prm.H);
  const int64_t b0 = 2 * p, b1 = 2 * p + 1;
  const bool has1 = b1 < prm.B;
  const T* __restrict__ u = reinterpret_cast<const T*>(prm.u);
  const T* __restrict__ w = reinterpret_cast<const T*>(prm.w);
  const int64_t Hg = prm.Hg ? prm.Hg : prm.H, hg = h + prm.h0;
  const int64_t g0 = b0 + 2 * prm.pair0, g1 = g0 + 1;
  int64_t r0, r1, s0 = 0, s1 = 0;
  if (MODE == 1) {
    const uint32_t nc = uint32_t(prm.NC);
    const int64_t q0 = uint32_t(g0) / nc, q1 = uint32_t(g1) / nc;
    s0 = (g0 - q0 * nc - 1) * prm.C;
    s1 = (g1 - q1 * nc - 1) * prm.C;
    r0 = (q0 * Hg + hg) * prm.N + s0 + n;
    r1 = (q1 * Hg + hg) * prm.N + s1 + n;
  } else {
    r0 = (g0 * Hg + hg) * prm.N + n;
    r1 = (g1 * Hg + hg) * prm.N + n;
  }
  CV<C2> z[NIN];
#pragma unroll
  for (int n0 = 0; n0 < NIN; ++n0) {
    const int64_t o = int64_t(n0) * prm.Lp;
    const bool hi_only = MODE == 1 && prm.win_hi_only && n0 < L0 / 2;
    // a pair's two windows are consecutive (j, j+1) of one row: the second
    // window's first half is the first window's second half (copied below)
    const bool reused = MODE == 1 && !prm.win_hi_only && n0 < L0 / 2;
    const bool ok0 = !hi_only && (MODE != 1 || s0 + o >= 0);
    const bool ok1 = !hi_only && !reused && has1 && (MODE != 1 || s1 + o >= 0);
    float a[COLS], c[COLS];
#pragma unroll
    for (int j = 0; j < COLS; ++j) a[j] = c[j] = 0.f;
    if (ok0) ld_cols<T, COLS>(u + r0 + o, a);
    if (ok1) ld_cols<T, COLS>(u + r1 + o, c);
    if (GATED) {
      float wa[COLS], wc[COLS];
#pragma unroll
      for (int j = 0; j < COLS; ++j) wa[j] = wc[j] = 0.f;
      if (ok0) ld_cols<T, COLS>(w + r0 + o, wa);
      if (ok1) ld_cols<T, COLS>(w + r1 + o, wc);
#pragma unroll
      for (int j = 0; j < COLS; ++j) { a[j] *= wa[j]; c[j] *= wc[j]; }
    }
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      z[n0].r[cc] = make_float2(a[2 * cc], a[2 * cc + 1]);
      z[n0].i[cc] = make_float2(c[2 * cc], c[2 * cc + 1]);
    }
  }
  if (MODE == 1 && !prm.win_hi_only && has1) {
#pragma unroll
    for (int n0 = 0; n0 < L0 / 2; ++n0)
#pragma unroll
      for (int cc = 0; cc < C2; ++cc) z[n0].i[cc] = z[n0 + L0 / 2].r[cc];
  }
  const float s = ldexpf(rsqrtf(float(L0)), -prm.shift);  // (headroom pre-scale)
  TT* __restrict__ Tre = reinterpret_cast<TT*>(prm.ws) + ((2 * p) * prm.H * L0 + h * L0) * int64_t(prm.Lp) + n;
  TT* __restrict__ Tim = Tre + prm.H * L0 * int64_t(prm.Lp);
  for (int q = 0; q < prm.nrow; ++q) {
    const int k0 = prm.row_map[q];
    CV<C2> acc;
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) acc.r[cc] = acc.i[cc] = make_float2(0.f, 0.f);
#pragma unroll
    for (int n0 = 0; n0 < NIN; ++n0) {
      const float2 wr = w_full<L0>(n0 * k0);
      const CV<C2> t = cv_mul_s(z[n0], wr.x, wr.y);
#pragma unroll
      for (int cc = 0; cc < C2; ++cc) { acc.r[cc] = add2(acc.r[cc], t.r[cc]); acc.i[cc] = add2(acc.i[cc], t.i[cc]); }
    }
    // twiddle W_L^{n' k0} (plan table), scale 1/sqrt(L0)
    const float4 q01 = *reinterpret_cast<const float4*>(prm.wtab + int64_t(k0) * prm.Lp + n);
    const float4 q23 = *reinterpret_cast<const float4*>(prm.wtab + int64_t(k0) * prm.Lp + n + 2);
    CV<C2> tw;
    tw.r[0] = make_float2(q01.x * s, q01.z * s); tw.i[0] = make_float2(q01.y * s, q01.w * s);
    tw.r[1] = make_float2(q23.x * s, q23.z * s); tw.i[1] = make_float2(q23.y * s, q23.w * s);
    const CV<C2> o = cv_mul(acc, tw);
    float fr[COLS], fi[COLS];
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      fr[2 * cc] = o.r[cc].x; fr[2 * cc + 1] = o.r[cc].y;
      fi[2 * cc] = o.i[cc].x; fi[2 * cc + 1] = o.i[cc].y;
    }
    st_cols<TT, COLS>(Tre + int64_t(k0) * prm.Lp, fr);
    st_cols<TT, COLS>(Tim + int64_t(k0) * prm.Lp, fi);
  }
}

template <int L0, int MODE, bool GATED, typename T, typename TT>
__global__ void __launch_bounds__(256, 2) mp_pass3_sparse_kernel(const MpParams prm) {
  constexpr int COLS = 4, C2 = 2;
  constexpr int NOUT = MODE == 2 ? L0 : L0 / 2;      // output rows n0
  constexpr int Q0 = MODE == 1 ? L0 / 2 : 0;         // first output n0
  const int64_t NCH = int64_t(prm.Lp) / COLS;
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t pairs = uint32_t((prm.B + 1) / 2);
  if (idx >= pairs * uint32_t(prm.H) * uint32_t(NCH)) return;
  const int n = int(idx & uint32_t(NCH - 1)) * COLS;
  const uint32_t ph = idx >> (31 - __clz(uint32_t(NCH)));
  const int64_t h = ph % uint32_t(prm.H), p = ph / uint32_t(prm.H);
  const TT* __restrict__ Tre =
      reinterpret_cast<const TT*>(prm.ws) + ((2 * p) * prm.H * L0 + h * L0) * int64_t(prm.Lp) + n;
  const TT* __restrict__ Tim = Tre + prm.H * L0 * int64_t(prm.Lp);
  const float s = ldexpf(rsqrtf(float(L0)), prm.shift);  // (undo the headroom pre-scale)
  CV<C2> x[NOUT];
#pragma unroll
  for (int m = 0; m < NOUT; ++m)
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) x[m].r[cc] = x[m].i[cc] = make_float2(0.f, 0.f);
  for (int q = 0; q < prm.nrow; ++q) {
    const int k0 = prm.row_map[q];
    float fr[COLS], fi[COLS];
    ld_cols<TT, COLS>(Tre + int64_t(k0) * prm.Lp, fr);
    ld_cols<TT, COLS>(Tim + int64_t(k0) * prm.Lp, fi);
    const float4 q01 = *reinterpret_cast<const float4*>(prm.wtab + int64_t(k0) * prm.Lp + n);
    const float4 q23 = *reinterpret_cast<const float4*>(prm.wtab + int64_t(k0) * prm.Lp + n + 2);
    CV<C2> v, tw;
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      v.r[cc] = make_float2(fr[2 * cc], fr[2 * cc + 1]);
      v.i[cc] = make_float2(fi[2 * cc], fi[2 * cc + 1]);
    }
    tw.r[0] = make_float2(q01.x * s, q01.z * s); tw.i[0] = make_float2(q01.y * s, q01.w * s);
    tw.r[1] = make_float2(q23.x * s, q23.z * s); tw.i[1] = make_float2(q23.y * s, q23.w * s);
    v = cv_mulc(v, tw);  // conj twiddle and 1/sqrt(L0)
#pragma unroll
    for (int m = 0; m < NOUT; ++m) {
      const float2 wr = w_full<L0>((Q0 + m) * k0);
      const CV<C2> t = cv_mul_s(v, wr.x, -wr.y);  // W_L0^{-n0 k0}
#pragma unroll
      for (int cc = 0; cc < C2; ++cc) { x[m].r[cc] = add2(x[m].r[cc], t.r[cc]); x[m].i[cc] = add2(x[m].i[cc], t.i[cc]); }
    }
  }
  const int64_t b0 = 2 * p, b1 = 2 * p + 1;
  const bool has1 = b1 < prm.B;
  T* __restrict__ y = reinterpret_cast<T*>(prm.y);
  const T* __restrict__ v = reinterpret_cast<const T*>(prm.v);
  const int64_t Hg = prm.Hg ? prm.Hg : prm.H, hg = h + prm.h0;
  const int64_t g0 = b0 + 2 * prm.pair0, g1 = g0 + 1;
  int64_t r0, r1;
  if (MODE == 1) {
    const uint32_t nc = uint32_t(prm.NC);
    const int64_t q0 = uint32_t(g0) / nc, q1 = uint32_t(g1) / nc;
    r0 = (q0 * Hg + hg) * prm.N + (g0 - q0 * nc) * prm.C + n;
    r1 = (q1 * Hg + hg) * prm.N + (g1 - q1 * nc) * prm.C + n;
  } else {
    r0 = (g0 * Hg + hg) * prm.N + n;
    r1 = (g1 * Hg + hg) * prm.N + n;
  }
#pragma unroll
  for (int m = 0; m < NOUT; ++m) {
    const int64_t off = int64_t(m) * prm.Lp;  // partial: rows start at the window's second half
    float a[COLS], c[COLS];
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      a[2 * cc] = x[m].r[cc].x; a[2 * cc + 1] = x[m].r[cc].y;
      c[2 * cc] = x[m].i[cc].x; c[2 * cc + 1] = x[m].i[cc].y;
    }
    if (prm.y2) {
      const T* v2 = reinterpret_cast<const T*>(prm.v2);
      T* y2 = reinterpret_cast<T*>(prm.y2);
      float g[COLS], qv[COLS];
      ld_cols<T, COLS>(v2 + r0 + off, g);
#pragma unroll
      for (int j = 0; j < COLS; ++j) qv[j] = a[j] * g[j];
      st_cols<T, COLS>(y2 + r0 + off, qv);
      if (has1) {
        ld_cols<T, COLS>(v2 + r1 + off, g);
#pragma unroll
        for (int j = 0; j < COLS; ++j) qv[j] = c[j] * g[j];
        st_cols<T, COLS>(y2 + r1 + off, qv);
      }
    }
    if (GATED) {
      float g[COLS];
      ld_cols<T, COLS>(v + r0 + off, g);
#pragma unroll
      for (int j = 0; j < COLS; ++j) a[j] *= g[j];
      if (has1) {
        ld_cols<T, COLS>(v + r1 + off, g);
#pragma unroll
        for (int j = 0; j < COLS; ++j) c[j] *= g[j];
      }
    }
    st_cols<T, COLS>(y + r0 + off, a);
    if (has1) st_cols<T, COLS>(y + r1 + off, c);
  }
}

// Backward of the partial convolution, dg by overlap-add: the circular
// correlation of window j (dc block j in its second half, zeros in its
// first) with k spans positions [(j-1)C, (j+1)C) of dg, so
// dg[jC : (j+1)C] = hi(window j) + lo(window j+1) (no wrap: K <= C).  A thread
// owns pair p = windows (2p, 2p+1) of one batch row (NC is even): block 2p is
// hi(re) + lo(im) of pair p, block 2p+1 is hi(im) of pair p + lo(re) of pair
// p+1 (absent for the row's last window).
template <int L0, typename TT, int C2>
FC_DEVICE void pair_idft(const MpParams& prm, int64_t p, int64_t h, int n, const CV<C2>& bw, CV<C2>* xl,
                         CV<C2>* xh) {
  constexpr int COLS = 2 * C2;
  const TT* Tre = reinterpret_cast<const TT*>(prm.ws) + ((2 * p) * prm.H * L0 + h * L0) * int64_t(prm.Lp) + n;
  const TT* Tim = Tre + prm.H * L0 * int64_t(prm.Lp);
  using RawT = Raw<TT, COLS>;
  RawT rr[L0], ri[L0];
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    rr[k0] = *reinterpret_cast<const RawT*>(Tre + int64_t(k0) * prm.Lp);
    ri[k0] = *reinterpret_cast<const RawT*>(Tim + int64_t(k0) * prm.Lp);
  }
  const float s = ldexpf(rsqrtf(float(L0)), prm.shift);  // (undo the headroom pre-scale)
  CV<C2> tw;
#pragma unroll
  for (int cc = 0; cc < C2; ++cc) {
    tw.r[cc] = make_float2(s, s);
    tw.i[cc] = make_float2(0.f, 0.f);
  }
  CV<C2> e[L0 / 2], o[L0 / 2];
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    float fr[COLS], fi[COLS];
    unpack_cols<TT, COLS>(rr[k0], fr);
    unpack_cols<TT, COLS>(ri[k0], fi);
    CV<C2> x;
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      x.r[cc] = make_float2(fr[2 * cc], fr[2 * cc + 1]);
      x.i[cc] = make_float2(fi[2 * cc], fi[2 * cc + 1]);
    }
    x = cv_mulc(x, tw);
    if (k0 + 1 < L0) tw = cv_mul(tw, bw);
    if (k0 & 1) o[k0 / 2] = x;
    else e[k0 / 2] = x;
  }
  DftVec<L0 / 2, true, C2>::run(e);
  DftVec<L0 / 2, true, C2>::run(o);
#pragma unroll
  for (int m = 0; m < L0 / 2; ++m) cv_bfly<L0, true>(m, e[m], o[m], xl[m], xh[m]);
}

template <int L0, bool GATED, typename T, typename TT>
__global__ void __launch_bounds__(256, 2) mp_pass3_ola_kernel(const MpParams prm) {
  constexpr int COLS = PassCfg<L0>::COLS, C2 = PassCfg<L0>::C2;
  const int64_t NCH = int64_t(prm.Lp) / COLS;
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t pairs = uint32_t((prm.B + 1) / 2);
  if (idx >= pairs * uint32_t(prm.H) * uint32_t(NCH)) return;
  const int n = int(idx & uint32_t(NCH - 1)) * COLS;
  const uint32_t ph = idx >> (31 - __clz(uint32_t(NCH)));
  const int64_t h = ph % uint32_t(prm.H), p = ph / uint32_t(prm.H);
  const CV<C2> bw = twiddle_base<C2>(prm, n);
  CV<C2> xl[L0 / 2], xh[L0 / 2], nl[L0 / 2], nh[L0 / 2];
  pair_idft<L0, TT, C2>(prm, p, h, n, bw, xl, xh);
  const uint32_t nc = uint32_t(prm.NC);
  const int64_t g0 = 2 * p, b = uint32_t(g0) / nc, j0 = g0 - b * int64_t(nc);
  const bool has_next = j0 + 2 < int64_t(nc);  // window j0 + 2 belongs to the same row
  if (has_next) pair_idft<L0, TT, C2>(prm, p + 1, h, n, bw, nl, nh);
  const int64_t Hg = prm.Hg ? prm.Hg : prm.H, hg = h + prm.h0;
  const int64_t row = (b * Hg + hg) * prm.N + n;
  T* __restrict__ y = reinterpret_cast<T*>(prm.y);
  auto emit = [&](float* a, int64_t off) {  // one output row segment of COLS
    if (prm.y2) {
      float g[COLS], q[COLS];
      ld_cols<T, COLS>(reinterpret_cast<const T*>(prm.v2) + off, g);
#pragma unroll
      for (int j = 0; j < COLS; ++j) q[j] = a[j] * g[j];
      st_cols<T, COLS>(reinterpret_cast<T*>(prm.y2) + off, q);
    }
    if (GATED) {
      float g[COLS];
      ld_cols<T, COLS>(reinterpret_cast<const T*>(prm.v) + off, g);
#pragma unroll
      for (int j = 0; j < COLS; ++j) a[j] *= g[j];
    }
    st_cols<T, COLS>(y + off, a);
  };
#pragma unroll
  for (int m = 0; m < L0 / 2; ++m) {
    float a[COLS], c[COLS];
#pragma unroll
    for (int cc = 0; cc < C2; ++cc) {
      // block j0: hi(window j0) + lo(window j0 + 1)
      a[2 * cc] = xh[m].r[cc].x + xl[m].i[cc].x;
      a[2 * cc + 1] = xh[m].r[cc].y + xl[m].i[cc].y;
      // block j0 + 1: hi(window j0 + 1) + lo(window j0 + 2)
      c[2 * cc] = xh[m].i[cc].x + (has_next ? nl[m].r[cc].x : 0.f);
      c[2 * cc + 1] = xh[m].i[cc].y + (has_next ? nl[m].r[cc].y : 0.f);
    }
    emit(a, row + j0 * prm.C + int64_t(m) * prm.Lp);
    emit(c, row + (j0 + 1) * prm.C + int64_t(m) * prm.Lp);
  }
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
    z[n0] = make_float2(prm.kb ? filter_tap(prm, h, t) : t < prm.K ? prm.k[h * prm.K + t] : 0.f, 0.f);
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
    if (!prm.row_keep || prm.row_keep[k0])  // masked rows: zero-filled by the rows step
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

// T: I/O type; the intermediate is fp16 except in the fp32 validation build
template <int L0, int MODE, bool G, typename T>
static void launch_pass_k(const MpParams& prm, int pass, unsigned grid, cudaStream_t s) {
  using TT = typename std::conditional<std::is_same<T, float>::value, float, __half>::type;
  if (prm.row_map && prm.wtab) {  // sparse one-level plans: kept rows only
    const int64_t total = ((prm.B + 1) / 2) * prm.H * (prm.Lp / 4);
    const unsigned g4 = unsigned((total + 255) / 256);
    if (pass == 1) mp_pass1_sparse_kernel<L0, MODE, G, T, TT><<<g4, 256, 0, s>>>(prm);
    else mp_pass3_sparse_kernel<L0, MODE, G, T, TT><<<g4, 256, 0, s>>>(prm);
    return;
  }
  if (pass == 1) mp_pass1_kernel<L0, MODE, G, T, TT><<<grid, 256, 0, s>>>(prm);
  else mp_pass3_kernel<L0, MODE, G, T, TT><<<grid, 256, 0, s>>>(prm);
}
template <int L0, int MODE>
static void launch_pass_m(const MpParams& prm, int pass, unsigned grid, cudaStream_t s) {
  const bool g = prm.gated != 0;
  if (prm.dtype == 2) {  // fp32 validation build
    if (g) launch_pass_k<L0, MODE, true, float>(prm, pass, grid, s);
    else launch_pass_k<L0, MODE, false, float>(prm, pass, grid, s);
  } else if (prm.dtype == 0) {
    if (g) launch_pass_k<L0, MODE, true, __half>(prm, pass, grid, s);
    else launch_pass_k<L0, MODE, false, __half>(prm, pass, grid, s);
  } else {
    if (g) launch_pass_k<L0, MODE, true, __nv_bfloat16>(prm, pass, grid, s);
    else launch_pass_k<L0, MODE, false, __nv_bfloat16>(prm, pass, grid, s);
  }
}

template <int L0>
static cudaError_t launch_mp_l0(const MpParams& prm, int pass, cudaStream_t s) {
  const int64_t total = ((prm.B + 1) / 2) * prm.H * (prm.Lp / PassCfg<L0>::COLS);
  const unsigned grid = unsigned((total + 255) / 256);
  if (total == 0) return cudaSuccess;
  if (total + 255 >= (int64_t(1) << 31) || (prm.Lp & (prm.Lp - 1))) return cudaErrorInvalidValue;
  if (2 * (prm.pair0 + (prm.B + 1) / 2) >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  if (prm.circ) {  // circular: deep levels (fp16 complex rows) or a circular plan's top level
    launch_pass_m<L0, 2>(prm, pass, grid, s);
  } else if (prm.partial && prm.ola && pass == 3) {  // backward dg of the partial conv
    if ((prm.NC & 1) || prm.pair0 || prm.h0) return cudaErrorInvalidValue;
    const bool g = prm.gated != 0;
    if (prm.dtype == 0) {
      if (g) mp_pass3_ola_kernel<L0, true, __half, __half><<<grid, 256, 0, s>>>(prm);
      else mp_pass3_ola_kernel<L0, false, __half, __half><<<grid, 256, 0, s>>>(prm);
    } else if (prm.dtype == 1) {
      if (g) mp_pass3_ola_kernel<L0, true, __nv_bfloat16, __half><<<grid, 256, 0, s>>>(prm);
      else mp_pass3_ola_kernel<L0, false, __nv_bfloat16, __half><<<grid, 256, 0, s>>>(prm);
    } else {  // fp32 validation build
      if (g) mp_pass3_ola_kernel<L0, true, float, float><<<grid, 256, 0, s>>>(prm);
      else mp_pass3_ola_kernel<L0, false, float, float><<<grid, 256, 0, s>>>(prm);
    }
  } else if (prm.partial) {
    // pass 1 pairs windows (2p, 2p+1) of one row (a pair's second window
    // reuses the first one's second half): needs an even window count
    if (pass == 1 && !prm.win_hi_only && (prm.NC & 1)) return cudaErrorInvalidValue;
    launch_pass_m<L0, 1>(prm, pass, grid, s);
  } else {
    launch_pass_m<L0, 0>(prm, pass, grid, s);
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
