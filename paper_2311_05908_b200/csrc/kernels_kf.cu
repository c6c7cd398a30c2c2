// kernels_kf.cu -- k_f = FFT_L(pad(k)) on the GPU in fp32.
//
// One CTA per head.  The zero-padded filter row is transformed by a
// Stockham autosort FFT (radix-8 passes, one radix-2/4 pass when log2 L is
// not a multiple of 3) ping-ponging between two shared-memory buffers; each
// thread transforms 8 (or 4, 2) elements in registers per pass.  Twiddles
// W_L^e come from the plan's fp32 table (built in fp64 on the host, exponent
// reduced mod L in integers).  The result is multiplied by the frequency mask
// (A13) and written in the fused kernel's plan layout: complex fp32 at
// f = k2 + L2 k1 stored as [k2][k1/2] element pairs {re, re', im, im'} with
// padded rows (layout.h).  No cuFFT.
#include <cuda_runtime.h>

#include "dft_small.cuh"
#include "fwd_params.h"
#include "launch_util.h"
#include "sm100.cuh"

namespace fc {

namespace {

FC_DEVICE float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
FC_DEVICE float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
FC_DEVICE float2 cmulf(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
FC_DEVICE float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // a * (-i)

// in-register forward DFTs, natural order in and out
FC_DEVICE void dft2(float2* v) {
  const float2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}
FC_DEVICE void dft4(float2* v) {
  const float2 e0 = cadd(v[0], v[2]), e1 = csub(v[0], v[2]);
  const float2 o0 = cadd(v[1], v[3]), o1 = mul_mi(csub(v[1], v[3]));
  v[0] = cadd(e0, o0);
  v[2] = csub(e0, o0);
  v[1] = cadd(e1, o1);
  v[3] = csub(e1, o1);
}
FC_DEVICE void dft8(float2* v) {
  float2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
  dft4(e);
  dft4(o);
  const float r = 0.70710678118654752f;
  o[1] = make_float2(r * (o[1].x + o[1].y), r * (o[1].y - o[1].x));    // * W8^1
  o[2] = mul_mi(o[2]);                                                 // * W8^2
  o[3] = make_float2(r * (o[3].y - o[3].x), -r * (o[3].x + o[3].y));   // * W8^3
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = cadd(e[k], o[k]);
    v[k + 4] = csub(e[k], o[k]);
  }
}

// Compile-time Stockham FFT for 256-thread blocks and L in {512, 1024,
// 2048}: every index and twiddle exponent is a constant expression of the
// thread index.  Data live at padded positions pd(i) = i + i/8 (one spare
// float2 per 8) so the strided butterfly stores of the early passes do not
// pile onto one shared-memory bank; a butterfly reads 3 twiddles
// (W^e, W^2e, W^4e) and forms the other 4 by at most two fp32 products.
FC_DEVICE int pd(int i) { return i + (i >> 3); }
template <int L>
constexpr int padded_len() { return L + L / 8; }

template <int R, int L, int NS>
FC_DEVICE void stockham_pass_ct(float2* x, const float2* __restrict__ tw) {
  constexpr int G = L / R, GPT = (G + 255) / 256;
  float2 v[GPT][R];
#pragma unroll
  for (int g = 0; g < GPT; ++g) {
    const int j = threadIdx.x + g * 256;
    if (G % 256 == 0 || j < G) {
      const int jm = j % NS;
#pragma unroll
      for (int r = 0; r < R; ++r) v[g][r] = x[pd(j + r * G)];
      if (NS > 1) {
        constexpr int step = L / (NS * R);  // W_{NS R}^{jm r} = W_L^{jm r step}
        const int e = jm * step;
        const float2 w1 = tw[pd(e & (L - 1))];
        if constexpr (R == 2) {
          v[g][1] = cmulf(v[g][1], w1);
        } else {
          const float2 w2 = tw[pd((2 * e) & (L - 1))];
          v[g][1] = cmulf(v[g][1], w1);
          v[g][2] = cmulf(v[g][2], w2);
          v[g][3] = cmulf(v[g][3], cmulf(w1, w2));
          if constexpr (R == 8) {
            const float2 w4 = tw[pd((4 * e) & (L - 1))];
            v[g][4] = cmulf(v[g][4], w4);
            v[g][5] = cmulf(v[g][5], cmulf(w1, w4));
            v[g][6] = cmulf(v[g][6], cmulf(w2, w4));
            v[g][7] = cmulf(v[g][7], cmulf(cmulf(w1, w2), w4));
          }
        }
      }
      if constexpr (R == 8) dft8(v[g]);
      else if constexpr (R == 4) dft4(v[g]);
      else dft2(v[g]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int g = 0; g < GPT; ++g) {
    const int j = threadIdx.x + g * 256;
    if (G % 256 == 0 || j < G) {
      const int jm = j % NS;
      const int base = (j / NS) * NS * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) x[pd(base + r * NS)] = v[g][r];
    }
  }
  __syncthreads();
}
template <int L>
FC_DEVICE void fft_inplace_ct(float2* xs, const float2* tws) {
  static_assert(L == 512 || L == 1024 || L == 2048 || L == 4096 || L == 8192, "compile-time FFT sizes");
  if constexpr (L == 8192) {  // 2 * 8 * 8 * 8 * 8
    stockham_pass_ct<2, L, 1>(xs, tws);
    stockham_pass_ct<8, L, 2>(xs, tws);
    stockham_pass_ct<8, L, 16>(xs, tws);
    stockham_pass_ct<8, L, 128>(xs, tws);
    stockham_pass_ct<8, L, 1024>(xs, tws);
  } else if constexpr (L == 4096) {  // 8 * 8 * 8 * 8
    stockham_pass_ct<8, L, 1>(xs, tws);
    stockham_pass_ct<8, L, 8>(xs, tws);
    stockham_pass_ct<8, L, 64>(xs, tws);
    stockham_pass_ct<8, L, 512>(xs, tws);
  } else if constexpr (L == 512) {  // 8 * 8 * 8
    stockham_pass_ct<8, L, 1>(xs, tws);
    stockham_pass_ct<8, L, 8>(xs, tws);
    stockham_pass_ct<8, L, 64>(xs, tws);
  } else if constexpr (L == 1024) {  // 2 * 8 * 8 * 8
    stockham_pass_ct<2, L, 1>(xs, tws);
    stockham_pass_ct<8, L, 2>(xs, tws);
    stockham_pass_ct<8, L, 16>(xs, tws);
    stockham_pass_ct<8, L, 128>(xs, tws);
  } else {  // 4 * 8 * 8 * 8
    stockham_pass_ct<4, L, 1>(xs, tws);
    stockham_pass_ct<8, L, 4>(xs, tws);
    stockham_pass_ct<8, L, 32>(xs, tws);
    stockham_pass_ct<8, L, 256>(xs, tws);
  }
}
// Forward FFT of the padded buffer xs (natural order; twiddles W_L^e also
// padded); the launchers use
// 256-thread blocks and L in {512, 1024, 2048} only.
FC_DEVICE void fft_inplace_any(float2* xs, const float2* tws, int L) {
  if (L == 2048) fft_inplace_ct<2048>(xs, tws);
  else if (L == 1024) fft_inplace_ct<1024>(xs, tws);
  else fft_inplace_ct<512>(xs, tws);
}
// One Stockham pass (radix R, stride NS) over L points in shared memory by
// TH threads, twiddles computed per butterfly (the order-3 k_f sizes do not
// leave room for a twiddle table beside the data at 16384 points).
template <int R, int L, int NS, int TH>
FC_DEVICE void stockham_pass_otf(float2* x) {
  constexpr int G = L / R, GPT = (G + TH - 1) / TH;
  static_assert(G % TH == 0 || G < TH, "whole butterflies per thread");
  float2 v[GPT][R];
#pragma unroll
  for (int g = 0; g < GPT; ++g) {
    const int j = threadIdx.x + g * TH;
    if (G < TH && j >= G) break;
    const int jm = j % NS;
#pragma unroll
    for (int r = 0; r < R; ++r) v[g][r] = x[pd(j + r * G)];
    if (NS > 1) {
      constexpr int step = L / (NS * R);  // W_{NS R}^{jm r} = W_L^{jm r step}
      const int e = jm * step;
      auto w = [](int ee) {
        float sn, cs;
        sincospif(-2.0f * float(ee & (L - 1)) / float(L), &sn, &cs);
        return make_float2(cs, sn);
      };
      const float2 w1 = w(e);
      if constexpr (R == 2) {
        v[g][1] = cmulf(v[g][1], w1);
      } else {
        const float2 w2 = w(2 * e);
        v[g][1] = cmulf(v[g][1], w1);
        v[g][2] = cmulf(v[g][2], w2);
        v[g][3] = cmulf(v[g][3], cmulf(w1, w2));
        if constexpr (R == 8) {
          const float2 w4 = w(4 * e);
          v[g][4] = cmulf(v[g][4], w4);
          v[g][5] = cmulf(v[g][5], cmulf(w1, w4));
          v[g][6] = cmulf(v[g][6], cmulf(w2, w4));
          v[g][7] = cmulf(v[g][7], cmulf(cmulf(w1, w2), w4));
        }
      }
    }
    if constexpr (R == 8) dft8(v[g]);
    else if constexpr (R == 4) dft4(v[g]);
    else dft2(v[g]);
  }
  __syncthreads();
#pragma unroll
  for (int g = 0; g < GPT; ++g) {
    const int j = threadIdx.x + g * TH;
    if (G < TH && j >= G) break;
    const int jm = j % NS;
    const int base = (j / NS) * NS * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) x[pd(base + r * NS)] = v[g][r];
  }
  __syncthreads();
}

// The fused plans' k_f transform (L = 512, 1024, 2048; 256 threads), the
// same passes as fft_inplace_ct with twiddles computed per butterfly: no
// table load, half the shared memory per CTA.
FC_DEVICE void fft_otf_any(float2* xs, int L) {
  if (L == 2048) {  // 4 * 8^3
    stockham_pass_otf<4, 2048, 1, 256>(xs);
    stockham_pass_otf<8, 2048, 4, 256>(xs);
    stockham_pass_otf<8, 2048, 32, 256>(xs);
    stockham_pass_otf<8, 2048, 256, 256>(xs);
  } else if (L == 1024) {  // 2 * 8^3
    stockham_pass_otf<2, 1024, 1, 256>(xs);
    stockham_pass_otf<8, 1024, 2, 256>(xs);
    stockham_pass_otf<8, 1024, 16, 256>(xs);
    stockham_pass_otf<8, 1024, 128, 256>(xs);
  } else {  // 8^3
    stockham_pass_otf<8, 512, 1, 256>(xs);
    stockham_pass_otf<8, 512, 8, 256>(xs);
    stockham_pass_otf<8, 512, 64, 256>(xs);
  }
}

// shared memory of the FFT kernels: padded data + L twiddles
inline size_t fft_smem_bytes(int64_t L) { return size_t(2 * (L + L / 8)) * sizeof(float2); }
// L float2 from global (16-byte aligned) into the padded layout
FC_DEVICE void load_padded(float2* dst, const float2* src, int L) {
  // 256 threads, L <= 2048: at most 4 16-byte loads per thread, all issued first
  float4 q[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = threadIdx.x + i * 256;
    if (c < L / 2) q[i] = reinterpret_cast<const float4*>(src)[c];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = threadIdx.x + i * 256;
    if (c < L / 2) {
      dst[pd(2 * c)] = make_float2(q[i].x, q[i].y);
      dst[pd(2 * c + 1)] = make_float2(q[i].z, q[i].w);
    }
  }
}

}  // namespace

// Two heads per CTA: both filters are real, so one complex transform of
// z = k_h + i k_{h+1} yields both spectra through the Hermitian split
// K_h[f] = (Z[f] + conj Z[-f]) / 2, K_{h+1}[f] = (Z[f] - conj Z[-f]) / (2i).
__global__ void __launch_bounds__(256) precompute_kf_kernel(const KfParams prm) {
  extern __shared__ float2 sm[];  // padded L data (twiddles per butterfly, fft_otf_any)
  const int64_t h0 = 2 * int64_t(blockIdx.x);
  const bool has1 = h0 + 1 < prm.H;
  const int L = int(prm.L), K = int(prm.K);
  griddep_wait();  // PDL: k is read and k_f written only after the previous kernel
  const float* k0row = prm.k + h0 * K;
  const float* k1row = k0row + K;
  // all of this thread's filter loads are issued before any is stored
  // (L <= 2048 = 8 per thread), so their latencies overlap
  {
    float2 kv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int n = threadIdx.x + i * 256;
      kv[i] = make_float2(0.f, 0.f);
      if (prm.kb) {  // bidirectional: two-sided taps (reading B1)
        if (n < L) kv[i] = make_float2(filter_tap(prm, h0, n), has1 ? filter_tap(prm, h0 + 1, n) : 0.f);
      } else if (n < L && n < K) {
        kv[i] = make_float2(k0row[n], has1 ? k1row[n] : 0.f);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int n = threadIdx.x + i * 256;
      if (n < L) sm[pd(n)] = kv[i];
    }
  }
  __syncthreads();
  fft_otf_any(sm, L);
  const float2* xs = sm;
  // plan layout: row k2 holds pairs (k1, k1 + 1) as {kr, kr', ki, ki'}
  const int L1 = prm.L1, L2 = prm.L2, cpr = L1 / 2;
  const size_t hbytes = size_t(L2) * tab_stride(uint32_t(cpr));
  uint8_t* out0 = reinterpret_cast<uint8_t*>(prm.kf) + h0 * int64_t(hbytes);
  uint8_t* out1 = out0 + hbytes;
  for (int q = threadIdx.x; q < L2 * cpr; q += blockDim.x) {
    // a warp covers 8 consecutive k2 x 4 column pairs: shared-memory reads
    // of consecutive f, 64-byte runs of each output row
    const int w = q >> 5, lane = q & 31;
    const int k2 = (w % (L2 / 8)) * 8 + (lane & 7);
    const int k1 = 2 * ((w / (L2 / 8)) * 4 + (lane >> 3));
    const int f0 = k2 + L2 * k1, f1 = f0 + L2;
    const float2 z0 = xs[pd(f0)], z1 = xs[pd(f1)], m0 = xs[pd((L - f0) & (L - 1))], m1 = xs[pd((L - f1) & (L - 1))];
    float2 a0 = make_float2(0.5f * (z0.x + m0.x), 0.5f * (z0.y - m0.y));
    float2 a1 = make_float2(0.5f * (z1.x + m1.x), 0.5f * (z1.y - m1.y));
    float2 b0 = make_float2(0.5f * (z0.y + m0.y), -0.5f * (z0.x - m0.x));
    float2 b1 = make_float2(0.5f * (z1.y + m1.y), -0.5f * (z1.x - m1.x));
    if (prm.mask) {
      const float w0 = prm.mask[f0], w1 = prm.mask[f1];
      a0.x *= w0; a0.y *= w0; a1.x *= w1; a1.y *= w1;
      b0.x *= w0; b0.y *= w0; b1.x *= w1; b1.y *= w1;
    }
    const uint32_t off = tab_off_rt(uint32_t(cpr), uint32_t(k2), uint32_t(k1 / 2));
    *reinterpret_cast<float4*>(out0 + off) = make_float4(a0.x, a1.x, a0.y, a1.y);
    if (has1) *reinterpret_cast<float4*>(out1 + off) = make_float4(b0.x, b1.x, b0.y, b1.y);
  }
  // PDL: the convolution may start its prologue once every CTA is here (an
  // early trigger let its CTAs take SMs the remaining k_f CTAs needed)
  griddep_launch();
}

// Multipass regime, k_f step 2: one CTA per (head, k0) transforms the L'
// complex values left by step 1 at the start of block (h, k0) and writes the
// inner plan layout of K_f[k0 + L0 f'] over the same block (in place).
__global__ void __launch_bounds__(256) mp_kf_rows_kernel(const KfParams prm, int L0, int Lp, size_t block_bytes) {
  extern __shared__ float2 sm[];  // padded Lp data + Lp twiddles
  const int L = Lp;
  float2* tws = sm + L + L / 8;
  const int64_t blk = blockIdx.x;  // h * L0 + k0
  const int k0 = int(blk % L0);
  uint8_t* block = reinterpret_cast<uint8_t*>(prm.kf) + blk * block_bytes;
  if (prm.row_keep && !prm.row_keep[k0]) {  // masked row: zeros, no transform (the
    // forward pass never reads it; the backward reads finite zeros)
    for (int o = threadIdx.x * 16; o < int(block_bytes); o += blockDim.x * 16)
      *reinterpret_cast<float4*>(block + o) = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  {
    load_padded(tws, prm.twiddle, L);
    // data: 16-byte loads into the padded layout (pd() breaks 16-byte
    // alignment of the shared destination, so no cp.async here)
    load_padded(sm, reinterpret_cast<const float2*>(block), L);
  }
  cp_async_wait_all();
  __syncthreads();
  fft_inplace_any(sm, tws, L);
  const float2* xs = sm;
  const int L1 = prm.L1, L2 = prm.L2, cpr = L1 / 2;
  for (int q = threadIdx.x; q < L2 * cpr; q += blockDim.x) {
    // a warp covers 8 consecutive k2 x 4 column pairs: shared-memory reads
    // of consecutive f, 64-byte runs of each output row
    const int w = q >> 5, lane = q & 31;
    const int k2 = (w % (L2 / 8)) * 8 + (lane & 7);
    const int k1 = 2 * ((w / (L2 / 8)) * 4 + (lane >> 3));
    const int f0 = k2 + L2 * k1, f1 = f0 + L2;
    float2 v0 = xs[pd(f0)], v1 = xs[pd(f1)];
    if (prm.mask) {
      const int64_t kd = row_freq_digit(k0, prm.nlev, prm.lev);
      const float m0 = prm.mask[kd + int64_t(L0) * f0], m1 = prm.mask[kd + int64_t(L0) * f1];
      v0.x *= m0; v0.y *= m0;
      v1.x *= m1; v1.y *= m1;
    }
    *reinterpret_cast<float4*>(block + tab_off_rt(uint32_t(cpr), uint32_t(k2), uint32_t(k1 / 2))) =
        make_float4(v0.x, v1.x, v0.y, v1.y);
  }
}

cudaError_t launch_mp_kf_rows(const KfParams& prm, int L0, int Lp, size_t block_bytes, cudaStream_t s) {
  const size_t smem = fft_smem_bytes(Lp);
  static int attr[64] = {0};
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(mp_kf_rows_kernel), int(smem), attr)) return e;
  mp_kf_rows_kernel<<<unsigned(prm.H * L0), 256, smem, s>>>(prm, L0, Lp, block_bytes);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- dk
// Fused regime: one CTA per head sums the head's per-tile partial spectra in
// tile order (deterministic), applies the mask, and takes
// dk[t] = Re sum_f acc[f] W_L^{-f t} = Re FFT(conj(acc))[t].
// Multipass regime, step 1: the same per (head, k0) over the inner length Lp,
// leaving a[k0][n'] = sum_f' acc[k0 + L0 f'] W_Lp^{-n' f'} (complex) in scratch.
__global__ void __launch_bounds__(256) dk_rows_kernel(const DkParams prm) {
  extern __shared__ float2 sm[];  // padded Lp data + Lp twiddles
  const int L = prm.Lp;
  float2* tws = sm + L + L / 8;
  const int64_t row = blockIdx.x;  // h * L0 + k0
  const int k0 = int(row % prm.L0);
  {
    load_padded(tws, prm.twiddle, L);
  }
  const float2* part = prm.part + row * prm.nbt * L;
  {  // 256 threads, L <= 2048: each thread's 8 columns summed over the tiles in
     // tile order (deterministic), one tile's loads in flight together
    float2 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = make_float2(0.f, 0.f);
    for (int64_t j = 0; j < prm.nbt; ++j) {
      float2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int f = threadIdx.x + i * 256;
        v[i] = f < L ? part[j * L + f] : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) { a[i].x += v[i].x; a[i].y += v[i].y; }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int f = threadIdx.x + i * 256;
      if (f >= L) continue;
      if (prm.mask) {
        const float mk = prm.mask[row_freq_digit(k0, prm.nlev, prm.lev) + int64_t(prm.L0) * f];
        a[i].x *= mk;
        a[i].y *= mk;
      }
      sm[pd(f)] = make_float2(a[i].x, -a[i].y);  // conj: inverse transform via the forward one
    }
  }
  cp_async_wait_all();
  __syncthreads();
  fft_inplace_any(sm, tws, L);
  const float2* xs = sm;
  if (prm.L0 == 1) {
    float* dk = prm.dk + row * prm.K;
    for (int t = threadIdx.x; t < prm.K; t += blockDim.x) dk[t] = xs[pd(t)].x;
    if (prm.dkb)  // bidirectional: lags -t at index L - t (t = 0 shared)
      for (int t = threadIdx.x; t < prm.K; t += blockDim.x) prm.dkb[row * prm.K + t] = xs[pd((L - t) & (L - 1))].x;
  } else {
    float2* a = prm.scratch + row * L;
    for (int t = threadIdx.x; t < L; t += blockDim.x) a[t] = make_float2(xs[pd(t)].x, -xs[pd(t)].y);  // undo conj
  }
}

// Multipass regime, step 2: per (head, n'):
// dk[n' + Lp n0] = Re sum_k0 W_L^{-n' k0} W_L0^{-n0 k0} a[k0][n'],
// i.e. an inverse DFT_L0 (in registers) of the conj-twiddled column.
template <int L0>
__global__ void __launch_bounds__(256) dk_cols_kernel(const DkParams prm) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= prm.H * prm.Lp) return;
  const int n = int(idx % prm.Lp);
  const int64_t h = idx / prm.Lp;
  float2 bw;
  if (prm.wbase) {
    bw = prm.wbase[n];
  } else {  // W_Lfull^{n}, exact dyadic argument
    float sn, cs;
    sincospif(-2.0f * float(n) / float(prm.Lfull), &sn, &cs);
    bw = make_float2(cs, sn);
  }
  float2 tw = make_float2(1.f, 0.f);
  float2 x[L0];
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) x[k0] = prm.scratch[(h * L0 + k0) * prm.Lp + n];
#pragma unroll
  for (int k0 = 0; k0 < L0; ++k0) {
    x[k0] = c_mulc(x[k0], tw);  // a * conj(W_L^{n' k0})
    tw = c_mul(tw, bw);
  }
  DftReg<L0, true>::run(x);  // sum_k0 x[k0] W_L0^{-n0 k0}
#pragma unroll
  for (int n0 = 0; n0 < L0; ++n0) {
    const int64_t t = int64_t(n) + int64_t(n0) * prm.Lp;
    dk_emit(prm, h, t, int64_t(prm.L0) * prm.Lp, ldexpf(x[n0].x, prm.shift2));
  }
}

cudaError_t launch_dk_finalize(const DkParams& prm, cudaStream_t s) {
  if (prm.H <= 0) return cudaSuccess;
  const size_t smem = fft_smem_bytes(prm.Lp);
  static int attr[64] = {0};
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(dk_rows_kernel), int(smem), attr)) return e;
  dk_rows_kernel<<<unsigned(prm.H * prm.L0), 256, smem, s>>>(prm);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || prm.L0 == 1) return e;
  DkParams c = prm;
  if (prm.nlev > 1) {  // invert the deeper levels in place, deepest first
    for (int l = prm.nlev - 1; l >= 1; --l) {
      int64_t rows = prm.H, Lrow = prm.Lfull;
      for (int j = 0; j < l; ++j) { rows *= prm.lev_L0[j]; Lrow /= prm.lev_L0[j]; }
      e = launch_mp_cols_inverse(prm.scratch, prm.lev_L0[l], rows, Lrow, s);
      if (e != cudaSuccess) return e;
    }
    c.L0 = prm.lev_L0[0];
    c.Lp = int32_t(prm.Lfull / prm.lev_L0[0]);
    c.wbase = nullptr;
  }
  const unsigned grid = unsigned((c.H * c.Lp + 255) / 256);
  switch (c.L0) {
    case 2: dk_cols_kernel<2><<<grid, 256, 0, s>>>(c); break;
    case 4: dk_cols_kernel<4><<<grid, 256, 0, s>>>(c); break;
    case 8: dk_cols_kernel<8><<<grid, 256, 0, s>>>(c); break;
    case 16: dk_cols_kernel<16><<<grid, 256, 0, s>>>(c); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Single-pass order-3 plans (fft_size LF = L0 * 2048, L0 = 2, 4, 8): two
// heads per CTA (one complex FFT of k_h + i k_{h+1}, Hermitian split), the
// LF-point Stockham transform in shared memory (data only, 37 / 74 / 147 KB)
// with twiddles W_LF^e computed per butterfly (sincospif of the exact dyadic
// argument -2e/LF), 512 / 1024 / 1024 threads, written as L0 blocks per head:
// block k0 holds K_f[f' + 2048 k0], f' = k2 + 64 k1, in the layout of
// layout.h dit_kf_off (DIT order: the forward kernel's outer DFT produces the
// frequency digit k0 = f / 2048).  (Round 2 sessions 1-2: 256 threads and a
// twiddle table, 4096 / 8192 only; fft_size 16384 went through the multipass
// transforms plus a re-layout, 202 us per step at N = 8192, now ~77 us.)
template <int LF>
constexpr int dit_threads() { return LF == 4096 ? 512 : 1024; }
template <int LF>
__global__ void __launch_bounds__(dit_threads<LF>()) precompute_kf_dit_kernel(const KfParams prm) {
  extern __shared__ float2 sm[];  // padded LF data
  constexpr int TH = dit_threads<LF>();
  const int64_t h0 = 2 * int64_t(blockIdx.x);
  const bool has1 = h0 + 1 < prm.H;
  const int K = int(prm.K);
  griddep_wait();  // PDL: k is read and k_f written only after the previous kernel
  const float* k0row = prm.k + h0 * K;
  const float* k1row = k0row + K;
  for (int n = threadIdx.x; n < LF; n += TH)
    sm[pd(n)] = prm.kb ? make_float2(filter_tap(prm, h0, n), has1 ? filter_tap(prm, h0 + 1, n) : 0.f)
              : n < K  ? make_float2(k0row[n], has1 ? k1row[n] : 0.f)
                       : make_float2(0.f, 0.f);
  __syncthreads();
  if constexpr (LF == 4096) {  // 8^4
    stockham_pass_otf<8, LF, 1, TH>(sm);
    stockham_pass_otf<8, LF, 8, TH>(sm);
    stockham_pass_otf<8, LF, 64, TH>(sm);
    stockham_pass_otf<8, LF, 512, TH>(sm);
  } else if constexpr (LF == 8192) {  // 2 * 8^4
    stockham_pass_otf<2, LF, 1, TH>(sm);
    stockham_pass_otf<8, LF, 2, TH>(sm);
    stockham_pass_otf<8, LF, 16, TH>(sm);
    stockham_pass_otf<8, LF, 128, TH>(sm);
    stockham_pass_otf<8, LF, 1024, TH>(sm);
  } else {  // 4 * 8^4
    static_assert(LF == 16384, "order-3 k_f sizes");
    stockham_pass_otf<4, LF, 1, TH>(sm);
    stockham_pass_otf<8, LF, 4, TH>(sm);
    stockham_pass_otf<8, LF, 32, TH>(sm);
    stockham_pass_otf<8, LF, 256, TH>(sm);
    stockham_pass_otf<8, LF, 2048, TH>(sm);
  }
  const float2* xs = sm;
  constexpr int L0 = LF / 2048, CPR = 16;
  const size_t hbytes = size_t(64) * tab_stride(CPR);
  uint8_t* out0 = reinterpret_cast<uint8_t*>(prm.kf) + h0 * int64_t(L0 * hbytes);
  uint8_t* out1 = out0 + L0 * hbytes;
  for (int q = threadIdx.x; q < L0 * 64 * CPR; q += TH) {  // one destination float4 per step, k2 fastest
    const int b = q >> 10, d = q & 1023;
    const int kp = (d >> 8) * 4 + (d & 3), k2 = (d >> 2) & 63;
    const int f0 = k2 + 64 * (2 * kp) + 2048 * b, f1 = f0 + 64;
    const float2 z0 = xs[pd(f0)], z1 = xs[pd(f1)], m0 = xs[pd((LF - f0) & (LF - 1))], m1 = xs[pd((LF - f1) & (LF - 1))];
    // Hermitian split (1/2) and the forward kernel's 1/L0 of the outer
    // inverse DFT, folded here (an exact power of two)
    constexpr float hs = 0.5f / float(L0);
    const float2 a0 = make_float2(hs * (z0.x + m0.x), hs * (z0.y - m0.y));
    const float2 a1 = make_float2(hs * (z1.x + m1.x), hs * (z1.y - m1.y));
    const float2 b0 = make_float2(hs * (z0.y + m0.y), -hs * (z0.x - m0.x));
    const float2 b1 = make_float2(hs * (z1.y + m1.y), -hs * (z1.x - m1.x));
    const uint32_t off = uint32_t(b * hbytes) + dit_kf_off(uint32_t(k2), uint32_t(kp));
    *reinterpret_cast<float4*>(out0 + off) = make_float4(a0.x, a1.x, a0.y, a1.y);
    if (has1) *reinterpret_cast<float4*>(out1 + off) = make_float4(b0.x, b1.x, b0.y, b1.y);
  }
  griddep_launch();
}

cudaError_t launch_precompute_kf_dit(const KfParams& prm, int L0, cudaStream_t s) {
  if (prm.H <= 0) return cudaSuccess;
  const unsigned grid = unsigned((prm.H + 1) / 2);
  static int attr[3][64] = {};
  auto go = [&](auto kern, int LF, int th, int* cache) -> cudaError_t {
    const size_t smem = size_t(LF + LF / 8) * sizeof(float2);
    if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(smem), cache)) return e;
    return launch_pdl(PDL_KF, kern, dim3(grid), dim3(th), smem, s, prm);
  };
  if (L0 == 2) return go(precompute_kf_dit_kernel<4096>, 4096, dit_threads<4096>(), attr[0]);
  if (L0 == 4) return go(precompute_kf_dit_kernel<8192>, 8192, dit_threads<8192>(), attr[1]);
  if (L0 == 8) return go(precompute_kf_dit_kernel<16384>, 16384, dit_threads<16384>(), attr[2]);
  return cudaErrorInvalidValue;
}

// The backward of an order-3 plan runs the multipass path, whose k_f layout
// is L0 blocks per head with block k0 = K_f[k0 + L0 f']: gather it from the
// order-3 layout (block f / 2048 at f % 2048), one float4 {re, re', im, im'}
// of the destination per thread.
__global__ void kf_dit_to_dif_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t H, int L0) {
  constexpr int CPR = 16;
  const size_t hb = size_t(64) * tab_stride(CPR);
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per_head = int64_t(L0) * 64 * CPR;
  if (idx >= H * per_head) return;
  const int64_t h = idx / per_head;
  const int rem = int(idx % per_head);
  const int k0 = rem / (64 * CPR), k2 = (rem % (64 * CPR)) / CPR, kp = rem % CPR;
  float v[4];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int f = k0 + L0 * (k2 + 64 * (2 * kp + s));
    const int b = f / 2048, g = f % 2048;
    const int k2s = g % 64, k1s = g / 64;
    const float4 q = *reinterpret_cast<const float4*>(src + (h * L0 + b) * hb + dit_kf_off(uint32_t(k2s), uint32_t(k1s / 2)));
    v[s] = float(L0) * ((k1s & 1) ? q.y : q.x);  // (undo the 1/L0 the order-3 layout carries)
    v[2 + s] = float(L0) * ((k1s & 1) ? q.w : q.z);
  }
  *reinterpret_cast<float4*>(dst + (h * L0 + k0) * hb + tab_off_rt(CPR, uint32_t(k2), uint32_t(kp))) =
      make_float4(v[0], v[1], v[2], v[3]);
}

cudaError_t launch_kf_dit_to_dif(const void* src, void* dst, int64_t H, int L0, cudaStream_t s) {
  const int64_t n = H * int64_t(L0) * 64 * 16;
  if (n == 0) return cudaSuccess;
  kf_dit_to_dif_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(static_cast<const uint8_t*>(src),
                                                                 static_cast<uint8_t*>(dst), H, L0);
  return cudaGetLastError();
}

cudaError_t launch_precompute_kf(const KfParams& prm, cudaStream_t s) {
  if (prm.H <= 0) return cudaSuccess;
  const size_t smem = size_t(prm.L + prm.L / 8) * sizeof(float2);
  static int attr[64] = {0};
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(precompute_kf_kernel), int(smem), attr)) return e;
  return launch_pdl(PDL_KF, precompute_kf_kernel, dim3(unsigned((prm.H + 1) / 2)), dim3(256), smem, s, prm);
}

}  // namespace fc
