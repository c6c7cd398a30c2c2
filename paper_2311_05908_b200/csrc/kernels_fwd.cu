// kernels_fwd.cu -- fused single-pass FFT convolution on sm_100a (tcgen05).
//
// One CTA processes "tiles" of P row pairs that share a head h.  Each pair
// (b, b+1) is packed as one complex sequence z = g_b + i g_{b+1} (two real
// rows per complex transform -- the real-to-complex packing of P:253-254,
// realised here by pairing rows instead of the one-stage DIT split of
// Appendix A.1).  Because k is
// real, conv(z, k) = conv(g_b, k) + i conv(g_{b+1}, k), so the output pair is
// read back from the real and imaginary parts.
//
// The length-L transform (L = fft_size) is an order-2 Monarch decomposition
// (Alg. 1) with L = L1 * L2, n = n1 + L1 n2,
// f = k2 + L2 k1:
//   stage A   : contract n2 -> k2 (DFT_L2)       [first half of n2 only when
//               causal: the zero padding is never loaded, P:255-256]
//   twiddle   : * W_L^{n1 k2}
//   stage B   : contract n1 -> k1 (DFT_L1)
//   pointwise : * k_f[k2 + L2 k1]
//   stage B^-1: contract k1 -> n1 (IDFT_L1)
//   twiddle   : * W_L^{-n1 k2}
//   stage A^-1: contract k2 -> n2 (IDFT_L2)       [only n2 < L2/2 stored
//               when causal]
// Every stage is one or more tcgen05.mma.kind::f16 (fp16 operands, fp32
// accumulators in TMEM); complex arithmetic is a real-pair GEMM with the
// real/imag planes stacked in K.  The elementwise steps between stages run
// on TMEM -> registers -> shared memory, where the write layout performs the
// "permutation as transpose" of P:226-234 for free: each stage's operand is
// written directly in the canonical UMMA layout (MN-major or K-major) the next
// MMA reads.  Gating (u*w on load, *v on store) is fused.
#include <cuda_runtime.h>

#include "fwd_params.h"
#include "sm100.cuh"

namespace fc {

template <typename T>
struct IO;
template <>
struct IO<__half> {
  static FC_DEVICE void to_f32x8(const uint4& v, float* f) {
    const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __half22float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  static FC_DEVICE uint32_t pack2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};
template <>
struct IO<__nv_bfloat16> {
  static FC_DEVICE void to_f32x8(const uint4& v, float* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  static FC_DEVICE uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

template <int L1, bool CAUSAL>
struct O2Cfg {
  static constexpr int L2 = 64;
  static constexpr int L = L1 * L2;
  static constexpr int P = 128 / L1;            // row pairs per tile
  static constexpr int R = 2 * P;               // batch rows per tile
  static constexpr int KA = CAUSAL ? L2 / 2 : L2;
  static constexpr int NOUT = CAUSAL ? L / 2 : L;  // row length N
  static constexpr int CH = NOUT / 8;           // 16-byte chunks per row (16-bit I/O)
  // tables (same offsets as the host image, see plan.cpp)
  static constexpr uint32_t GA_BYTES = 2 * L2 * 2 * KA * 2;
  static constexpr uint32_t GB_BYTES = 2 * L1 * 2 * L1 * 2;
  static constexpr uint32_t GAI_BYTES = 2 * L2 * 2 * L2 * 2;
  static constexpr uint32_t TW_BYTES = L * 8;
  static constexpr uint32_t al(uint32_t x) { return (x + 1023u) / 1024u * 1024u; }
  static constexpr uint32_t OFF_GA = 0;
  static constexpr uint32_t OFF_GB = al(OFF_GA + GA_BYTES);
  static constexpr uint32_t OFF_GBI = al(OFF_GB + GB_BYTES);
  static constexpr uint32_t OFF_GAI = al(OFF_GBI + GB_BYTES);
  static constexpr uint32_t OFF_TW = al(OFF_GAI + GAI_BYTES);
  static constexpr uint32_t TABLES = al(OFF_TW + TW_BYTES);
  // working buffers
  static constexpr uint32_t KF_BYTES = L * 8;
  static constexpr uint32_t BUFA_BYTES = 128 * 2 * KA * 2;     // stage A operand
  static constexpr uint32_t BUFX_BYTES = P * L * 4;            // complex fp16 per tile
  static constexpr bool STAGE = CAUSAL;                        // cp.async prefetch staging
  static constexpr uint32_t ST_BYTES = STAGE ? R * NOUT * 2 : 0;
  static constexpr uint32_t OFF_KF = TABLES;
  static constexpr uint32_t OFF_BUFA = al(OFF_KF + KF_BYTES);
  static constexpr uint32_t OFF_BUFX = al(OFF_BUFA + BUFA_BYTES);
  static constexpr uint32_t OFF_STU = al(OFF_BUFX + BUFX_BYTES);
  static constexpr uint32_t OFF_STW = al(OFF_STU + ST_BYTES);
  static constexpr uint32_t SMEM = al(OFF_STW + ST_BYTES) + 1024;  // + alignment slack
  // operand strides
  static constexpr uint32_t SBO_A = (2 * KA / 8) * 128;   // bufA: MN-group stride (K groups contiguous)
  static constexpr uint32_t LBO_B = (P * L2 / 8) * 128;   // epi1 -> stage B (MN-major, K-group stride)
  static constexpr uint32_t SBO_BP = (2 * L1 / 8) * 128;  // epi2 -> stage B^-1 (K-major, row-group stride)
  static constexpr uint32_t SBO_GB = (2 * L1 / 8) * 128;  // G_B / G_B^-1 row-group stride
  static constexpr uint32_t SBO_GA = (2 * KA / 8) * 128;
  static constexpr uint32_t SBO_GAI = (2 * L2 / 8) * 128;
  static constexpr uint32_t SBO_XA = (2 * L2 / 8) * 128;  // epi3 -> stage A^-1 (MN-major B, N-group stride)
  static_assert(P * L1 == 128, "stage A covers one 128-row MMA group");
  static_assert(P % 2 == 0, "stage B groups hold two pairs");
};

// Complex multiply helpers (fp32).
FC_DEVICE void cmul(float& xr, float& xi, float wr, float wi) {
  float r = xr * wr - xi * wi;
  float i = xr * wi + xi * wr;
  xr = r;
  xi = i;
}
FC_DEVICE void cmulc(float& xr, float& xi, float wr, float wi) {  // x * conj(w)
  float r = xr * wr + xi * wi;
  float i = xi * wr - xr * wi;
  xr = r;
  xi = i;
}

template <int L1, bool CAUSAL, bool GATED, typename T>
__global__ void __launch_bounds__(128, 1) fftconv_fwd_o2_kernel(const FwdParams prm) {
  using C = O2Cfg<L1, CAUSAL>;
  constexpr int L2 = C::L2;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t mma_bar;
  __shared__ uint32_t tmem_slot;
  // 1024-aligned base
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sGA = base + C::OFF_GA, sGB = base + C::OFF_GB, sGBI = base + C::OFF_GBI,
                 sGAI = base + C::OFF_GAI, sTW = base + C::OFF_TW, sKF = base + C::OFF_KF,
                 bufA = base + C::OFF_BUFA, bufX = base + C::OFF_BUFX, stU = base + C::OFF_STU,
                 stW = base + C::OFF_STW;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t B = prm.B, H = prm.H, N = prm.N;
  const int64_t nbt = (B + C::R - 1) / C::R;
  const int64_t tiles = H * nbt;
  const int64_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  if (t0 >= t1) return;

  const T* __restrict__ gu = reinterpret_cast<const T*>(prm.u);
  const T* __restrict__ gw = reinterpret_cast<const T*>(prm.w);
  const T* __restrict__ gv = reinterpret_cast<const T*>(prm.v);
  T* __restrict__ gy = reinterpret_cast<T*>(prm.y);
  const uint8_t* __restrict__ gkf = reinterpret_cast<const uint8_t*>(prm.kf);

  // ---- one-time setup: tables -> smem, barrier, TMEM
  {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(prm.tables);
    for (uint32_t o = tid * 16; o < C::TABLES; o += 128 * 16) cp_async16(base + o, src + o, true);
    cp_async_commit();
  }
  if (tid == 0) {
    mbar_init(&mma_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<128>(&tmem_slot);

  // ---- input staging (cp.async prefetch) of tile t
  auto issue_input = [&](int64_t t) {
    const int64_t h = t / nbt, bt = t % nbt;
    for (int q = tid; q < C::R * C::CH; q += 128) {
      const int r = q / C::CH, pos = q % C::CH;
      const int64_t b = bt * C::R + r;
      const bool ok = b < B;
      const int64_t goff = ((ok ? b : 0) * H + h) * N + int64_t(pos) * 8;
      const uint32_t so = swz128(uint32_t(q) * 16);
      cp_async16(stU + so, gu + goff, ok);
      if (GATED) cp_async16(stW + so, gw + goff, ok);
    }
    cp_async_commit();
  };

  // ---- staging (or global) -> bufA, gating u*w, fp16 operand
  auto convert_input = [&](int64_t t) {
    const int64_t h = t / nbt, bt = t % nbt;
    constexpr int KROWS = C::KA;                 // n2 rows per row
    constexpr int JC = L1 / 8;                   // 8-element n1 chunks
    for (int q = tid; q < C::R * C::CH; q += 128) {
      // n2 fastest so 8 consecutive threads fill one 128 B core matrix
      const int n2 = q % KROWS;
      const int j = (q / KROWS) % JC;
      const int r = q / (KROWS * JC);
      const int pos = n2 * JC + j;  // chunk index in the row (n = 8*pos)
      float g[8];
      if (C::STAGE) {
        const uint32_t so = swz128(uint32_t(r * C::CH + pos) * 16);
        uint4 uv = ld_shared_u4(stU + so);
        IO<T>::to_f32x8(uv, g);
        if (GATED) {
          float wv[8];
          IO<T>::to_f32x8(ld_shared_u4(stW + so), wv);
#pragma unroll
          for (int e = 0; e < 8; ++e) g[e] *= wv[e];
        }
      } else {
        const int64_t b = bt * C::R + r;
        if (b < B) {
          const int64_t goff = (b * H + h) * N + int64_t(pos) * 8;
          uint4 uv = *reinterpret_cast<const uint4*>(gu + goff);
          IO<T>::to_f32x8(uv, g);
          if (GATED) {
            float wv[8];
            IO<T>::to_f32x8(*reinterpret_cast<const uint4*>(gw + goff), wv);
#pragma unroll
            for (int e = 0; e < 8; ++e) g[e] *= wv[e];
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) g[e] = 0.f;
        }
      }
      const int p = r >> 1, c = r & 1;
      const int mg = p * JC + j;
      const int k = c * C::KA + n2;
      const uint32_t off = mg * C::SBO_A + (k >> 3) * 128 + (k & 7) * 16;
      st_shared_v4(bufA + off, pack_half2(g[0], g[1]), pack_half2(g[2], g[3]), pack_half2(g[4], g[5]),
                   pack_half2(g[6], g[7]));
    }
  };

  cp_async_wait_all();
  if (C::STAGE) issue_input(t0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  uint32_t phase = 0;
  int64_t cur_h = -1;

  auto sync_and_issue = [&](auto&& issue) {
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      issue();
      mma_commit(&mma_bar);
    }
    mbar_wait(&mma_bar, phase);
    phase ^= 1;
    tc_fence_after();
  };

  for (int64_t t = t0; t < t1; ++t) {
    const int64_t h = t / nbt, bt = t % nbt;
    if (h != cur_h) {
      const uint8_t* src = gkf + h * int64_t(C::KF_BYTES);
      for (uint32_t o = tid * 16; o < C::KF_BYTES; o += 128 * 16) cp_async16(sKF + o, src + o, true);
      cp_async_commit();
      cur_h = h;
    }
    cp_async_wait_all();
    __syncthreads();
    convert_input(t);
    if (C::STAGE && t + 1 < t1) {
      __syncthreads();  // everyone finished reading the staging buffers
      issue_input(t + 1);
    }

    // ---------------- stage A: D[(p,n1)][(c',k2)] = X[(p,n1)][(c,n2)] * G_A
    sync_and_issue([&] {
      constexpr uint32_t idesc = idesc_f16(128, 2 * L2, true, false);
#pragma unroll
      for (int s = 0; s < 2 * C::KA / 16; ++s) {
        uint64_t ad = smem_desc(bufA + 256 * s, 128, C::SBO_A);
        uint64_t bd = smem_desc(sGA + 256 * s, 128, C::SBO_GA);
        mma_f16_ss(tmem, ad, bd, idesc, s > 0);
      }
    });

    // ---------------- epilogue 1: twiddle, transpose -> stage B operand (MN-major)
    {
      const int m = tid, p = m / L1, n1 = m % L1;
#pragma unroll 1
      for (int k2c = 0; k2c < L2 / 8; ++k2c) {
        float re[8], im[8];
        tmem_ld8(tmem + lane_base + k2c * 8, re);
        tmem_ld8(tmem + lane_base + L2 + k2c * 8, im);
        tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          float4 w = ld_shared_f4(sTW + swz128(uint32_t(n1 * L2 + k2c * 8 + 2 * jj) * 8));
          cmul(re[2 * jj], im[2 * jj], w.x, w.y);
          cmul(re[2 * jj + 1], im[2 * jj + 1], w.z, w.w);
        }
        const int mg = p * (L2 / 8) + k2c;
        const uint32_t o_re = mg * 128 + (n1 >> 3) * C::LBO_B + (n1 & 7) * 16;
        const uint32_t o_im = mg * 128 + ((L1 + n1) >> 3) * C::LBO_B + (n1 & 7) * 16;
        st_shared_v4(bufX + o_re, pack_half2(re[0], re[1]), pack_half2(re[2], re[3]), pack_half2(re[4], re[5]),
                     pack_half2(re[6], re[7]));
        st_shared_v4(bufX + o_im, pack_half2(im[0], im[1]), pack_half2(im[2], im[3]), pack_half2(im[4], im[5]),
                     pack_half2(im[6], im[7]));
      }
    }

    // ---------------- stage B: per group of 128 rows (p,k2), contract n1 -> k1
    sync_and_issue([&] {
      constexpr uint32_t idesc = idesc_f16(128, 2 * L1, true, false);
#pragma unroll 1
      for (int gi = 0; gi < C::P / 2; ++gi) {
#pragma unroll
        for (int s = 0; s < 2 * L1 / 16; ++s) {
          uint64_t ad = smem_desc(bufX + gi * 2048 + 2 * s * C::LBO_B, C::LBO_B, 128);
          uint64_t bd = smem_desc(sGB + 256 * s, 128, C::SBO_GB);
          mma_f16_ss(tmem + gi * 2 * L1, ad, bd, idesc, s > 0);
        }
      }
    });

    // ---------------- epilogue 2: pointwise * k_f -> stage B^-1 operand (K-major)
#pragma unroll 1
    for (int gi = 0; gi < C::P / 2; ++gi) {
      const int m = tid, k2 = m & 63;
      const int row = gi * 128 + m;  // (p, k2) with p = 2 gi + m / 64
#pragma unroll 1
      for (int k1c = 0; k1c < L1 / 8; ++k1c) {
        float re[8], im[8];
        tmem_ld8(tmem + lane_base + gi * 2 * L1 + k1c * 8, re);
        tmem_ld8(tmem + lane_base + gi * 2 * L1 + L1 + k1c * 8, im);
        tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          float4 kf = ld_shared_f4(sKF + swz128(uint32_t(k2 * L1 + k1c * 8 + 2 * jj) * 8));
          cmul(re[2 * jj], im[2 * jj], kf.x, kf.y);
          cmul(re[2 * jj + 1], im[2 * jj + 1], kf.z, kf.w);
        }
        const uint32_t o_re = (row >> 3) * C::SBO_BP + k1c * 128 + (row & 7) * 16;
        const uint32_t o_im = (row >> 3) * C::SBO_BP + (L1 / 8 + k1c) * 128 + (row & 7) * 16;
        st_shared_v4(bufX + o_re, pack_half2(re[0], re[1]), pack_half2(re[2], re[3]), pack_half2(re[4], re[5]),
                     pack_half2(re[6], re[7]));
        st_shared_v4(bufX + o_im, pack_half2(im[0], im[1]), pack_half2(im[2], im[3]), pack_half2(im[4], im[5]),
                     pack_half2(im[6], im[7]));
      }
    }

    // ---------------- stage B^-1: contract k1 -> n1
    sync_and_issue([&] {
      constexpr uint32_t idesc = idesc_f16(128, 2 * L1, false, false);
#pragma unroll 1
      for (int gi = 0; gi < C::P / 2; ++gi) {
#pragma unroll
        for (int s = 0; s < 2 * L1 / 16; ++s) {
          uint64_t ad = smem_desc(bufX + gi * 16 * C::SBO_BP + 256 * s, 128, C::SBO_BP);
          uint64_t bd = smem_desc(sGBI + 256 * s, 128, C::SBO_GB);
          mma_f16_ss(tmem + gi * 2 * L1, ad, bd, idesc, s > 0);
        }
      }
    });

    // ---------------- epilogue 3: conj twiddle, transpose -> stage A^-1 operand (MN-major B)
#pragma unroll 1
    for (int gi = 0; gi < C::P / 2; ++gi) {
      const int m = tid, k2 = m & 63;
      const int p = gi * 2 + (m >> 6);
#pragma unroll 1
      for (int n1c = 0; n1c < L1 / 8; ++n1c) {
        float re[8], im[8];
        tmem_ld8(tmem + lane_base + gi * 2 * L1 + n1c * 8, re);
        tmem_ld8(tmem + lane_base + gi * 2 * L1 + L1 + n1c * 8, im);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int n1 = n1c * 8 + e;
          float2 w = ld_shared_f2(sTW + swz128(uint32_t(n1 * L2 + k2) * 8));
          cmulc(re[e], im[e], w.x, w.y);
        }
        const int ng = (p * L1) / 8 + n1c;
        const uint32_t o_re = ng * C::SBO_XA + (k2 >> 3) * 128 + (k2 & 7) * 16;
        const uint32_t o_im = ng * C::SBO_XA + ((L2 + k2) >> 3) * 128 + (k2 & 7) * 16;
        st_shared_v4(bufX + o_re, pack_half2(re[0], re[1]), pack_half2(re[2], re[3]), pack_half2(re[4], re[5]),
                     pack_half2(re[6], re[7]));
        st_shared_v4(bufX + o_im, pack_half2(im[0], im[1]), pack_half2(im[2], im[3]), pack_half2(im[4], im[5]),
                     pack_half2(im[6], im[7]));
      }
    }

    // ---------------- stage A^-1: D[(c',n2)][(p,n1)] = G_A^-1 * X[(c,k2)][(p,n1)]
    sync_and_issue([&] {
      constexpr uint32_t idesc = idesc_f16(128, 128, false, true);
#pragma unroll
      for (int s = 0; s < 2 * L2 / 16; ++s) {
        uint64_t ad = smem_desc(sGAI + 256 * s, 128, C::SBO_GAI);
        uint64_t bd = smem_desc(bufX + 256 * s, 128, C::SBO_XA);
        mma_f16_ss(tmem, ad, bd, idesc, s > 0);
      }
    });

    // ---------------- epilogue 4: (gate), convert, store y
    {
      const int m = tid, cp = m >> 6, n2 = m & 63;
      if (!CAUSAL || n2 < L2 / 2) {  // warp-uniform
#pragma unroll 1
        for (int p = 0; p < C::P; ++p) {
          const int64_t b = bt * C::R + 2 * p + cp;
          if (b >= B) continue;  // warp-uniform
          const int64_t goff = (b * H + h) * N + int64_t(L1) * n2;
#pragma unroll
          for (int n1c = 0; n1c < L1 / 8; ++n1c) {
            float o[8];
            tmem_ld8(tmem + lane_base + p * L1 + n1c * 8, o);
            tmem_ld_wait();
            if (GATED) {
              float vv[8];
              IO<T>::to_f32x8(*reinterpret_cast<const uint4*>(gv + goff + n1c * 8), vv);
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] *= vv[e];
            }
            uint4 st;
            st.x = IO<T>::pack2(o[0], o[1]);
            st.y = IO<T>::pack2(o[2], o[3]);
            st.z = IO<T>::pack2(o[4], o[5]);
            st.w = IO<T>::pack2(o[6], o[7]);
            *reinterpret_cast<uint4*>(gy + goff + n1c * 8) = st;
          }
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem);
}

// ------------------------------------------------------------------ launch
template <int L1, bool CAUSAL, bool GATED, typename T>
static cudaError_t launch_o2(const FwdParams& prm, cudaStream_t stream) {
  using C = O2Cfg<L1, CAUSAL>;
  auto kern = fftconv_fwd_o2_kernel<L1, CAUSAL, GATED, T>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int64_t nbt = (prm.B + C::R - 1) / C::R;
  const int64_t tiles = prm.H * nbt;
  int grid = int(tiles < prm.num_sms ? tiles : prm.num_sms);
  if (grid < 1) return cudaSuccess;
  kern<<<grid, 128, C::SMEM, stream>>>(prm);
  return cudaGetLastError();
}

template <bool CAUSAL, bool GATED, typename T>
static cudaError_t dispatch_l1(const FwdParams& prm, cudaStream_t s) {
  switch (prm.L1) {
    case 8: return launch_o2<8, CAUSAL, GATED, T>(prm, s);
    case 16: return launch_o2<16, CAUSAL, GATED, T>(prm, s);
    case 32: return launch_o2<32, CAUSAL, GATED, T>(prm, s);
    default: return cudaErrorInvalidValue;
  }
}

template <bool CAUSAL, bool GATED>
static cudaError_t dispatch_t(const FwdParams& prm, cudaStream_t s) {
  if (prm.dtype == 0) return dispatch_l1<CAUSAL, GATED, __half>(prm, s);
  return dispatch_l1<CAUSAL, GATED, __nv_bfloat16>(prm, s);
}

cudaError_t launch_fwd_fused(const FwdParams& prm, cudaStream_t s) {
  if (prm.causal) return prm.gated ? dispatch_t<true, true>(prm, s) : dispatch_t<true, false>(prm, s);
  return prm.gated ? dispatch_t<false, true>(prm, s) : dispatch_t<false, false>(prm, s);
}

size_t fwd_fused_smem_bytes(int L1, int causal) {
  switch (L1 * 2 + (causal ? 1 : 0)) {
    case 17: return O2Cfg<8, true>::SMEM;
    case 16: return O2Cfg<8, false>::SMEM;
    case 33: return O2Cfg<16, true>::SMEM;
    case 32: return O2Cfg<16, false>::SMEM;
    case 65: return O2Cfg<32, true>::SMEM;
    case 64: return O2Cfg<32, false>::SMEM;
  }
  return 0;
}

}  // namespace fc
