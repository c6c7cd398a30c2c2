// fused_common.cuh -- pieces shared by the fused forward and backward
// order-2 kernels: I/O conversions, the tile configuration (shared-memory
// table offsets must match the host image built in plan.cpp), operand store
// helpers and the f32x2 complex multiplies.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

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

constexpr int kWGThreads = 256;        // 8 warps: 4 TMEM lane quadrants x 2 column slices

template <int L1, bool CAUSAL>
struct O2Cfg {
  static constexpr int L2 = 64;
  static constexpr int L = L1 * L2;
  static constexpr int P = 128 / L1;            // row pairs per tile
  static constexpr int R = 2 * P;               // batch rows per tile
  static constexpr int KA = CAUSAL ? L2 / 2 : L2;
  static constexpr int NOUT = CAUSAL ? L / 2 : L;  // row length N
  static constexpr int CH = NOUT / 8;           // 16-byte chunks per row (16-bit I/O)
  // stage A N: re | im (the -im plane is negated in registers)
  static constexpr bool NEG_A = false;
  static constexpr int NA = 2 * L2;
  static constexpr int NB = (3 * L1 + 15) / 16 * 16;  // stage B/B^-1 N: re | im | -im (-re) | pad
  // table image (same offsets as plan.cpp): GA | GB | GBI | TW | GAI | TWT.
  // The forward kernel copies the prefix through GAI's first GAI_FWD bytes
  // (causal: the rows n2 < L2/2 only); the backward copies everything.
  static constexpr uint32_t GA_BYTES = NA * 2 * KA * 2;
  static constexpr uint32_t GB_BYTES = NB * 2 * L1 * 2;
  static constexpr uint32_t GAI_BYTES = 2 * L2 * 2 * L2 * 2;
  static constexpr uint32_t GAI_FWD_BYTES = (CAUSAL ? L2 : 2 * L2) * 2 * L2 * 2;
  static constexpr uint32_t TW_BYTES = L1 * (L2 / 2 * 16 + 16);    // padded rows, see layout.h
  static constexpr uint32_t TWT_BYTES = L2 * (L1 / 2 * 16 + 16);
  static constexpr uint32_t al(uint32_t x) { return (x + 1023u) / 1024u * 1024u; }
  static constexpr uint32_t OFF_GA = 0;
  static constexpr uint32_t OFF_GB = al(OFF_GA + GA_BYTES);
  static constexpr uint32_t OFF_GBI = al(OFF_GB + GB_BYTES);
  static constexpr uint32_t OFF_TW = al(OFF_GBI + GB_BYTES);    // [n1][k2/2] {wr,wr',wi,wi'}
  static constexpr uint32_t OFF_GAI = al(OFF_TW + TW_BYTES);
  static constexpr uint32_t OFF_TWT = al(OFF_GAI + GAI_BYTES);  // [k2][n1/2] {wr,wr',wi,wi'}
  static constexpr uint32_t TABLES = al(OFF_TWT + TWT_BYTES);
  static constexpr uint32_t TABLES_FWD = al(OFF_GAI + GAI_FWD_BYTES);
  // per-warpgroup working buffers
  static constexpr uint32_t KF_BYTES = L2 * (L1 / 2 * 16 + 16); // [k2][k1/2] {kr,kr',ki,ki'}, padded rows
  static constexpr uint32_t BUFX_BYTES = P * L * 4;            // complex fp16 per tile (stage A operand aliases it)
  static constexpr uint32_t WG_BYTES = al(KF_BYTES) + al(BUFX_BYTES);
  // operand strides
  static constexpr uint32_t SBO_A = (2 * KA / 8) * 128;   // stage A operand: MN-group stride (K groups contiguous)
  static constexpr uint32_t LBO_B = (P * L2 / 8) * 128;   // epi1 -> stage B (MN-major, K-group stride)
  static constexpr uint32_t SBO_BP = (2 * L1 / 8) * 128;  // epi2 -> stage B^-1 (K-major, row-group stride)
  static constexpr uint32_t SBO_GB = (2 * L1 / 8) * 128;  // G_B / G_B^-1 row-group stride
  static constexpr uint32_t SBO_GA = (2 * KA / 8) * 128;
  static constexpr uint32_t SBO_GAI = (2 * L2 / 8) * 128;
  static constexpr uint32_t SBO_XA = (2 * L2 / 8) * 128;  // epi3 -> stage A^-1 (MN-major B, N-group stride)
  static constexpr uint32_t TMEM_COLS = 256;              // per warpgroup
  // stage B^-1 reads its data operand from TMEM (epilogue 2 writes it into
  // its own lanes: 2*L1 fp16 = L1 columns per 128-row group) when those
  // columns fit beside stage B's accumulators; else from shared memory
  static constexpr uint32_t TS_COLS = (P / 2) * L1;
  static constexpr bool TS_BI = (P / 2) * NB + TS_COLS <= TMEM_COLS;
  static constexpr uint32_t CA = TMEM_COLS - TS_COLS;     // first column of that operand
  static_assert(P * L1 == 128, "stage A covers one 128-row MMA group");
  static_assert(P % 4 == 0, "stage B halves hold whole groups of two pairs");
  static_assert((P / 2) * NB <= 256 && NA <= 256, "TMEM budget");
  static_assert(128 * 2 * KA * 2 <= BUFX_BYTES, "stage A operand fits in bufX");
};

// W_L^e = exp(-2 pi i e / L) (e reduced mod L to (-L/2, L/2]) with the
// MUFU sin/cos: absolute error <= 2^-21.4 on [-pi, pi] (CUDA math API),
// far below the fp16 operand rounding (2^-11) every stage applies.
template <int L>
FC_DEVICE float2 wroot(int e) {
  e &= (L - 1);
  if (e > L / 2) e -= L;
  float sn, cs;
  __sincosf(float(e) * (-6.28318530717958647692f / float(L)), &sn, &cs);
  return make_float2(cs, sn);
}

FC_DEVICE void st_half8(uint32_t addr, const float* v) {
  st_shared_v4(addr, pack_half2(v[0], v[1]), pack_half2(v[2], v[3]), pack_half2(v[4], v[5]),
               pack_half2(v[6], v[7]));
}

// x <- x * w for 8 consecutive elements held as planes (xr, xi, -xi);
// w given as 4 float4 {wr_j, wr_j+1, wi_j, wi_j+1}.
FC_DEVICE void cmul8(float* xr, float* xi, const float* nxi, const float4* w) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 r = make_float2(xr[2 * j], xr[2 * j + 1]);
    const float2 i = make_float2(xi[2 * j], xi[2 * j + 1]);
    const float2 ni = make_float2(nxi[2 * j], nxi[2 * j + 1]);
    const float2 wr = make_float2(w[j].x, w[j].y), wi = make_float2(w[j].z, w[j].w);
    const float2 orr = fma2(r, wr, mul2(ni, wi));
    const float2 oi = fma2(i, wr, mul2(r, wi));
    xr[2 * j] = orr.x; xr[2 * j + 1] = orr.y;
    xi[2 * j] = oi.x;  xi[2 * j + 1] = oi.y;
  }
}
// Twiddle pair {wr_j, wr_j+1, wi_j, wi_j+1} -> the next pair (j + 2), i.e.
// both elements times the complex step c (fp32).
FC_DEVICE float4 cstep(const float4& w, float2 c) {
  const float2 wr = make_float2(w.x, w.y), wi = make_float2(w.z, w.w);
  const float2 nr = fma2(wr, make_float2(c.x, c.x), mul2(wi, make_float2(-c.y, -c.y)));
  const float2 ni = fma2(wr, make_float2(c.y, c.y), mul2(wi, make_float2(c.x, c.x)));
  return make_float4(nr.x, nr.y, ni.x, ni.y);
}
// x <- x * conj(w); planes (xr, xi, -xr).
FC_DEVICE void cmulc8(float* xr, float* xi, const float* nxr, const float4* w) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 r = make_float2(xr[2 * j], xr[2 * j + 1]);
    const float2 i = make_float2(xi[2 * j], xi[2 * j + 1]);
    const float2 nr = make_float2(nxr[2 * j], nxr[2 * j + 1]);
    const float2 wr = make_float2(w[j].x, w[j].y), wi = make_float2(w[j].z, w[j].w);
    const float2 orr = fma2(r, wr, mul2(i, wi));
    const float2 oi = fma2(i, wr, mul2(nr, wi));
    xr[2 * j] = orr.x; xr[2 * j + 1] = orr.y;
    xi[2 * j] = oi.x;  xi[2 * j + 1] = oi.y;
  }
}

}  // namespace fc
