// dft_small.cuh -- in-register complex DFTs of small power-of-two length
// (fp32, natural order in and out), used by the outer passes of the
// multipass regime and by the k_f precompute.
#pragma once
#include <cuda_runtime.h>

#include "sm100.cuh"

namespace fc {

FC_DEVICE float2 c_add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
FC_DEVICE float2 c_sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
FC_DEVICE float2 c_mul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
FC_DEVICE float2 c_mulc(float2 a, float2 b) { return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); }

// W_64^k = exp(-2 pi i k / 64), k < 32 (fp32-rounded from fp64).
__device__ __constant__ float2 c_w64[32] = {
    {1.000000000e+00f, -0.000000000e+00f}, {9.951847267e-01f, -9.801714033e-02f},
    {9.807852804e-01f, -1.950903220e-01f}, {9.569403357e-01f, -2.902846773e-01f},
    {9.238795325e-01f, -3.826834324e-01f}, {8.819212643e-01f, -4.713967368e-01f},
    {8.314696123e-01f, -5.555702330e-01f}, {7.730104534e-01f, -6.343932842e-01f},
    {7.071067812e-01f, -7.071067812e-01f}, {6.343932842e-01f, -7.730104534e-01f},
    {5.555702330e-01f, -8.314696123e-01f}, {4.713967368e-01f, -8.819212643e-01f},
    {3.826834324e-01f, -9.238795325e-01f}, {2.902846773e-01f, -9.569403357e-01f},
    {1.950903220e-01f, -9.807852804e-01f}, {9.801714033e-02f, -9.951847267e-01f},
    {6.123233996e-17f, -1.000000000e+00f}, {-9.801714033e-02f, -9.951847267e-01f},
    {-1.950903220e-01f, -9.807852804e-01f}, {-2.902846773e-01f, -9.569403357e-01f},
    {-3.826834324e-01f, -9.238795325e-01f}, {-4.713967368e-01f, -8.819212643e-01f},
    {-5.555702330e-01f, -8.314696123e-01f}, {-6.343932842e-01f, -7.730104534e-01f},
    {-7.071067812e-01f, -7.071067812e-01f}, {-7.730104534e-01f, -6.343932842e-01f},
    {-8.314696123e-01f, -5.555702330e-01f}, {-8.819212643e-01f, -4.713967368e-01f},
    {-9.238795325e-01f, -3.826834324e-01f}, {-9.569403357e-01f, -2.902846773e-01f},
    {-9.807852804e-01f, -1.950903220e-01f}, {-9.951847267e-01f, -9.801714033e-02f}};

// W_n^k for compile-time n <= 64 (k < n / 2)
template <int NPT>
FC_DEVICE float2 w_root(int k) {
  static_assert(NPT <= 64, "small DFT only");
  return c_w64[k * (64 / NPT)];
}

// Forward (INV=false) or inverse-without-scaling (INV=true) DFT of length NPT
// by recursive even/odd splitting; all loops unroll at compile time.
template <int NPT, bool INV>
struct DftReg {
  static FC_DEVICE void run(float2* v) {
    float2 e[NPT / 2], o[NPT / 2];
#pragma unroll
    for (int i = 0; i < NPT / 2; ++i) {
      e[i] = v[2 * i];
      o[i] = v[2 * i + 1];
    }
    DftReg<NPT / 2, INV>::run(e);
    DftReg<NPT / 2, INV>::run(o);
#pragma unroll
    for (int k = 0; k < NPT / 2; ++k) {
      float2 w = w_root<NPT>(k);
      if (INV) w.y = -w.y;
      const float2 t = c_mul(o[k], w);
      v[k] = c_add(e[k], t);
      v[k + NPT / 2] = c_sub(e[k], t);
    }
  }
};
template <bool INV>
struct DftReg<1, INV> {
  static FC_DEVICE void run(float2*) {}
};

}  // namespace fc
