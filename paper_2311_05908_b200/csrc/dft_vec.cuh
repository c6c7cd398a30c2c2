// dft_vec.cuh -- small in-register DFTs over "column vectors": every complex
// value is C2 pairs of adjacent columns held as packed fp32 pairs, so one
// f32x2 instruction (FADD2/FMUL2/FFMA2) advances two columns.  Used by the
// outer passes of the multipass regime (the DFT_L0 over n0 of Alg. 4,
// P:979-1004), where every thread owns 2*C2 adjacent columns n'.
// Trivial twiddles (1, -+i) are resolved at compile time.
#pragma once
#include <cuda_runtime.h>

#include "dft_small.cuh"
#include "sm100.cuh"

namespace fc {

FC_DEVICE float2 add2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
FC_DEVICE float2 sub2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

template <int C2>
struct CV {
  float2 r[C2], i[C2];
};

// x * w for a per-column twiddle vector w (runtime)
template <int C2>
FC_DEVICE CV<C2> cv_mul(const CV<C2>& x, const CV<C2>& w) {
  CV<C2> o;
#pragma unroll
  for (int c = 0; c < C2; ++c) {
    o.r[c] = fma2(x.r[c], w.r[c], mul2(make_float2(-x.i[c].x, -x.i[c].y), w.i[c]));
    o.i[c] = fma2(x.r[c], w.i[c], mul2(x.i[c], w.r[c]));
  }
  return o;
}
// x * conj(w)
template <int C2>
FC_DEVICE CV<C2> cv_mulc(const CV<C2>& x, const CV<C2>& w) {
  CV<C2> o;
#pragma unroll
  for (int c = 0; c < C2; ++c) {
    o.r[c] = fma2(x.r[c], w.r[c], mul2(x.i[c], w.i[c]));
    o.i[c] = fma2(x.i[c], w.r[c], mul2(make_float2(-x.r[c].x, -x.r[c].y), w.i[c]));
  }
  return o;
}
// x * (wr + i wi), a scalar twiddle broadcast to every column
template <int C2>
FC_DEVICE CV<C2> cv_mul_s(const CV<C2>& x, float wr, float wi) {
  CV<C2> o;
  const float2 r2 = make_float2(wr, wr), i2 = make_float2(wi, wi), ni2 = make_float2(-wi, -wi);
#pragma unroll
  for (int c = 0; c < C2; ++c) {
    o.r[c] = fma2(x.r[c], r2, mul2(x.i[c], ni2));
    o.i[c] = fma2(x.r[c], i2, mul2(x.i[c], r2));
  }
  return o;
}

// Butterfly v[k] = e + W t, v[k + NPT/2] = e - W t with W = W_NPT^{+-k}
// (INV: conjugate).  k is a compile-time constant after unrolling.
template <int NPT, bool INV, int C2>
FC_DEVICE void cv_bfly(int k, const CV<C2>& e, const CV<C2>& o, CV<C2>& lo, CV<C2>& hi) {
  if (k == 0) {
#pragma unroll
    for (int c = 0; c < C2; ++c) {
      lo.r[c] = add2(e.r[c], o.r[c]); lo.i[c] = add2(e.i[c], o.i[c]);
      hi.r[c] = sub2(e.r[c], o.r[c]); hi.i[c] = sub2(e.i[c], o.i[c]);
    }
  } else if (4 * k == NPT) {  // W = -i (forward) or +i (inverse)
#pragma unroll
    for (int c = 0; c < C2; ++c) {
      if (!INV) {  // e + (-i) o = (e.r + o.i, e.i - o.r)
        lo.r[c] = add2(e.r[c], o.i[c]); lo.i[c] = sub2(e.i[c], o.r[c]);
        hi.r[c] = sub2(e.r[c], o.i[c]); hi.i[c] = add2(e.i[c], o.r[c]);
      } else {     // e + i o = (e.r - o.i, e.i + o.r)
        lo.r[c] = sub2(e.r[c], o.i[c]); lo.i[c] = add2(e.i[c], o.r[c]);
        hi.r[c] = add2(e.r[c], o.i[c]); hi.i[c] = sub2(e.i[c], o.r[c]);
      }
    }
  } else {
    const float2 w = w_root<NPT>(k);
    const CV<C2> t = cv_mul_s(o, w.x, INV ? -w.y : w.y);
#pragma unroll
    for (int c = 0; c < C2; ++c) {
      lo.r[c] = add2(e.r[c], t.r[c]); lo.i[c] = add2(e.i[c], t.i[c]);
      hi.r[c] = sub2(e.r[c], t.r[c]); hi.i[c] = sub2(e.i[c], t.i[c]);
    }
  }
}

// Natural-order DFT of length NPT (INV: inverse without 1/NPT), in place.
template <int NPT, bool INV, int C2>
struct DftVec {
  static FC_DEVICE void run(CV<C2>* v) {
    CV<C2> e[NPT / 2], o[NPT / 2];
#pragma unroll
    for (int j = 0; j < NPT / 2; ++j) {
      e[j] = v[2 * j];
      o[j] = v[2 * j + 1];
    }
    DftVec<NPT / 2, INV, C2>::run(e);
    DftVec<NPT / 2, INV, C2>::run(o);
#pragma unroll
    for (int k = 0; k < NPT / 2; ++k) cv_bfly<NPT, INV>(k, e[k], o[k], v[k], v[k + NPT / 2]);
  }
};
template <bool INV, int C2>
struct DftVec<1, INV, C2> {
  static FC_DEVICE void run(CV<C2>*) {}
};

}  // namespace fc
