// kernels_bwd.cu -- fused backward of the FFT convolution on sm_100a
// (recomputation; gradient formulas A15 / SURVEY 8(c) c.1).
//
// For a tile of P row pairs of head h (two real rows per complex sequence,
// as in the forward kernel) the kernel
//   1. recomputes G  = FFT(pad g),  g  = u*w (gated) or u     [stages A, B]
//   2. computes   DC = FFT(pad dc), dc = dy*v (gated) or dy   [stages A, B]
//   3. (gated) c  = IFFT(G k_f)        -> dv = dy * c          [B^-1, A^-1]
//   4.         dg = IFFT(DC conj(k_f)) -> du = dg * w (or dg), dw = dg * u
//   5. accumulates sum_pairs DC conj(G) over the tile in fp32 and writes the
//      tile's partial spectrum; with two rows packed per complex sequence
//      Re IFFT(sum_pairs Z_dc conj(Z_g)) = sum_b corr(dc_b, g_b) = dk, so no
//      real/imag unpacking is needed.  A finalize kernel sums the partials of
//      each head in a fixed order (deterministic, no atomics) and inverse
//      transforms them (fp32) into dk[h, :K].
// Correlation with k is convolution with conj(k_f) (no wrap for the
// zero-padded causal case).  Template CAUSAL=false runs the same kernel on the
// complex rows of the multipass regime's intermediate (circular, no gating).
#include <cuda_runtime.h>

#include <type_traits>

#include "fused_common.cuh"
#include "fwd_params.h"
#include "launch_util.h"
#include "sm100.cuh"

namespace fc {

// Two independent warpgroups per CTA (as the forward kernel): each owns 256
// TMEM columns (G spectrum in [0, 128), DC in [128, 256): stage B / B^-1 emit
// re | im only, the negated plane a complex multiply needs is a register
// negation) and its own k_f copy, operand buffer and reduction buffer; the
// DFT tables are shared (G_B / G_B^-1 only their re | im rows; twiddles from
// MUFU sin/cos and fp32 recurrences instead of tables).
template <int L1, bool CAUSAL>
struct BwdCfg {
  using C = O2Cfg<L1, CAUSAL>;
  static constexpr int NBF = 2 * L1;                          // stage B / B^-1 N: re | im
  static constexpr uint32_t GB_SM = uint32_t(NBF) * (2 * L1) * 2;
  static constexpr uint32_t S_GA = 0;
  static constexpr uint32_t S_GB = C::al(S_GA + C::GA_BYTES);
  static constexpr uint32_t S_GBI = C::al(S_GB + GB_SM);
  static constexpr uint32_t S_GAI = C::al(S_GBI + GB_SM);
  static constexpr uint32_t TABLES = C::al(S_GAI + C::GAI_BYTES);  // full G_A^-1 (M = 128)
  static constexpr uint32_t RED_BYTES = 64 * (L1 * 8 + 16);  // tile partial spectrum, padded rows
  static constexpr uint32_t WG_BYTES = C::al(C::KF_BYTES) + C::al(C::BUFX_BYTES) + C::al(RED_BYTES);
  static constexpr uint32_t bytes_for(int wg) { return TABLES + wg * WG_BYTES + 1024; }  // + alignment slack
  static constexpr int WG = bytes_for(2) <= 227 * 1024 ? 2 : 1;
  static constexpr int THREADS = WG * kWGThreads;
  static constexpr uint32_t SMEM = bytes_for(WG);
  static constexpr uint32_t TMEM_COLS = 256;  // per warpgroup
  static constexpr uint32_t RD = 128;         // TMEM column base of the DC spectrum (G uses [0, 128))
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert((C::P / 2) * NBF <= 128 && C::NA <= 128, "G and DC spectra in 128 TMEM columns each");
};

template <int L1, bool CAUSAL, bool GATE_IO, bool NEED_C, typename T>
__global__ void __launch_bounds__(BwdCfg<L1, CAUSAL>::THREADS, 1) fftconv_bwd_o2_kernel(const BwdParams prm) {
  using C = O2Cfg<L1, CAUSAL>;
  using BC = BwdCfg<L1, CAUSAL>;
  constexpr int L2 = C::L2;
  constexpr int NBF = BC::NBF;
  constexpr int kWG = BC::WG;
  constexpr int kThreads = BC::THREADS;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t mma_bars[kWG][2];
  __shared__ uint32_t tmem_slot;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sGA = base + BC::S_GA, sGB = base + BC::S_GB, sGBI = base + BC::S_GBI, sGAI = base + BC::S_GAI;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wg = int(warp_uniform(warp >> 3));
  const int wtid = tid & (kWGThreads - 1);
  const int quad = warp & 3, slice = (warp >> 2) & 1;
  const int m = quad * 32 + lane;
  const uint32_t sKF = base + BC::TABLES + wg * BC::WG_BYTES;
  const uint32_t bufX = sKF + C::al(C::KF_BYTES), sRED = bufX + C::al(C::BUFX_BYTES);
  uint64_t* mma_bar = mma_bars[wg];
  const uint32_t bar_id = 1 + wg;
  const int64_t B = prm.B, H = prm.H, N = prm.N;
  const int64_t nbt = (B + C::R - 1) / C::R;
  const int64_t tiles = H * nbt;
  const int64_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  if (t0 >= t1) return;

  const T* __restrict__ gu = reinterpret_cast<const T*>(prm.u);
  const T* __restrict__ gw = reinterpret_cast<const T*>(prm.w);
  const T* __restrict__ gv = reinterpret_cast<const T*>(prm.v);
  const T* __restrict__ gdy = reinterpret_cast<const T*>(prm.dy);
  T* __restrict__ gdu = reinterpret_cast<T*>(prm.du);
  T* __restrict__ gdw = reinterpret_cast<T*>(prm.dw);
  T* __restrict__ gdv = reinterpret_cast<T*>(prm.dv);
  const uint8_t* __restrict__ gkf = reinterpret_cast<const uint8_t*>(prm.kf);

  {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(prm.tables);
    auto seg = [&](uint32_t dst, uint32_t img_off, uint32_t bytes) {
      for (uint32_t o = tid * 16; o < bytes; o += kThreads * 16) cp_async16(base + dst + o, src + img_off + o, true);
    };
    seg(BC::S_GA, C::OFF_GA, C::GA_BYTES);
    seg(BC::S_GB, C::OFF_GB, BC::GB_SM);   // rows re | im (the first NBF rows)
    seg(BC::S_GBI, C::OFF_GBI, BC::GB_SM);
    seg(BC::S_GAI, C::OFF_GAI, C::GAI_BYTES);
    cp_async_commit();
  }
  if (tid == 0) {
    for (int g = 0; g < kWG; ++g) {
      mbar_init(&mma_bars[g][0], 1);
      mbar_init(&mma_bars[g][1], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<kWG * BC::TMEM_COLS>(&tmem_slot);
  cp_async_wait_all();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = warp_uniform(tmem_slot) + wg * BC::TMEM_COLS;
  const uint32_t tq = tmem + (uint32_t(quad * 32) << 16);
  uint32_t phase = 0;
  int64_t cur_h = -1;

  const uint64_t dXA = smem_desc(bufX, 128, C::SBO_A);
  const uint64_t dGA = smem_desc(sGA, 128, C::SBO_GA);
  const uint64_t dXB = smem_desc(bufX, C::LBO_B, 128);
  const uint64_t dGB = smem_desc(sGB, 128, C::SBO_GB);
  const uint64_t dXBP = smem_desc(bufX, 128, C::SBO_BP);
  const uint64_t dGBI = smem_desc(sGBI, 128, C::SBO_GB);
  const uint64_t dGAI = smem_desc(sGAI, 128, C::SBO_GAI);
  const uint64_t dXAI = smem_desc(bufX, 128, C::SBO_XA);
  auto dadd = [](uint64_t d, uint32_t off) { return d + uint64_t(off >> 4); };

  auto wg_sync = [&] { named_sync(bar_id, kWGThreads); };
  auto sync_and_issue = [&](auto&& issue_half) {
    fence_async_smem();
    tc_fence_before();
    wg_sync();
    if (wtid < 32 && elect_one()) {
      tc_fence_after();
      issue_half(0);
      mma_commit(&mma_bar[0]);
      issue_half(1);
      mma_commit(&mma_bar[1]);
    }
    phase ^= 1;
  };
  auto wait_half = [&](int hh) {
    mbar_wait_warp(&mma_bar[hh], phase ^ 1);
    tc_fence_after();
  };
  auto wait_both = [&] {
    wait_half(0);
    wait_half(1);
  };

  constexpr int KROWS = C::KA;
  constexpr int JC = L1 / 8;
  constexpr int RSTEP = kWGThreads / (KROWS * JC);
  const int64_t HN = H * N;
  const int ld_n2 = wtid % KROWS, ld_j = (wtid / KROWS) % JC, ld_r0 = wtid / (KROWS * JC);
  const int64_t ld_off0 = int64_t(ld_r0) * HN + int64_t(ld_n2 * JC + ld_j) * 8;
  // stage A^-1 output lane m = G_AI row (n2 half, c', n2 mod 32), see plan.cpp
  const int64_t st_off0 = int64_t((m >> 5) & 1) * HN + int64_t(L1) * ((m >> 6) * 32 + (m & 31));

  auto chunk_dst = [&](int r, int n2, int j) -> uint32_t {
    const int k = (r & 1) * C::KA + n2;
    return bufX + ((r >> 1) * JC + j) * C::SBO_A + (k >> 3) * 128 + (k & 7) * 16;
  };
  // product a*b -> fp16 operand chunk (b == nullptr: a alone)
  auto mul8 = [&](uint4 a, uint4 b, bool use_b) -> uint4 {
    if constexpr (std::is_same<T, __half>::value) {
      if (use_b) {
        __half2* x = reinterpret_cast<__half2*>(&a);
        const __half2* y = reinterpret_cast<const __half2*>(&b);
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = __hmul2(x[e], y[e]);
      }
      return a;
    } else {
      float g[8];
      IO<T>::to_f32x8(a, g);
      if (use_b) {
        float w8[8];
        IO<T>::to_f32x8(b, w8);
#pragma unroll
        for (int e = 0; e < 8; ++e) g[e] *= w8[e];
      }
      return make_uint4(pack_half2(g[0], g[1]), pack_half2(g[2], g[3]), pack_half2(g[4], g[5]),
                        pack_half2(g[6], g[7]));
    }
  };
  constexpr int PER_ALL = (C::R * C::CH) / kWGThreads;
  // load x (* y) rows of the tile into registers (issue only)
  auto load_rows = [&](const T* x, const T* y, bool use_y, int64_t tile_base, int rows_left, uint4* xa, uint4* ya) {
#pragma unroll
    for (int i = 0; i < PER_ALL; ++i) {
      const int r = ld_r0 + i * RSTEP;
      if (r < rows_left) {
        const int64_t goff = tile_base + ld_off0 + int64_t(i * RSTEP) * HN;
        xa[i] = *reinterpret_cast<const uint4*>(x + goff);
        if (use_y) ya[i] = *reinterpret_cast<const uint4*>(y + goff);
      } else {
        xa[i] = make_uint4(0, 0, 0, 0);
        ya[i] = make_uint4(0, 0, 0, 0);
      }
    }
  };
  auto store_rows = [&](const uint4* xa, const uint4* ya, bool use_y) {
#pragma unroll
    for (int i = 0; i < PER_ALL; ++i) {
      const uint4 g = mul8(xa[i], ya[i], use_y);
      st_shared_v4(chunk_dst(ld_r0 + i * RSTEP, ld_n2, ld_j), g.x, g.y, g.z, g.w);
    }
  };

  // ---- forward stages A, twiddle, B of one spectrum into TMEM columns [rb, rb + 256)
  auto forward_AB = [&](uint32_t rb) {
    sync_and_issue([&](int hh) {  // TMEM column of (block, k2): (k2 / 32) * NA/2 + 32 * block + k2 % 32
      constexpr uint32_t idesc = idesc_f16(128, C::NA / 2, true, false);
#pragma unroll
      for (int s = 0; s < 2 * C::KA / 16; ++s)
        mma_f16_ss(tmem + rb + hh * (C::NA / 2), dadd(dXA, 256 * s),
                   dadd(dGA, hh * (C::NA / 16) * C::SBO_GA + 256 * s), idesc, s > 0);
    });
    {
      const int p = m / L1, n1 = m % L1;
      wait_half(slice);
#pragma unroll 1
      for (int sub = 0; sub < 2; ++sub) {
        const int k20 = slice * 32 + sub * 16;
        const uint32_t c0 = rb + slice * (C::NA / 2) + sub * 16;
        float re[16], im[16], ni[16];
        tmem_ld16(tq + c0, re);
        tmem_ld16(tq + c0 + 32, im);
        if constexpr (C::NEG_A) tmem_ld16(tq + c0 + 64, ni);
        // W_L^{n1 k2}, k2 = k20 .. k20 + 15: MUFU pair at k20, fp32 steps by W^{2 n1}
        float4 w[8];
        {
          const float2 a = wroot<C::L>(n1 * k20), b = wroot<C::L>(n1 * (k20 + 1));
          w[0] = make_float4(a.x, b.x, a.y, b.y);
          const float2 st = wroot<C::L>(2 * n1);
#pragma unroll
          for (int jj = 1; jj < 8; ++jj) w[jj] = cstep(w[jj - 1], st);
        }
        tmem_ld_wait();
        if constexpr (!C::NEG_A) {
#pragma unroll
          for (int e = 0; e < 16; ++e) ni[e] = -im[e];
        }
        cmul8(re, im, ni, w);
        cmul8(re + 8, im + 8, ni + 8, w + 4);
        if (sub == 0) wait_half(slice ^ 1);
#pragma unroll
        for (int hh2 = 0; hh2 < 2; ++hh2) {
          const int mg = p * (L2 / 8) + k20 / 8 + hh2;
          st_half8(bufX + mg * 128 + (n1 >> 3) * C::LBO_B + (n1 & 7) * 16, re + 8 * hh2);
          st_half8(bufX + mg * 128 + ((L1 + n1) >> 3) * C::LBO_B + (n1 & 7) * 16, im + 8 * hh2);
        }
      }
    }
    sync_and_issue([&](int hh) {
      constexpr uint32_t idesc = idesc_f16(128, NBF, true, false);
#pragma unroll
      for (int gi = hh * (C::P / 4); gi < (hh + 1) * (C::P / 4); ++gi) {
#pragma unroll
        for (int s = 0; s < 2 * L1 / 16; ++s)
          mma_f16_ss(tmem + rb + gi * NBF, dadd(dXB, gi * 2048 + 2 * s * C::LBO_B), dadd(dGB, 256 * s), idesc,
                     s > 0);
      }
    });
  };

  // ---- inverse stages B^-1, conj twiddle, A^-1 of the operand in bufX (TMEM [0, 256))
  auto inverse_BA = [&] {
    sync_and_issue([&](int hh) {
      constexpr uint32_t idesc = idesc_f16(128, NBF, false, false);
#pragma unroll
      for (int gi = hh * (C::P / 4); gi < (hh + 1) * (C::P / 4); ++gi) {
#pragma unroll
        for (int s = 0; s < 2 * L1 / 16; ++s)
          mma_f16_ss(tmem + gi * NBF, dadd(dXBP, gi * 16 * C::SBO_BP + 256 * s), dadd(dGBI, 256 * s), idesc,
                     s > 0);
      }
    });
    {
      const int k2 = m & 63;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;
        const int gi = it / (L1 / 8), n1c = it % (L1 / 8);
        const int p = gi * 2 + (m >> 6);
        if (i == 0) wait_half(0);
        const uint32_t col = gi * NBF + n1c * 8;
        float re[8], im[8], nr[8];
        tmem_ld8(tq + col, re);
        tmem_ld8(tq + col + L1, im);
        // W^{n1 k2}, n1 = 8 n1c .. 8 n1c + 7: MUFU pair, fp32 steps by W^{2 k2}
        float4 w[4];
        {
          const float2 a = wroot<C::L>(8 * n1c * k2), c1 = wroot<C::L>(k2), c2 = wroot<C::L>(2 * k2);
          w[0] = make_float4(a.x, a.x * c1.x - a.y * c1.y, a.y, a.x * c1.y + a.y * c1.x);
#pragma unroll
          for (int jj = 1; jj < 4; ++jj) w[jj] = cstep(w[jj - 1], c2);
        }
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) nr[e] = -re[e];
        cmulc8(re, im, nr, w);
        if (i == 0) wait_half(1);
        const int ng = (p * L1) / 8 + n1c;
        st_half8(bufX + ng * C::SBO_XA + (k2 >> 3) * 128 + (k2 & 7) * 16, re);
        st_half8(bufX + ng * C::SBO_XA + ((L2 + k2) >> 3) * 128 + (k2 & 7) * 16, im);
      }
    }
    sync_and_issue([&](int hh) {
      constexpr uint32_t idesc = idesc_f16(128, 64, false, true);
#pragma unroll
      for (int s = 0; s < 2 * L2 / 16; ++s)
        mma_f16_ss(tmem + hh * 64, dadd(dGAI, 256 * s), dadd(dXAI, hh * 8 * C::SBO_XA + 256 * s), idesc, s > 0);
    });
  };

  // ---- epilogue 4 variants: out1 = o * a1 (or o), out2 = o * a2 (optional)
  auto epi_out = [&](int64_t tile_base, int rows_left, const T* a1, T* out1, const T* a2, T* out2, bool gate) {
    const int cp = (m >> 5) & 1;
    if (!CAUSAL || m < 64) {  // warp-uniform
      constexpr int NIT = C::P * (L1 / 8);
      constexpr int PER = NIT / 2;
      // the gate vectors of item i + 1 are loaded while item i is processed
      // (the first before the MMA wait): their global latency is hidden
      uint4 ga[2], gb[2];
      auto ld_gate = [&](int i, uint4& a, uint4& b) {
        const int it = slice * PER + i;
        const int p = it / (L1 / 8), n1c = it % (L1 / 8);
        const int64_t goff = tile_base + st_off0 + int64_t(2 * p) * HN + n1c * 8;
        a = make_uint4(0, 0, 0, 0);
        b = make_uint4(0, 0, 0, 0);
        if (gate && 2 * p + cp < rows_left) {
          a = *reinterpret_cast<const uint4*>(a1 + goff);
          if (out2) b = *reinterpret_cast<const uint4*>(a2 + goff);
        }
      };
      ld_gate(0, ga[0], gb[0]);
      wait_half(slice);
#pragma unroll 2
      for (int i = 0; i < PER; ++i) {
        const int it = slice * PER + i;
        const int p = it / (L1 / 8), n1c = it % (L1 / 8);
        const bool ok = 2 * p + cp < rows_left;
        const int64_t goff = tile_base + st_off0 + int64_t(2 * p) * HN + n1c * 8;
        if (i + 1 < PER) ld_gate(i + 1, ga[(i + 1) & 1], gb[(i + 1) & 1]);
        const uint4 va = ga[i & 1], vb = gb[i & 1];
        float o[8];
        tmem_ld8(tq + p * L1 + n1c * 8, o);
        tmem_ld_wait();
        float r1[8];
        if (gate) {
          IO<T>::to_f32x8(va, r1);
#pragma unroll
          for (int e = 0; e < 8; ++e) r1[e] *= o[e];
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) r1[e] = o[e];
        }
        if (ok)
          *reinterpret_cast<uint4*>(out1 + goff) = make_uint4(IO<T>::pack2(r1[0], r1[1]), IO<T>::pack2(r1[2], r1[3]),
                                                              IO<T>::pack2(r1[4], r1[5]), IO<T>::pack2(r1[6], r1[7]));
        if (out2 && ok) {
          float r2[8];
          IO<T>::to_f32x8(vb, r2);
#pragma unroll
          for (int e = 0; e < 8; ++e) r2[e] *= o[e];
          *reinterpret_cast<uint4*>(out2 + goff) = make_uint4(IO<T>::pack2(r2[0], r2[1]), IO<T>::pack2(r2[2], r2[3]),
                                                              IO<T>::pack2(r2[4], r2[5]), IO<T>::pack2(r2[6], r2[7]));
        }
      }
    }
  };

  constexpr int NK1C = (L1 / 8) / 2 > 0 ? (L1 / 8) / 2 : 1;  // distinct k1 chunks per thread
  // warpgroup wg processes tiles t0 + wg, t0 + wg + kWG, ...
  int64_t h = (t0 + wg) / nbt, bt = (t0 + wg) % nbt;
  uint4 nxa[PER_ALL], nya[PER_ALL];  // g rows of the next tile (prefetched)
  for (int64_t t = t0 + wg; t < t1; t += kWG, bt += kWG) {
    while (bt >= nbt) { bt -= nbt; ++h; }
    const int64_t tile_base = (bt * C::R * H + h) * N;
    const int rows_left = int(B - bt * C::R < C::R ? B - bt * C::R : C::R);
    if (h != cur_h) {
      const uint8_t* src = gkf + h * int64_t(C::KF_BYTES);
      for (uint32_t o = wtid * 16; o < C::KF_BYTES; o += kWGThreads * 16) cp_async16(sKF + o, src + o, true);
      cp_async_commit();
      cur_h = h;
    }
    uint4 xa[PER_ALL], ya[PER_ALL];
    // 1. G = FFT(g) (its rows were prefetched during the previous tile's
    // last epilogue)
    if (t == t0 + wg) load_rows(gu, gw, GATE_IO, tile_base, rows_left, nxa, nya);
    store_rows(nxa, nya, GATE_IO);
    cp_async_wait_all();
    forward_AB(0);
    // 2. DC = FFT(dc): issue loads, then wait until stage B(G) has read bufX
    load_rows(gdy, gv, GATE_IO, tile_base, rows_left, xa, ya);
    wait_both();
    store_rows(xa, ya, GATE_IO);
    forward_AB(BC::RD);
    wait_both();

    // 3. pointwise: X1 = G k_f (-> c), partial sum DC conj(G) (-> dk)
    float acc[NK1C][16];
#pragma unroll
    for (int a = 0; a < NK1C; ++a)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[a][e] = 0.f;
    {
      const int k2 = m & 63;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;
        const int gi = it / (L1 / 8), k1c = it % (L1 / 8);
        const int ai = (k1c >> 1) % NK1C;  // k1c = slice + 2 * ai for L1 = 32
        const int row = gi * 128 + m;
        const uint32_t col = gi * NBF + k1c * 8;
        float gr[8], gim[8], gni[8], dr[8], di[8];
        tmem_ld8(tq + col, gr);
        tmem_ld8(tq + col + L1, gim);
        tmem_ld8(tq + BC::RD + col, dr);
        tmem_ld8(tq + BC::RD + col + L1, di);
        float4 kf[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kf[jj] = ld_shared_f4(sKF + tab_off<L1 / 2>(k2, k1c * 4 + jj));
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) gni[e] = -gim[e];
        // acc += DC * conj(G): re = dr gr + di gi, im = di gr - dr gi (= di gr + dr (-gi))
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 Dr = make_float2(dr[2 * j], dr[2 * j + 1]), Di = make_float2(di[2 * j], di[2 * j + 1]);
          const float2 Gr = make_float2(gr[2 * j], gr[2 * j + 1]), Gi = make_float2(gim[2 * j], gim[2 * j + 1]);
          const float2 Gn = make_float2(gni[2 * j], gni[2 * j + 1]);
          float2 ar = make_float2(acc[ai][4 * j], acc[ai][4 * j + 1]);
          float2 aim = make_float2(acc[ai][4 * j + 2], acc[ai][4 * j + 3]);
          ar = fma2(Dr, Gr, fma2(Di, Gi, ar));
          aim = fma2(Di, Gr, fma2(Dr, Gn, aim));
          acc[ai][4 * j] = ar.x; acc[ai][4 * j + 1] = ar.y;
          acc[ai][4 * j + 2] = aim.x; acc[ai][4 * j + 3] = aim.y;
        }
        if (NEED_C) {
          cmul8(gr, gim, gni, kf);
          st_half8(bufX + (row >> 3) * C::SBO_BP + k1c * 128 + (row & 7) * 16, gr);
          st_half8(bufX + (row >> 3) * C::SBO_BP + (L1 / 8 + k1c) * 128 + (row & 7) * 16, gim);
        }
      }
    }
    // reduce the partial sums held by the four thread classes (lane half x
    // column slice; for L1 = 8 both slices hold the same k1) in a fixed
    // order through shared memory, then write the tile's partial spectrum
    // part[t][f], f = k2 + L2 k1 (natural order), coalesced.
    {
      constexpr uint32_t RS = L1 * 8 + 16;  // padded row stride of red[k2][k1]
      const int k2 = m & 63;
      const int cls = (m >= 64 ? 2 : 0) + slice;
      // L1 >= 16: the two column slices hold disjoint k1 chunks, so classes
      // 0 and 1 store in one step and classes 2 and 3 add in the next (the
      // same per-element order as four steps: class 0 (1), then + class 2 (3))
      constexpr bool TWO = L1 / 8 >= 2;
#pragma unroll 1
      for (int c = 0; c < (TWO ? 2 : 4); ++c) {
        if ((TWO ? (cls >> 1) : cls) == c) {
#pragma unroll
          for (int a = 0; a < NK1C; ++a) {
            const int k1c = TWO ? slice + 2 * a : 0;
            const bool add = TWO ? c == 1 : c >= 1;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const uint32_t o = sRED + k2 * RS + (k1c * 8 + e) * 8;
              float2 v = make_float2(acc[a][4 * (e / 2) + (e % 2)], acc[a][4 * (e / 2) + 2 + (e % 2)]);
              if (add) {
                const float2 old = ld_shared_f2(o);
                v.x += old.x;
                v.y += old.y;
              }
              asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(o), "f"(v.x), "f"(v.y) : "memory");
            }
          }
        }
        wg_sync();
      }
      float2* part = reinterpret_cast<float2*>(prm.acc) + t * int64_t(C::L);
      for (int q = wtid; q < C::L; q += kWGThreads) part[q] = ld_shared_f2(sRED + (q % L2) * RS + (q / L2) * 8);
    }

    // 4. (gated / inner) c = IFFT(X1)
    if (NEED_C) {
      inverse_BA();
      epi_out(tile_base, rows_left, gdy, gdv, nullptr, nullptr, GATE_IO);
      wait_both();
    }
    // 5. X2 = DC conj(k_f) -> dg
    {
      const int k2 = m & 63;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;
        const int gi = it / (L1 / 8), k1c = it % (L1 / 8);
        const int row = gi * 128 + m;
        const uint32_t col = BC::RD + gi * NBF + k1c * 8;
        float dr[8], di[8];
        tmem_ld8(tq + col, dr);
        tmem_ld8(tq + col + L1, di);
        float4 kf[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kf[jj] = ld_shared_f4(sKF + tab_off<L1 / 2>(k2, k1c * 4 + jj));
        tmem_ld_wait();
        // x * conj(k): re = dr kr + di ki, im = di kr + (-dr) ki
        float nr[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) nr[e] = -dr[e];
        cmulc8(dr, di, nr, kf);
        st_half8(bufX + (row >> 3) * C::SBO_BP + k1c * 128 + (row & 7) * 16, dr);
        st_half8(bufX + (row >> 3) * C::SBO_BP + (L1 / 8 + k1c) * 128 + (row & 7) * 16, di);
      }
    }
    inverse_BA();
    if (t + kWG < t1) {  // prefetch the next tile's g rows behind the last epilogue
      int64_t h2 = h, bt2 = bt + kWG;
      while (bt2 >= nbt) { bt2 -= nbt; ++h2; }
      const int64_t base2 = (bt2 * C::R * H + h2) * N;
      load_rows(gu, gw, GATE_IO, base2, int(B - bt2 * C::R < C::R ? B - bt2 * C::R : C::R), nxa, nya);
    }
    if (GATE_IO) epi_out(tile_base, rows_left, gw, gdu, gu, gdw, true);
    else epi_out(tile_base, rows_left, nullptr, gdu, nullptr, nullptr, false);
    tc_fence_before();
    wg_sync();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<kWG * BC::TMEM_COLS>(warp_uniform(tmem_slot));
}

int64_t bwd_tiles_per_head(int64_t B, int L1) {
  const int64_t R = 2 * (128 / L1);
  return (B + R - 1) / R;
}

template <int L1, bool CAUSAL, bool GATE_IO, bool NEED_C, typename T>
static cudaError_t launch_bwd_t(const BwdParams& prm, cudaStream_t s) {
  using BC = BwdCfg<L1, CAUSAL>;
  auto kern = fftconv_bwd_o2_kernel<L1, CAUSAL, GATE_IO, NEED_C, T>;
  static int attr[64] = {0};
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(BC::SMEM), attr)) return e;
  const int64_t tiles = prm.H * bwd_tiles_per_head(prm.B, L1);
  const int grid = int(tiles < prm.num_sms ? tiles : prm.num_sms);
  if (grid < 1) return cudaSuccess;
  kern<<<grid, BC::THREADS, BC::SMEM, s>>>(prm);
  return cudaGetLastError();
}

template <bool CAUSAL, bool GATE_IO, bool NEED_C, typename T>
static cudaError_t bwd_l1(const BwdParams& prm, cudaStream_t s) {
  switch (prm.L1) {
    case 8: return launch_bwd_t<8, CAUSAL, GATE_IO, NEED_C, T>(prm, s);
    case 16: return launch_bwd_t<16, CAUSAL, GATE_IO, NEED_C, T>(prm, s);
    case 32: return launch_bwd_t<32, CAUSAL, GATE_IO, NEED_C, T>(prm, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_bwd_fused(const BwdParams& prm, cudaStream_t s) {
  // (gate_io, need_c): fused plain (0, 0), fused gated (1, 1), multipass
  // inner on fp16 complex rows (0, gated)
  const bool half = prm.dtype == 0;
  if (prm.gate_io) {
    if (prm.causal) return half ? bwd_l1<true, true, true, __half>(prm, s) : bwd_l1<true, true, true, __nv_bfloat16>(prm, s);
    return half ? bwd_l1<false, true, true, __half>(prm, s) : bwd_l1<false, true, true, __nv_bfloat16>(prm, s);
  }
  if (prm.need_c) {
    if (!half) return cudaErrorInvalidValue;
    return prm.causal ? bwd_l1<true, false, true, __half>(prm, s) : bwd_l1<false, false, true, __half>(prm, s);
  }
  if (prm.causal) return half ? bwd_l1<true, false, false, __half>(prm, s) : bwd_l1<true, false, false, __nv_bfloat16>(prm, s);
  return half ? bwd_l1<false, false, false, __half>(prm, s) : bwd_l1<false, false, false, __nv_bfloat16>(prm, s);
}

}  // namespace fc
