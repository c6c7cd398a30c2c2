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
// real/imag planes stacked in K.  Stages followed by a complex multiply also
// emit a negated copy of one plane (an extra block of N columns -- tensor
// cores are idle in this HBM-bound regime) so the multiply is two FMUL2 and
// two FFMA2 per element pair with no sign fix-ups.
// The elementwise steps between stages run TMEM -> registers -> shared
// memory, where the write layout performs the "permutation as transpose" of
// P:226-234 for free: each stage's operand is written directly in the
// canonical UMMA layout (MN-major or K-major) the next MMA reads.  Gating
// (u*w on load, *v on store) is fused.  16 warps split every
// elementwise phase by TMEM column slices.
#include <cuda_runtime.h>

#include <type_traits>

#include "fused_common.cuh"
#include "fwd_params.h"
#include "sm100.cuh"

namespace fc {

#ifdef FC_TRACE
// experiment-only phase timestamps (CTA 0, warpgroup 0, warps 0 and 4)
__device__ long long fc_trace_buf[2][64][16];
#endif

// Each CTA runs kWG independent warpgroups; warpgroup g processes tiles
// t0 + g, t0 + g + kWG, ... of the CTA's contiguous tile range, with its own
// TMEM columns, mbarriers, named barrier, k_f copy and operand buffer, so one
// warpgroup's MMAs, memory waits and barriers overlap the other's math.
template <int L1, bool CAUSAL, bool GATED, typename T>
__global__ void __launch_bounds__(O2Cfg<L1, CAUSAL>::THREADS, 1) fftconv_fwd_o2_kernel(const FwdParams prm) {
  using C = O2Cfg<L1, CAUSAL>;
  constexpr int kWG = C::WG;
  constexpr int kThreads = C::THREADS;
  constexpr int L2 = C::L2;
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint64_t mma_bar[kWG][2];  // completion of the first / second half of a stage
  __shared__ uint32_t tmem_slot;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;  // 1024-aligned
  const uint32_t sGA = base + C::OFF_GA, sGB = base + C::OFF_GB, sGBI = base + C::OFF_GBI,
                 sGAI = base + C::OFF_GAI, sTW = base + C::OFF_TW, sTWT = base + C::OFF_TWT;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wg = int(warp_uniform(warp >> 3));  // warpgroup
  const int wtid = tid & (kWGThreads - 1);
  const int quad = warp & 3;             // TMEM lane quadrant this warp may access
  const int slice = (warp >> 2) & 1;     // column slice 0..1
  const int m = quad * 32 + lane;        // TMEM lane / MMA row owned by this thread
  const uint32_t sKF = base + C::OFF_WG + wg * C::WG_BYTES;
  const uint32_t bufX = sKF + C::al(C::KF_BYTES);
  const int64_t B = prm.B, H = prm.H, N = prm.N;
  const int64_t nbt = (B + C::R - 1) / C::R;
  const int64_t Hi = prm.row_map ? (H / prm.row_L0) * prm.nrow : H;  // heads iterated
  auto phys_head = [&](int64_t hh) -> int64_t {
    return prm.row_map ? (hh / prm.nrow) * prm.row_L0 + prm.row_map[hh % prm.nrow] : hh;
  };
  const int64_t tiles = Hi * nbt;
  const int64_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  if (t0 >= t1) return;

  const T* __restrict__ gu = reinterpret_cast<const T*>(prm.u);
  const T* __restrict__ gw = reinterpret_cast<const T*>(prm.w);
  const T* __restrict__ gv = reinterpret_cast<const T*>(prm.v);
  T* __restrict__ gy = reinterpret_cast<T*>(prm.y);
  const uint8_t* __restrict__ gkf = reinterpret_cast<const uint8_t*>(prm.kf);

  // ---- one-time setup: tables -> smem, barriers, TMEM (both warpgroups)
  {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(prm.tables);
    for (uint32_t o = tid * 16; o < C::TABLES; o += kThreads * 16) cp_async16(base + o, src + o, true);
    cp_async_commit();
  }
  if (tid == 0) {
    for (int g = 0; g < kWG; ++g) {
      mbar_init(&mma_bar[g][0], 1);
      mbar_init(&mma_bar[g][1], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<(kWG * C::TMEM_COLS > 512 ? 512 : kWG * C::TMEM_COLS)>(&tmem_slot);
  cp_async_wait_all();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = warp_uniform(tmem_slot) + wg * C::TMEM_COLS;
  const uint32_t tq = tmem + (uint32_t(quad * 32) << 16);  // this warp's lane quadrant
  uint64_t* bars = mma_bar[wg];
  const uint32_t bar_id = 1 + wg;  // named barrier of this warpgroup
  uint32_t phase = 0;
  int64_t cur_h = -1;

  // UMMA shared-memory descriptors: built once, offsets added as (bytes >> 4)
  const uint64_t dXA = smem_desc(bufX, 128, C::SBO_A);          // stage A operand (MN-major)
  const uint64_t dGA = smem_desc(sGA, 128, C::SBO_GA);
  const uint64_t dXB = smem_desc(bufX, C::LBO_B, 128);          // stage B operand (MN-major)
  const uint64_t dGB = smem_desc(sGB, 128, C::SBO_GB);
  const uint64_t dXBP = smem_desc(bufX, 128, C::SBO_BP);        // stage B^-1 operand (K-major)
  const uint64_t dGBI = smem_desc(sGBI, 128, C::SBO_GB);
  const uint64_t dGAI = smem_desc(sGAI, 128, C::SBO_GAI);
  const uint64_t dXAI = smem_desc(bufX, 128, C::SBO_XA);        // stage A^-1 operand (MN-major B)
  auto dadd = [](uint64_t d, uint32_t off) { return d + uint64_t(off >> 4); };

  int trace_tile = 0;
  auto stamp = [&](int k) {
#ifdef FC_TRACE
    if (blockIdx.x == 0 && wg == 0 && (wtid == 0 || wtid == 128) && trace_tile < 64)
      fc_trace_buf[wtid >> 7][trace_tile][k] = clock64();
#endif
  };
  int stage_no = 0;
  auto wg_sync = [&] { named_sync(bar_id, kWGThreads); };
  // Operands written -> warpgroup barrier -> one thread issues the stage as
  // two halves, each committed to its own mbarrier so the epilogue of the
  // first half overlaps the MMAs of the second.
  auto sync_and_issue = [&](auto&& issue_half) {
    fence_async_smem();
    tc_fence_before();
    wg_sync();
    stamp(2 + 3 * stage_no);
    if (wtid < 32 && elect_one()) {
      tc_fence_after();
      issue_half(0);
      mma_commit(&bars[0]);
      issue_half(1);
      mma_commit(&bars[1]);
    }
    stamp(3 + 3 * stage_no);
    ++stage_no;
    phase ^= 1;  // both barriers complete once per stage
  };
  auto wait_half = [&](int hh) {  // parity of the stage issued last
    mbar_wait_warp(&bars[hh], phase ^ 1);
    tc_fence_after();
  };

  // Per-thread invariants of the input loader: chunk q = wtid + i * 256 maps
  // to (n2, j, r) with n2, j fixed and r = r0 + i * RSTEP.
  constexpr int KROWS = C::KA;  // n2 rows per row
  constexpr int JC = L1 / 8;    // 8-element n1 chunks
  constexpr int RSTEP = kWGThreads / (KROWS * JC);
  static_assert(kWGThreads % (KROWS * JC) == 0, "loader mapping");
  const int64_t HN = H * N;
  const int ld_n2 = wtid % KROWS, ld_j = (wtid / KROWS) % JC, ld_r0 = wtid / (KROWS * JC);
  const int64_t ld_off0 = int64_t(ld_r0) * HN + int64_t(ld_n2 * JC + ld_j) * 8;
  // epilogue-4 invariants: row (2p + cp) of the tile, positions L1*n2 + 8*n1c
  const int64_t st_off0 = int64_t(m >> 6) * HN + int64_t(L1) * (m & 63);

  // u (*w) -> fp16 operand chunk of 8 elements
  auto gate8 = [&](uint4 uv, uint4 wv) -> uint4 {
    if constexpr (std::is_same<T, __half>::value) {
      // the fp16 product of two fp16 values equals the fp32 product rounded
      // to fp16, so gate with HMUL2 and skip conversions
      if (GATED) {
        __half2* a = reinterpret_cast<__half2*>(&uv);
        const __half2* bb = reinterpret_cast<const __half2*>(&wv);
#pragma unroll
        for (int e = 0; e < 4; ++e) a[e] = __hmul2(a[e], bb[e]);
      }
      return uv;
    } else {
      float g[8];
      IO<T>::to_f32x8(uv, g);
      if (GATED) {
        float w8[8];
        IO<T>::to_f32x8(wv, w8);
#pragma unroll
        for (int e = 0; e < 8; ++e) g[e] *= w8[e];
      }
      return make_uint4(pack_half2(g[0], g[1]), pack_half2(g[2], g[3]), pack_half2(g[4], g[5]),
                        pack_half2(g[6], g[7]));
    }
  };
  // stage A operand address of (row r of the tile, n2, n1 chunk j)
  auto chunk_dst = [&](int r, int n2, int j) -> uint32_t {
    const int k = (r & 1) * C::KA + n2;
    return bufX + ((r >> 1) * JC + j) * C::SBO_A + (k >> 3) * 128 + (k & 7) * 16;
  };
  // Causal tiles leave TMEM lane quadrants 1 and 3 idle in epilogue 4 (their
  // rows are the discarded n2 >= L2/2 half): those 4 warps prefetch the next
  // tile's (gated) input into spare TMEM columns [192, 256) of their own
  // lanes (the two column slices of a quadrant share lanes: 32 columns each).
  constexpr bool PF = CAUSAL;
  const uint32_t PF_COL = 192 + 32 * slice;
  // live from epilogue 4 of tile t to the start of tile t+1: only stage A^-1
  // (columns < 128) and the next stage A (< NA) write TMEM in between
  static_assert(C::NA <= 192, "prefetch columns are free");
  constexpr int PF_CH = (C::R * C::CH) / 128;  // chunks per idle thread
  const bool idle4 = CAUSAL && (quad & 1);
  const int pf_ii = ((quad >> 1) * 2 + slice) * 32 + lane;  // 0..127 among idle threads
  const int pf_n2 = pf_ii % KROWS, pf_j = (pf_ii / KROWS) % JC, pf_r0 = pf_ii / (KROWS * JC);
  constexpr int PF_RSTEP = 128 / (KROWS * JC);
  static_assert(!PF || (128 % (KROWS * JC) == 0 && PF_CH == 8), "prefetch mapping");
  const int64_t pf_off0 = int64_t(pf_r0) * HN + int64_t(pf_n2 * JC + pf_j) * 8;
  bool prefetched = false;

  int64_t hh = (t0 + wg) / nbt, bt = (t0 + wg) % nbt;
  for (int64_t t = t0 + wg; t < t1; t += kWG, bt += kWG) {
    while (bt >= nbt) { bt -= nbt; ++hh; }
    stage_no = 0;
    stamp(0);
    const int64_t h = phys_head(hh);
    const int64_t tile_base = (bt * C::R * H + h) * N;  // element offset of row (bt*R, h)
    const int rows_left = int(B - bt * C::R < C::R ? B - bt * C::R : C::R);
    const bool new_h = h != cur_h;
    if (new_h) {  // refresh this warpgroup's k_f copy (previous tile's epi2 is long done)
      const uint8_t* src = gkf + h * int64_t(C::KF_BYTES);
      for (uint32_t o = wtid * 16; o < C::KF_BYTES; o += kWGThreads * 16) cp_async16(sKF + o, src + o, true);
      cp_async_commit();
      cur_h = h;
    }

    // ---------------- load (+ gate) the tile's rows straight into the stage A operand
    if (prefetched) {
      if (idle4) {
        uint32_t v[32];
        tmem_ld16(tq + PF_COL, reinterpret_cast<float*>(v));
        tmem_ld16(tq + PF_COL + 16, reinterpret_cast<float*>(v + 16));
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < PF_CH; ++i)
          st_shared_v4(chunk_dst(pf_r0 + i * PF_RSTEP, pf_n2, pf_j), v[4 * i], v[4 * i + 1], v[4 * i + 2],
                       v[4 * i + 3]);
      }
    } else {
      constexpr int NCH = C::R * C::CH;
      constexpr int PER_ALL = NCH / kWGThreads;
      constexpr int PER = PER_ALL < 4 ? PER_ALL : 4;  // loads in flight per batch (register budget)
#pragma unroll 1
      for (int i0 = 0; i0 < PER_ALL; i0 += PER) {
      uint4 uv[PER], wv[PER];
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int r = ld_r0 + (i0 + i) * RSTEP;
        if (r < rows_left) {
          const int64_t goff = tile_base + ld_off0 + int64_t((i0 + i) * RSTEP) * HN;
          uv[i] = *reinterpret_cast<const uint4*>(gu + goff);
          if (GATED) wv[i] = *reinterpret_cast<const uint4*>(gw + goff);
        } else {
          uv[i] = make_uint4(0, 0, 0, 0);
          wv[i] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        // n2 fastest so 8 consecutive threads fill one 128 B core matrix
        const uint4 g = gate8(uv[i], wv[i]);
        st_shared_v4(chunk_dst(ld_r0 + (i0 + i) * RSTEP, ld_n2, ld_j), g.x, g.y, g.z, g.w);
      }
    }
    }
    if (new_h) cp_async_wait_all();
    stamp(1);

    // ---------------- stage A: D[(p,n1)][(re|im|-im, k2)] = X[(p,n1)][(c,n2)] * G_A
    // TMEM column of (block, k2): (k2 / 32) * NA/2 + 32 * block + k2 % 32
    sync_and_issue([&](int hh) {  // half hh: k2 in [32 hh, 32 hh + 32) of every block, one MMA per K step
      constexpr uint32_t idesc = idesc_f16(128, C::NA / 2, true, false);
#pragma unroll
      for (int s = 0; s < 2 * C::KA / 16; ++s)
        mma_f16_ss(tmem + hh * (C::NA / 2), dadd(dXA, 256 * s),
                   dadd(dGA, hh * (C::NA / 16) * C::SBO_GA + 256 * s), idesc, s > 0);
    });

    // ---------------- epilogue 1: twiddle W^{n1 k2}, transpose -> stage B operand (MN-major)
    // Every stage's operand aliases bufX, so stores wait for BOTH halves of
    // the stage (the other half's MMAs may still read bufX); math on the
    // first item only needs this warp's half.
    {
      const int p = m / L1, n1 = m % L1;
      wait_half(slice);
#pragma unroll 1
      for (int sub = 0; sub < 2; ++sub) {
        const int k20 = slice * 32 + sub * 16;  // 16 k2 per item
        const uint32_t c0 = slice * (C::NA / 2) + sub * 16;
        float re[16], im[16], ni[16];
        tmem_ld16(tq + c0, re);
        tmem_ld16(tq + c0 + 32, im);
        if constexpr (C::NEG_A) tmem_ld16(tq + c0 + 64, ni);
        float4 w[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) w[jj] = ld_shared_f4(sTW + tab_off<L2 / 2>(n1, k20 / 2 + jj));
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

    stamp(4);
    // ---------------- stage B: per group of 128 rows (p,k2), contract n1 -> k1
    sync_and_issue([&](int hh) {
      constexpr uint32_t idesc = idesc_f16(128, C::NB, true, false);
#pragma unroll
      for (int gi = hh * (C::P / 4); gi < (hh + 1) * (C::P / 4); ++gi) {
#pragma unroll
        for (int s = 0; s < 2 * L1 / 16; ++s) {
          uint64_t ad = dadd(dXB, gi * 2048 + 2 * s * C::LBO_B);
          uint64_t bd = dadd(dGB, 256 * s);
          mma_f16_ss(tmem + gi * C::NB, ad, bd, idesc, s > 0);
        }
      }
    });

    // ---------------- epilogue 2: pointwise * k_f -> stage B^-1 operand (K-major, own row)
    {
      const int k2 = m & 63;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;  // items 0..3 in half 0, 4..7 in half 1
        const int gi = it / (L1 / 8), k1c = it % (L1 / 8);
        const int row = gi * 128 + m;  // (p, k2) with p = 2 gi + m / 64
        if (i == 0) wait_half(0);
        const uint32_t col = gi * C::NB + k1c * 8;
        float re[8], im[8], ni[8];
        tmem_ld8(tq + col, re);
        tmem_ld8(tq + col + L1, im);
        tmem_ld8(tq + col + 2 * L1, ni);
        float4 kf[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kf[jj] = ld_shared_f4(sKF + tab_off<L1 / 2>(k2, k1c * 4 + jj));
        tmem_ld_wait();
        cmul8(re, im, ni, kf);
        if (i == 0) wait_half(1);  // stores may overwrite operands of the second half
        st_half8(bufX + (row >> 3) * C::SBO_BP + k1c * 128 + (row & 7) * 16, re);
        st_half8(bufX + (row >> 3) * C::SBO_BP + (L1 / 8 + k1c) * 128 + (row & 7) * 16, im);
      }
    }

    stamp(7);
    // ---------------- stage B^-1: contract k1 -> n1
    sync_and_issue([&](int hh) {
      constexpr uint32_t idesc = idesc_f16(128, C::NB, false, false);
#pragma unroll
      for (int gi = hh * (C::P / 4); gi < (hh + 1) * (C::P / 4); ++gi) {
#pragma unroll
        for (int s = 0; s < 2 * L1 / 16; ++s) {
          uint64_t ad = dadd(dXBP, gi * 16 * C::SBO_BP + 256 * s);
          uint64_t bd = dadd(dGBI, 256 * s);
          mma_f16_ss(tmem + gi * C::NB, ad, bd, idesc, s > 0);
        }
      }
    });

    // ---------------- epilogue 3: conj twiddle, transpose -> stage A^-1 operand (MN-major B)
    {
      const int k2 = m & 63;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;
        const int gi = it / (L1 / 8), n1c = it % (L1 / 8);
        const int p = gi * 2 + (m >> 6);
        if (i == 0) wait_half(0);
        const uint32_t col = gi * C::NB + n1c * 8;
        float re[8], im[8], nr[8];
        tmem_ld8(tq + col, re);
        tmem_ld8(tq + col + L1, im);
        tmem_ld8(tq + col + 2 * L1, nr);
        float4 w[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) w[jj] = ld_shared_f4(sTWT + tab_off<L1 / 2>(k2, n1c * 4 + jj));
        tmem_ld_wait();
        cmulc8(re, im, nr, w);
        if (i == 0) wait_half(1);  // stores may overwrite operands of the second half
        const int ng = (p * L1) / 8 + n1c;
        st_half8(bufX + ng * C::SBO_XA + (k2 >> 3) * 128 + (k2 & 7) * 16, re);
        st_half8(bufX + ng * C::SBO_XA + ((L2 + k2) >> 3) * 128 + (k2 & 7) * 16, im);
      }
    }

    stamp(10);
    // ---------------- stage A^-1: D[(c',n2)][(p,n1)] = G_A^-1 * X[(c,k2)][(p,n1)]
    sync_and_issue([&](int hh) {  // half hh: output columns (p, n1) in [64 hh, 64 hh + 64)
      constexpr uint32_t idesc = idesc_f16(128, 64, false, true);
#pragma unroll
      for (int s = 0; s < 2 * L2 / 16; ++s) {
        uint64_t ad = dadd(dGAI, 256 * s);
        uint64_t bd = dadd(dXAI, hh * 8 * C::SBO_XA + 256 * s);
        mma_f16_ss(tmem + hh * 64, ad, bd, idesc, s > 0);
      }
    });

    // ---------------- epilogue 4: (gate), convert, store y
    {
      const int cp = m >> 6;
      const bool has_next = t + kWG < t1;
      if (idle4) {  // warp-uniform: prefetch the next tile's input into TMEM
        if (has_next) {
          int64_t hh2 = hh, bt2 = bt + kWG;
          while (bt2 >= nbt) { bt2 -= nbt; ++hh2; }
          const int64_t h2 = phys_head(hh2);
          const int64_t base2 = (bt2 * C::R * H + h2) * N;
          const int left2 = int(B - bt2 * C::R < C::R ? B - bt2 * C::R : C::R);
          uint4 uv[PF_CH], wv[PF_CH];
#pragma unroll
          for (int i = 0; i < PF_CH; ++i) {
            const int r = pf_r0 + i * PF_RSTEP;
            if (r < left2) {
              const int64_t goff = base2 + pf_off0 + int64_t(i * PF_RSTEP) * HN;
              uv[i] = *reinterpret_cast<const uint4*>(gu + goff);
              if (GATED) wv[i] = *reinterpret_cast<const uint4*>(gw + goff);
            } else {
              uv[i] = make_uint4(0, 0, 0, 0);
              wv[i] = make_uint4(0, 0, 0, 0);
            }
          }
          uint32_t v[32];
#pragma unroll
          for (int i = 0; i < PF_CH; ++i) {
            const uint4 g = gate8(uv[i], wv[i]);
            v[4 * i] = g.x; v[4 * i + 1] = g.y; v[4 * i + 2] = g.z; v[4 * i + 3] = g.w;
          }
          tmem_st32(tq + PF_COL, v);
          tmem_st_wait();
        }
      } else if (!CAUSAL || (m & 63) < L2 / 2) {  // warp-uniform
        // this warp's items cover output columns [64 slice, 64 slice + 64)
        constexpr int NIT = C::P * (L1 / 8);  // (pair, 8-wide n1 chunk) items
        constexpr int PER = NIT / 2;
        int64_t goff[PER];
        bool ok[PER];
        uint4 vv[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int it = slice * PER + i;
          const int p = it / (L1 / 8), n1c = it % (L1 / 8);
          ok[i] = 2 * p + cp < rows_left;
          goff[i] = tile_base + st_off0 + int64_t(2 * p) * HN + n1c * 8;
          if (GATED && ok[i]) vv[i] = *reinterpret_cast<const uint4*>(gv + goff[i]);
        }
        wait_half(slice);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int it = slice * PER + i;
          const int p = it / (L1 / 8), n1c = it % (L1 / 8);
          float o[8];
          tmem_ld8(tq + p * L1 + n1c * 8, o);
          tmem_ld_wait();
          if (GATED) {
            float v8[8];
            IO<T>::to_f32x8(vv[i], v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] *= v8[e];
          }
          uint4 st;
          st.x = IO<T>::pack2(o[0], o[1]);
          st.y = IO<T>::pack2(o[2], o[3]);
          st.z = IO<T>::pack2(o[4], o[5]);
          st.w = IO<T>::pack2(o[6], o[7]);
          if (ok[i]) *reinterpret_cast<uint4*>(gy + goff[i]) = st;
        }
      }
    }
    stamp(13);
    tc_fence_before();
    wg_sync();  // TMEM columns and bufX are reused by the next tile
    stamp(14);
    ++trace_tile;
    prefetched = PF && (t + kWG < t1);
  }
  __syncthreads();
  if (warp == 0) tmem_dealloc<(kWG * C::TMEM_COLS > 512 ? 512 : kWG * C::TMEM_COLS)>(tmem_slot);
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
  const int64_t tiles = (prm.row_map ? (prm.H / prm.row_L0) * prm.nrow : prm.H) * nbt;
  int grid = int(tiles < prm.num_sms ? tiles : prm.num_sms);
  if (grid < 1) return cudaSuccess;
  kern<<<grid, C::THREADS, C::SMEM, stream>>>(prm);
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

}  // namespace fc

#ifdef FC_TRACE
extern "C" int fc_trace_dump(long long* host) {
  return int(cudaMemcpyFromSymbol(host, fc::fc_trace_buf, sizeof(fc::fc_trace_buf)));
}
#endif
