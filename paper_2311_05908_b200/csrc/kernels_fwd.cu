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

#include "dft_vec.cuh"
#include "fused_common.cuh"
#include "fwd_params.h"
#include "launch_util.h"
#include "sm100.cuh"

namespace fc {

#ifdef FC_TRACE
// experiment-only phase timestamps (CTA 0, warpgroup 0, lane 0 of warps 0..7)
__device__ long long fc_trace_buf[8][64][24];
#endif

#ifndef FC_NEG_B
#define FC_NEG_B 0
#endif
#ifndef FC_A_FULL
#define FC_A_FULL 1
#endif
#ifndef FC_EPI_PIPE
#define FC_EPI_PIPE 0
#endif
#ifndef FC_SPLIT_ISSUE
#define FC_SPLIT_ISSUE 0
#endif
#ifndef FC_EPI1_PIPE
#define FC_EPI1_PIPE 0
#endif
#ifndef FC_CIRC_STG
#define FC_CIRC_STG 1
#endif
#ifndef FC_CIRC_TS
#define FC_CIRC_TS 1
#endif
#ifndef FC_AI_TS
#define FC_AI_TS 0
#endif
#ifndef FC_DIT_KFS
#define FC_DIT_KFS 1
#endif
#ifndef FC_EPI1_UNROLL_DIT  // (experiment: 1 or 2 for every order-3 tile; 0 = the rule below)
#define FC_EPI1_UNROLL_DIT 0
#endif
#ifndef FC_CPL_UNROLL
#define FC_CPL_UNROLL 2
#endif
#ifndef FC_DIT_SLOT_WG
#define FC_DIT_SLOT_WG 0
#endif
#ifndef FC_O3_FRAG
#define FC_O3_FRAG 1
#endif

// Shared-memory plan of the forward kernel: tables | per-warpgroup (k_f,
// operand buffer) | staging.  Causal tiles move their rows with bulk (TMA)
// copies through two slots shared by the warpgroups in tile order: the
// input slot (u [| w], filled a tile ahead) and the output slot (v arrives
// there for the gate; y leaves from it).
template <int L1, bool CAUSAL, bool GATED, int L0I = 1>
struct FwdCfg {
  using C = O2Cfg<L1, CAUSAL>;
  static constexpr bool STG = CAUSAL;
  // circular plain tiles (the multipass inner pass) stage their input rows
  // the same way (one TMA tensor load per tile into a slot shared in tile
  // order, filled a tile ahead) instead of register loads issued in the
  // previous tile's last epilogue
  static constexpr bool CIN = !CAUSAL && !GATED && FC_CIRC_STG;
  static constexpr bool STG_IN = STG || CIN;
  // L0I > 1 (single-pass order 3, causal only): the tile's P complex rows
  // are the L0I decimated inner rows z[n0 + L0I n'] of P / L0I row pairs;
  // real rows of length NROW = L0I * NOUT, RR = R / L0I rows per tile
  static constexpr bool DIT = L0I > 1;
  // L0I = 8 (fft_size 16384): one row pair's 8 inner rows are 256 stage-A
  // rows, two warpgroup tiles -- the warpgroups work on the same pair
  // ("coupled"), warpgroup g holding inner rows n0 = 4 g + p, and meet in
  // epilogue 2 (the outer DFT_8 reads both warpgroups' TMEM) and epilogue 4
  // (each writes 4 of every 8 output samples)
  static constexpr bool CPL = L0I == 8;
  static_assert(!DIT || (CAUSAL && L1 == 32 && (C::P % L0I == 0 || CPL) && (L0I == 2 || L0I == 4 || CPL)),
                "single-pass order 3");
  static constexpr int RR = CPL ? 2 : C::R / L0I;
  static constexpr int NROW = C::NOUT * L0I;
  // Stage B / B^-1 N: re | im only (the negated plane the complex multiply
  // needs is a sign folded into the f32x2 multiplies); FC_NEG_B=1 has the
  // tensor core emit it as a third block of the G_B table instead.
  static constexpr int NBF = FC_NEG_B ? C::NB : (2 * L1 + 15) / 16 * 16;
  // The forward's shared-memory table layout is a compacted copy of the
  // plan image: G_A | G_B, G_B^-1 (only the NBF rows the forward reads) |
  // G_A^-1 (causal: rows n2 < L2/2 only).  Twiddles are not stored: they
  // are computed on the fly (MUFU sin/cos, fp32 recurrences).
  static constexpr uint32_t GB_SM = uint32_t(NBF) * (2 * L1) * 2;
  static constexpr uint32_t S_GA = 0;
  static constexpr uint32_t S_GB = C::al(S_GA + C::GA_BYTES);
  static constexpr uint32_t S_GBI = C::al(S_GB + GB_SM);
  static constexpr uint32_t S_GAI = C::al(S_GBI + GB_SM);
  // circular tiles keep G_A^-1 in TMEM (stage A^-1 reads its A operand
  // there), not in shared memory
  static constexpr bool GAI_TMEM = !CAUSAL && FC_CIRC_TS;
  static constexpr uint32_t TABLES = C::al(S_GAI + (GAI_TMEM ? 0 : C::GAI_FWD_BYTES));
  static constexpr uint32_t ROW_BYTES = NROW * 2;  // one 16-bit input row
  // one u [| w] input slot per warpgroup: a warpgroup refills its own slot
  // for its next tile right after reading it (a whole tile of prefetch
  // distance, past the HBM latency); v arrives in one slot shared in tile order
  static constexpr uint32_t UW_BYTES = STG_IN ? RR * ROW_BYTES * (GATED ? 2 : 1) : 0;
  static constexpr uint32_t V_BYTES = STG ? RR * ROW_BYTES : 0;
  // mbarriers + TMEM slot live at the end of the dynamic buffer (no static
  // shared memory: the dynamic base is 1024-aligned, no alignment slack)
  static constexpr uint32_t BAR_BYTES = 128;
  // per-warpgroup buffers: k_f copy (L0I = 1; the order-3 tiles read their
  // L0I k_f blocks from global memory / L2) and the operand buffer
  static constexpr uint32_t KF_SM = DIT ? 0 : C::al(C::KF_BYTES);
  // order 3: the L0I k_f blocks of the current head (16 KB each, layout.h
  // dit_kf_off) in one buffer both warpgroups read, refilled by bulk copies
  // when the head changes (FC_DIT_KFS=0: epilogue 2 reads them from L2)
  // (measured: L0I = 4 4 % faster, L0I = 2 1 % slower -> L0I = 4 only)
  static constexpr bool KFS = DIT && FC_DIT_KFS && L0I == 4;
  static constexpr uint32_t KFD_BLOCK = 16384;
  static constexpr uint32_t KFD_SM = KFS ? L0I * KFD_BLOCK : 0;
  // per warpgroup: [k_f | operand buffer bufX | u [| w] input slot]; the
  // order-3 tiles and circular tiles keep one slot shared in tile order
  // (measured: per-warpgroup slots made the order-2 kernels 2 % faster, the
  // gated order-3 kernel 20 % and plain L0 = 4 4 % slower -- register
  // spills --, plain L0 = 2 0.7 % faster; circular tiles have no SMEM for two)
  static constexpr bool SLOT_WG = (!DIT || (FC_DIT_SLOT_WG && !CPL)) && !CIN;
  static constexpr uint32_t WG_BYTES = KF_SM + C::al(C::BUFX_BYTES) + (SLOT_WG ? C::al(UW_BYTES) : 0);
  // circular plain tiles (the multipass inner pass): y staging shared by
  // the warpgroups in tile order, leaving by one TMA tensor store each
  static constexpr uint32_t YS_BYTES = (!CAUSAL && !GATED) ? C::R * C::NOUT * 2 : 0;
  static constexpr uint32_t bytes_for(int wg) {
    return C::al(C::al(C::al(C::al(TABLES + wg * WG_BYTES) + (SLOT_WG ? 0 : UW_BYTES)) + V_BYTES) + KFD_SM) + YS_BYTES +
           BAR_BYTES;
  }
  static constexpr int WG = bytes_for(2) <= 227 * 1024 ? 2 : 1;
  static constexpr int THREADS = WG * kWGThreads;
  static constexpr uint32_t OFF_WG = TABLES;
  static constexpr uint32_t UW_IN_WG = KF_SM + C::al(C::BUFX_BYTES);  // the slot's offset in its warpgroup's block
  static constexpr uint32_t OFF_UW = C::al(OFF_WG + WG * WG_BYTES);    // (shared slot, !SLOT_WG)
  static constexpr uint32_t OFF_V = C::al(OFF_UW + (SLOT_WG ? 0 : UW_BYTES));
  static constexpr uint32_t OFF_KFD = C::al(OFF_V + V_BYTES);
  static constexpr uint32_t OFF_YS = C::al(OFF_KFD + KFD_SM);
  static constexpr uint32_t OFF_BAR = OFF_YS + YS_BYTES;
  static constexpr uint32_t SMEM = bytes_for(WG);
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(GB_SM <= C::GB_BYTES, "G_B prefix");
};


// Each CTA runs kWG independent warpgroups; warpgroup g processes tiles
// t0 + g, t0 + g + kWG, ... of the CTA's contiguous tile range, with its own
// TMEM columns, mbarriers, named barrier, k_f copy and operand buffer, so one
// warpgroup's MMAs, memory waits and barriers overlap the other's math.
template <int L1, bool CAUSAL, bool GATED, typename T, int L0I, bool SKP>
__global__ void __launch_bounds__(FwdCfg<L1, CAUSAL, GATED, L0I>::THREADS, 1) fftconv_fwd_o2_kernel(const __grid_constant__ FwdParams prm) {
  using C = O2Cfg<L1, CAUSAL>;
  using F = FwdCfg<L1, CAUSAL, GATED, L0I>;
  constexpr bool DIT = F::DIT;
  constexpr int RR = F::RR;        // real rows per tile
  constexpr int NROW = F::NROW;    // real row length (N)
  constexpr int LF = C::L * L0I;   // the whole transform (fft_size)
  constexpr int kWG = F::WG;
  constexpr int kThreads = F::THREADS;
  constexpr bool CPL = F::CPL;            // coupled warpgroups (order 3, L0I = 8)
  constexpr int TSTEP = CPL ? 1 : kWG;     // tile stride of a warpgroup
  static_assert(!CPL || kWG == 2, "coupled tiles need both warpgroups");
  constexpr bool STG = F::STG;      // input staging by bulk copies (causal: + v slot, y by bulk stores)
  constexpr bool STG_IN = F::STG_IN;  // input staging (causal or circular plain)
  constexpr int L2 = C::L2;
  constexpr bool TS = C::TS_BI;     // stage B^-1 data operand in TMEM
  constexpr int NBF = F::NBF;
  constexpr bool M64 = CAUSAL;      // stage A^-1 as M = 64 MMAs (rows n2 < L2/2 only)
  // epilogues 2/3 prefetch the next item's TMEM load: on for gated order-2
  // tiles (measured with the converged waits: cfg2 -1.4 %, gated N = 512
  // -4 %); plain causal +0.5 %, circular 0 %, and before the converged
  // waits 1-3 % slower on circular tiles (spills), so off there
  // (FC_EPI_PIPE=1 forces it); epilogue 1 likewise (FC_EPI1_PIPE): 1-9 % slower
  constexpr bool EPI_PIPE = (FC_EPI_PIPE || (GATED && !DIT)) && !FC_NEG_B;
  constexpr bool EPI1_PIPE = FC_EPI1_PIPE && !C::NEG_A && !DIT;  // epilogue 1 likewise
  constexpr bool A_FULL = FC_A_FULL && !DIT;  // stage A as one MMA chain (measured: o2 -1.3 %, order 3 +2 %)
  // circular tiles: stage A^-1 reads G_A^-1 from TMEM (loaded once per CTA
  // into warpgroup 0's free columns [128, 192)) as one N = 128 MMA chain:
  // a shared-memory A operand costs ~32 extra cycles per K = 16 MMA
  // (tools/microbench.py) and both halves re-read it
  // (Experiment, off: FC_AI_TS=1.  Measured on B200: circular tiles 4.5 %
  // slower -- the single chain loses the half overlap of epilogue 4 --,
  // causal order 2 within 0.5 %, and the order-3 L0I = 4 instance failed
  // parity.)
  // Causal tiles keep only rows n2 < L2/2 (64 of 128): two N = 64 chains,
  // column half h against a copy of G_A^-1 rotated by 64 h rows (copy 1 in
  // warpgroup 1's free columns), so the useful rows of half h land in lane
  // quadrants 2h, 2h + 1 and every epilogue-4 thread keeps 32 columns
  constexpr bool AI_TS = (FC_AI_TS && kWG == 2 && !DIT) || F::GAI_TMEM;  // (causal: measured +-1 %, off)
  constexpr uint32_t GAI_COL = 128;
  static_assert(!AI_TS || (C::TMEM_COLS == 256 && C::NA <= 128 && (C::P / 2) * NBF <= 128 && C::CA >= 192),
                "TMEM columns [128, 192) of each warpgroup hold a G_A^-1 copy");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  struct Bars {
    uint64_t mma[2][2];  // [warpgroup]: completion of the first / second half of a stage
    uint64_t stg[2][2];  // [u|w slot, v slot][consuming warpgroup]: bulk copy landed
    uint64_t ys;         // circular TMA-y staging: use j - 1 has been read (phase j - 1)
    uint64_t kff;        // order 3: k_f buffer refill r landed (phase r)
    uint64_t e2d[2];     // order 3: [warpgroup] epilogue 2 of its j-th tile done (phase j)
    uint64_t bdone[2];   // coupled tiles: [warpgroup] stage B of its j-th tile complete (phase j)
    uint32_t tmem_slot;
    uint32_t uw_cnt;     // coupled tiles: warpgroups past stage A (the second refills the input slot)
  };
  static_assert(sizeof(Bars) <= F::BAR_BYTES, "barrier block");
  Bars& bb = *reinterpret_cast<Bars*>(smem_raw + F::OFF_BAR);
  auto& mma_bar = bb.mma;
  auto& stg_bar = bb.stg;
  auto& ys_bar = bb.ys;
  auto& tmem_slot = bb.tmem_slot;
  const uint32_t base = smem_u32(smem_raw);
  if (base & 1023u) __trap();  // operand layouts and the 128 B swizzle need 1024-byte alignment
  const uint32_t sGA = base + F::S_GA, sGB = base + F::S_GB, sGBI = base + F::S_GBI, sGAI = base + F::S_GAI;
  const uint32_t sYS = base + F::OFF_YS;
  const uint32_t sV = base + F::OFF_V;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wg = int(warp_uniform(warp >> 3));  // warpgroup
  const int wtid = tid & (kWGThreads - 1);
  const int quad = warp & 3;             // TMEM lane quadrant this warp may access
  const int slice = (warp >> 2) & 1;     // column slice 0..1
  const int m = quad * 32 + lane;        // TMEM lane / MMA row owned by this thread
  const uint32_t sKF = base + F::OFF_WG + wg * F::WG_BYTES;
  const uint32_t bufX = sKF + F::KF_SM;
  const uint32_t sY = bufX + C::BUFX_BYTES / 2;  // causal: y rows staged for the bulk stores
  const int64_t B = prm.B, H = prm.H, N = prm.N;
  const int64_t nbt = (B + RR - 1) / RR;
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
    auto seg = [&](uint32_t dst, uint32_t img_off, uint32_t bytes) {
      for (uint32_t o = tid * 16; o < bytes; o += kThreads * 16) cp_async16(base + dst + o, src + img_off + o, true);
    };
    seg(F::S_GA, C::OFF_GA, C::GA_BYTES);
    seg(F::S_GB, prm.kcn ? prm.off_gb : C::OFF_GB, F::GB_SM);  // (compacted copies: slow-digit skip)
    seg(F::S_GBI, prm.kcn ? prm.off_gbi : C::OFF_GBI, F::GB_SM);
    if (!F::GAI_TMEM) seg(F::S_GAI, C::OFF_GAI, C::GAI_FWD_BYTES);
    cp_async_commit();
  }
  if (tid == 0) {
    for (int g = 0; g < kWG; ++g) {
      mbar_init(&mma_bar[g][0], 1);
      mbar_init(&mma_bar[g][1], 1);
      mbar_init(&stg_bar[0][g], 1);
      mbar_init(&stg_bar[1][g], 1);
    }
    mbar_init(&ys_bar, 1);
    mbar_init(&bb.kff, 1);
    mbar_init(&bb.e2d[0], 1);
    mbar_init(&bb.e2d[1], 1);
    bb.uw_cnt = 0;
    mbar_init(&bb.bdone[0], 1);
    mbar_init(&bb.bdone[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<(kWG * C::TMEM_COLS > 512 ? 512 : kWG * C::TMEM_COLS)>(&tmem_slot);
  cp_async_wait_all();
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (AI_TS) {
    // G_A^-1 (128 rows (n2 half, c', n2 mod 32) x K = 2 L2 fp16, K-major
    // canonical in the table image) -> TMEM lane = row, column j = K pair
    // (2j, 2j + 1); warp w writes lanes of quadrant w & 3, K range quarter w >> 2
    constexpr int KQ = 2 * L2 / (kThreads / 128);  // K elements per thread
    const int k0 = (warp >> 2) * KQ;
    const uint8_t* g = reinterpret_cast<const uint8_t*>(prm.tables) + C::OFF_GAI;
#pragma unroll
    for (int cp = 0; cp < (M64 ? 2 : 1); ++cp) {
      const int r = ((warp & 3) * 32 + lane + 64 * cp) & 127;  // table row held by this lane in copy cp
      const uint32_t tg = warp_uniform(tmem_slot) + cp * C::TMEM_COLS + GAI_COL + (uint32_t((warp & 3) * 32) << 16);
#pragma unroll
      for (int k = k0; k < k0 + KQ; k += 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(g + (r >> 3) * C::SBO_GAI + (k >> 3) * 128 + (r & 7) * 16);
        tmem_st4(tg + k / 2, v.x, v.y, v.z, v.w);
      }
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const uint32_t tmem = warp_uniform(tmem_slot) + wg * C::TMEM_COLS;
  const uint32_t tq = tmem + (uint32_t(quad * 32) << 16);  // this warp's lane quadrant
  uint64_t* bars = mma_bar[wg];
  const uint32_t bar_id = 1 + wg;  // named barrier of this warpgroup
  uint32_t phase = 0;
  int64_t cur_h = -1;

  // Input staging (STG).  Slot `kind` (0: the tile's u [| w] rows, 1: its v
  // rows) is filled for tile t by one elected thread with one bulk copy per
  // row, completing on stg_bar[kind][(t - t0) % kWG]; the warpgroup that
  // consumes tile t refills the slot for tile t + 1 right after it has read
  // it, so fills (and reads) follow tile order and each slot's fill for the
  // next warpgroup's tile overlaps the rest of the current tile.
  auto fill = [&](int kind, int64_t t, int64_t th, int64_t tb) {  // tile t = th * nbt + tb
    const int64_t tbase = (tb * RR * H + phys_head(th)) * N;
    const int rows = int(B - tb * RR < RR ? B - tb * RR : RR);
    uint64_t* bar = &stg_bar[kind][CPL ? 0 : (t - t0) % kWG];
    const uint32_t sUW = F::SLOT_WG ? base + F::OFF_WG + uint32_t((t - t0) % kWG) * F::WG_BYTES + F::UW_IN_WG
                                    : base + F::OFF_UW;  // the consumer's slot
    const int planes = (kind == 0 && GATED) ? 2 : 1;
    if (prm.tma_io) {  // one tensor copy per plane; rows past B arrive as zeros (full box counted)
      mbar_arrive_expect_tx(bar, uint32_t(RR * planes) * F::ROW_BYTES);
      const int hc = int(phys_head(th)), b0 = int(tb * RR);
      if (kind == 0) {
        tma_load_4d(sUW, &prm.tmap_u, 0, 0, hc, b0, bar);
        if (GATED) tma_load_4d(sUW + RR * F::ROW_BYTES, &prm.tmap_w, 0, 0, hc, b0, bar);
      } else if (CPL) {  // (n0, n2, n1)-ordered boxes, one per row (api.cu make_tmap_cpl)
        tma_load_4d(sV, &prm.tmap_v, 0, 0, 0, int(b0 * H + hc), bar);
        tma_load_4d(sV + F::ROW_BYTES, &prm.tmap_v, 0, 0, 0, int((b0 + 1) * H + hc), bar);
      } else {
        tma_load_4d(sV, &prm.tmap_v, 0, 0, hc, b0, bar);
      }
      return;
    }
    mbar_arrive_expect_tx(bar, uint32_t(rows * planes) * F::ROW_BYTES);
    for (int r = 0; r < rows; ++r) {
      const int64_t go = tbase + r * H * N;
      if (kind == 0) {
        bulk_g2s(sUW + r * F::ROW_BYTES, gu + go, F::ROW_BYTES, bar);
        if (GATED) bulk_g2s(sUW + (RR + r) * F::ROW_BYTES, gw + go, F::ROW_BYTES, bar);
      } else {
        bulk_g2s(sV + r * F::ROW_BYTES, gv + go, F::ROW_BYTES, bar);
      }
    }
  };
  uint32_t stg_phase[2] = {0, 0};
  auto stg_wait = [&](int kind) {  // every thread waits (bulk-copied data)
    mbar_wait(&stg_bar[kind][CPL ? 0 : wg], stg_phase[kind]);
    stg_phase[kind] ^= 1;
  };
  // output slot hand-over for tile t: v landed (gated) or the previous
  // tile's y stores have read the slot (plain)
  auto release_out = [&](int64_t t, int64_t th, int64_t tb) {
    if (GATED) fill(1, t, th, tb);
    else mbar_arrive(&stg_bar[1][CPL ? 0 : (t - t0) % kWG]);
  };
#ifdef FC_HANG_DEBUG
  if (tid == 0 && blockIdx.x == 0) printf("smem base %u bars %u (mma, stg, ys, kff, e2d)\n", base, base + F::OFF_BAR);
#endif
  // PDL: everything above (tables, barriers, TMEM) overlapped the previous
  // kernel (the k_f precompute); u, w, v and k_f are read only below
  griddep_wait();
  griddep_launch();
  // order 3: head hh's L0I k_f blocks -> the shared buffer (one elected thread)
  const uint32_t sKFD = base + F::OFF_KFD;
  auto kf_fill = [&](int64_t hh_) {
    const uint8_t* src = gkf + phys_head(hh_) * int64_t(L0I) * C::KF_BYTES;
    mbar_arrive_expect_tx(&bb.kff, F::KFD_SM);
#pragma unroll
    for (int k0 = 0; k0 < L0I; ++k0) bulk_g2s(sKFD + k0 * F::KFD_BLOCK, src + k0 * C::KF_BYTES, F::KFD_BLOCK, &bb.kff);
  };
  if (F::KFS && tid == 0) kf_fill(t0 / nbt);
  if (STG_IN && tid == 0) {
    for (int64_t t = t0; t < t0 + (F::SLOT_WG ? kWG : 1) && t < t1; ++t) fill(0, t, t / nbt, t % nbt);
    if (STG) release_out(t0, t0 / nbt, t0 % nbt);
  }
  // a thread other than the MMA issuer (warp 1 of the warpgroup) refills the slots
  auto filler = [&]() { return (wtid >> 5) == 1 && elect_one(); };

  // UMMA shared-memory descriptors: built once, offsets added as (bytes >> 4)
  const uint64_t dXA = smem_desc(bufX, 128, C::SBO_A);          // stage A operand (MN-major)
  const uint64_t dGA = smem_desc(sGA, 128, C::SBO_GA);
  const uint64_t dXB = smem_desc(bufX, C::LBO_B, 128);          // stage B operand (MN-major)
  const uint64_t dGB = smem_desc(sGB, 128, C::SBO_GB);
  const uint64_t dXBP = smem_desc(bufX, 128, C::SBO_BP);        // stage B^-1 operand (K-major, !TS)
  const uint64_t dGBI = smem_desc(sGBI, 128, C::SBO_GB);
  const uint64_t dGAI = smem_desc(sGAI, 128, C::SBO_GAI);
  const uint64_t dXAI = smem_desc(bufX, 128, C::SBO_XA);        // stage A^-1 operand (MN-major B)
  auto dadd = [](uint64_t d, uint32_t off) { return d + uint64_t(off >> 4); };

  int trace_tile = 0;
  auto stamp = [&](int k) {
#ifdef FC_TRACE
    if (blockIdx.x == 0 && wg == 0 && (wtid & 31) == 0 && trace_tile < 64)
      fc_trace_buf[wtid >> 5][trace_tile][k] = clock64();
#endif
  };
  int stage_no = 0;
  auto wg_sync = [&] { named_sync(bar_id, kWGThreads); };
  // Operands written -> warpgroup barrier -> one elected thread issues the
  // stage as two halves, each committed to its own mbarrier so the epilogue
  // of the first half overlaps the MMAs of the second.
  // split = true (experiment, FC_SPLIT_ISSUE=1, off): the halves are
  // independent MMA chains issued by two threads (warps 0 and 4), so no warp
  // blocks on the tensor queue for a whole stage (a half with no MMAs must
  // not be split: its commit would complete at once).  Measured 2-8 %
  // slower on every workload.
  auto sync_and_issue = [&](auto&& issue_half, bool split = false, bool cta = false, uint64_t* extra = nullptr) {
    fence_async_smem();
    tc_fence_before();
    if (cta) named_sync(3, kThreads);  // coupled tiles: both warpgroups wrote this stage's operands
    else wg_sync();
    stamp(2 + 3 * stage_no);
    if (FC_SPLIT_ISSUE && split) {
      if (wtid < 32 && elect_one()) {
        tc_fence_after();
        issue_half(0);
        mma_commit(&bars[0]);
      } else if ((wtid >> 5) == 4 && elect_one()) {
        tc_fence_after();
        issue_half(1);
        mma_commit(&bars[1]);
      }
    } else if (wtid < 32 && elect_one()) {
      tc_fence_after();
      issue_half(0);
      mma_commit(&bars[0]);
      issue_half(1);
      mma_commit(&bars[1]);
      if (extra) mma_commit(extra);  // a once-per-tile completion signal (coupled tiles)
    }
    stamp(3 + 3 * stage_no);
    ++stage_no;
    phase ^= 1;  // both barriers complete once per stage
  };
  auto wait_half = [&](int hh) {  // parity of the stage issued last
    mbar_wait_warp(&bars[hh], phase ^ 1);
    tc_fence_after();
  };

  // Row orders.  Stage A rows (TMEM lanes) m <-> (pair p, n1) and stage B /
  // B^-1 rows (group gi, lane m) <-> (p, k2) put 4 pairs x 8 consecutive n1
  // (k2) in each warp, so every twiddle / k_f table word a warp reads is
  // shared by 4 lanes (one shared-memory wavefront per 8 distinct words).
  constexpr int JC = L1 / 8;    // 8-element n1 chunks
  // frequency-sparse slow-digit skip: stage B / pointwise / B^-1 run over
  // kc of the JC chunks of 8 k1 (kept chunk j = original chunk k1c_of(j));
  // stage-B columns re | im of the kept k1, B^-1 contracts 2 * kk of them
  static_assert(!SKP || (!DIT && TS && !FC_NEG_B && L1 == 32), "slow-digit skip variant");
  const int kc = SKP ? prm.kcn : JC;
  const int kk = 8 * kc;
  const uint32_t k1map = kc < JC ? prm.k1map : 0xE4u;  // identity 0, 1, 2, 3
  auto k1c_of = [&](int j) { return int((k1map >> (2 * j)) & 3u); };
  const int pA = ((m >> 5) / JC) * 4 + ((m >> 3) & 3), n1A = ((m >> 5) % JC) * 8 + (m & 7);
  // Order 3 (DIT): inner row p = q L0I + n0 holds z_q[n0 + L0I n'], so the
  // transform index of stage-A row (p, n1) is n0 + L0I n1 and the stage-B /
  // B^-1 rows put n0 where the outer DFT_L0I can reach it: its low bit in
  // the group gi (both in this thread's TMEM columns), its high bit (L0I =
  // 4; for L0I = 2 the pair q) in lane bit 3 (one shuffle away).
  auto rowB_p = [&](int gi) { return DIT ? ((m >> 3) & 1) * 2 + gi : (gi >> 1) * 4 + ((m >> 3) & 3); };
  auto rowB_k2 = [&](int gi) {
    return DIT ? (m & 7) + 8 * (m >> 5) + 32 * ((m >> 4) & 1) : (gi & 1) * 32 + (m >> 5) * 8 + (m & 7);
  };
  // Twiddle-recurrence constants: epilogue 1 steps k2 by 2 at fixed
  // transform index e1 = n0 + L0I n1 (W^{2 e1}); epilogue 3 steps n1 at
  // fixed (n0, k2) (W^{L0I k2}, W^{2 L0I k2}) for the thread's two k2.
  auto tw_at = [&](int e1, int k2) { return wroot<LF>(e1 * k2); };  // W_LF^{e1 k2}
  // inner row p of this warpgroup's tile -> n0 (coupled tiles: n0 = 4 wg + p)
  auto n0_of_p = [&](int p) { return CPL ? 4 * wg + p : p % L0I; };
  const int e1A = n0_of_p(pA) + L0I * n1A;
  const float2 tw1_c2 = tw_at(e1A, 2);
  float4 tw3_c[2];
#pragma unroll
  for (int par = 0; par < 2; ++par) {
    const int k2 = rowB_k2(par);
    const float2 w1 = tw_at(L0I, k2), w2 = tw_at(2 * L0I, k2);
    tw3_c[par] = make_float4(w1.x, w1.y, w2.x, w2.y);
  }
  // 8-row group of stage-B row (p, k2) (k2 a multiple of 8)
  auto grpB = [](int p, int k2) {
    return DIT ? (p & 1) * 16 + ((k2 >> 3) & 3) * 4 + ((k2 >> 5) & 1) * 2 + (p >> 1)
               : (((p >> 2) * 2 + (k2 >> 5)) * 16) + ((k2 & 31) >> 3) * 4 + (p & 3);
  };

  // Input loader: each warp instruction reads 32 consecutive 16 B chunks of
  // one row (memory chunk cm = n2 * JC + j); lanes are permuted so that each
  // 8-lane phase writes 8 distinct n2 of one core matrix (conflict-free).
  // Thread chunk i is row r0 + i * RSTEP with (n2, j) fixed.
  constexpr int KROWS = C::KA;  // n2 rows per row
  constexpr int WPR = KROWS * JC / 32;  // warp instructions per row
  constexpr int RSTEP = 8 / WPR;
  constexpr int NCH = RR * (NROW / 8);
  constexpr int PER_ALL = NCH / kWGThreads;  // chunks per thread and tile
  static_assert(WPR >= 1 && 8 % WPR == 0 && NCH % kWGThreads == 0, "loader mapping");
  const int64_t HN = H * N;
  const uint32_t sUW = F::SLOT_WG ? bufX + C::al(C::BUFX_BYTES) : base + F::OFF_UW;  // this warpgroup's input slot
  // From staging (STG) the lanes of each 8-lane phase take 8 consecutive n2
  // and n1 chunks j rotated so that both the staging read (chunk cm mod 8)
  // and the operand write (n2 mod 8) are bank-conflict-free.
  constexpr int LJC = JC == 4 ? 2 : JC == 2 ? 1 : 0;
  const int ld_n2 = STG_IN ? ((wtid >> 5) % WPR) * (32 / JC) + ((lane >> 3) >> LJC) * 8 + (lane & 7)
                        : (((wtid >> 5) % WPR) * 32 + (lane % (32 / JC)) * JC + lane / (32 / JC)) / JC;
  const int ld_j = STG_IN ? (((lane & 7) >> (3 - LJC)) + (lane >> 3)) & (JC - 1)
                       : (((wtid >> 5) % WPR) * 32 + (lane % (32 / JC)) * JC + lane / (32 / JC)) % JC;
  const int ld_r0 = (wtid >> 5) / WPR;
  const int ld_cm = ld_n2 * JC + ld_j;
  const int64_t ld_off0 = int64_t(ld_r0) * HN + int64_t(ld_cm) * 8;

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
  // stage A operand address of chunk i of this thread: row r = 2p + c of the
  // tile, (n2, n1 chunk j) -> K index c*KA + n2, 8-row group of (p, 8j)
  auto chunk_dst = [&](int i) -> uint32_t {
    const int r = ld_r0 + i * RSTEP, p = r >> 1;
    const int k = (r & 1) * C::KA + ld_n2;
    const int g8 = ((p >> 2) * JC + ld_j) * 4 + (p & 3);
    return bufX + g8 * C::SBO_A + (k >> 3) * 128 + (k & 7) * 16;
  };
  auto load_chunks = [&](int64_t tbase, int left, uint4* uv, uint4* wv) {
#pragma unroll
    for (int i = 0; i < PER_ALL; ++i) {
      if (ld_r0 + i * RSTEP < left) {
        const int64_t goff = tbase + ld_off0 + int64_t(i * RSTEP) * HN;
        uv[i] = *reinterpret_cast<const uint4*>(gu + goff);
        if (GATED) wv[i] = *reinterpret_cast<const uint4*>(gw + goff);
      } else {
        uv[i] = make_uint4(0, 0, 0, 0);
        wv[i] = make_uint4(0, 0, 0, 0);
      }
    }
  };
  auto build_from_staging = [&](int left) {  // staging rows -> (gated) stage A operand
#pragma unroll
    for (int i = 0; i < PER_ALL; ++i) {
      const int r = ld_r0 + i * RSTEP;
      uint4 uv = make_uint4(0, 0, 0, 0), wv = make_uint4(0, 0, 0, 0);
      if (r < left) {
        uv = ld_shared_u4(sUW + r * F::ROW_BYTES + ld_cm * 16);
        if (GATED) wv = ld_shared_u4(sUW + (RR + r) * F::ROW_BYTES + ld_cm * 16);
      }
      const uint4 g = gate8(uv, wv);
      st_shared_v4(chunk_dst(i), g.x, g.y, g.z, g.w);
    }
  };
  // Order 3 (DIT): a thread's super-chunk (row r, n2, j) is the 8 L0I
  // samples [8 L0I (n2 JC + j), +8 L0I) of real row r = 2q + c; gated, then
  // de-interleaved into the L0I operand chunks of inner rows p = q L0I + n0
  // (samples n0 + L0I (8 j + e + 32 n2), e < 8).
  constexpr int PER_SC = DIT ? RR * (NROW / (8 * L0I)) / kWGThreads : 1;
  auto build_dit = [&](int left) {
    if constexpr (CPL) {
      // coupled tiles: this warpgroup's inner rows n0 = 4 wg + p are the 8
      // bytes at 8 wg of every 16 B chunk (chunk sc = sample n' = 8 (n2 JC +
      // j) + sc of the row, its 8 n0; the thread's 8 chunks are one 128 B
      // line, staged 128 B swizzled so 8 lanes' lines hit distinct banks):
      // 16 B loads, this warpgroup's halves gated on pairs of chunks, then
      // transposed into the 4 operand chunks (p, j)
      static_assert(PER_SC == 1, "coupled build");
      const int r = ld_r0;
      uint32_t wd[16];  // [sc][2]: halves (p 0, 1), (p 2, 3) of chunk sc
      auto half8 = [&](uint4 q) { return wg ? make_uint2(q.z, q.w) : make_uint2(q.x, q.y); };
#pragma unroll
      for (int sp = 0; sp < 4; ++sp) {
        uint4 uv = make_uint4(0, 0, 0, 0), wv = make_uint4(0, 0, 0, 0);
        if (r < left) {
          const uint32_t o = r * F::ROW_BYTES + (ld_cm * L0I + 2 * sp) * 16;
          const uint2 a = half8(ld_shared_u4(sUW + swz128(o))), b = half8(ld_shared_u4(sUW + swz128(o + 16)));
          uv = make_uint4(a.x, a.y, b.x, b.y);
          if (GATED) {
            const uint32_t ow = RR * F::ROW_BYTES + o;
            const uint2 c = half8(ld_shared_u4(sUW + swz128(ow))), d = half8(ld_shared_u4(sUW + swz128(ow + 16)));
            wv = make_uint4(c.x, c.y, d.x, d.y);
          }
        }
        const uint4 g = gate8(uv, wv);
        wd[4 * sp + 0] = g.x; wd[4 * sp + 1] = g.y; wd[4 * sp + 2] = g.z; wd[4 * sp + 3] = g.w;
      }
      const int c = r & 1, k = c * C::KA + ld_n2;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        uint32_t o[4];
#pragma unroll
        for (int t2 = 0; t2 < 4; ++t2)  // samples n' = 2 t2, 2 t2 + 1 of inner row p
          o[t2] = __byte_perm(wd[2 * (2 * t2) + (p >> 1)], wd[2 * (2 * t2 + 1) + (p >> 1)], (p & 1) ? 0x7632u : 0x5410u);
        const int g8 = ld_j * 4 + p;
        st_shared_v4(bufX + g8 * C::SBO_A + (k >> 3) * 128 + (k & 7) * 16, o[0], o[1], o[2], o[3]);
      }
    } else {
#pragma unroll
    for (int i = 0; i < PER_SC; ++i) {
      const int r = ld_r0 + i * RSTEP;
      uint32_t wd[4 * L0I];
#pragma unroll
      for (int sc = 0; sc < L0I; ++sc) {
        uint4 uv = make_uint4(0, 0, 0, 0), wv = make_uint4(0, 0, 0, 0);
        if (r < left) {
          const uint32_t o = (ld_cm * L0I + sc) * 16;
          uv = ld_shared_u4(sUW + r * F::ROW_BYTES + o);
          if (GATED) wv = ld_shared_u4(sUW + (RR + r) * F::ROW_BYTES + o);
        }
        const uint4 g = gate8(uv, wv);
        wd[4 * sc + 0] = g.x; wd[4 * sc + 1] = g.y; wd[4 * sc + 2] = g.z; wd[4 * sc + 3] = g.w;
      }
      const int q = r >> 1, c = r & 1, k = c * C::KA + ld_n2;
#pragma unroll
      for (int n0 = 0; n0 < L0I; ++n0) {
        // output word t = samples (n0 + L0I (2t), n0 + L0I (2t + 1)) of the super-chunk
        uint32_t o[4];
#pragma unroll
        for (int t2 = 0; t2 < 4; ++t2) {
          const int a = n0 + L0I * 2 * t2, b = a + L0I;  // half indices
          o[t2] = __byte_perm(wd[a >> 1], wd[b >> 1], ((a & 1) ? 0x32u : 0x10u) | ((b & 1) ? 0x7600u : 0x5400u));
        }
        const int p = q * L0I + n0;
        const int g8 = ((p >> 2) * JC + ld_j) * 4 + (p & 3);
        st_shared_v4(bufX + g8 * C::SBO_A + (k >> 3) * 128 + (k & 7) * 16, o[0], o[1], o[2], o[3]);
      }
    }
    }
  };
  auto store_chunks = [&](const uint4* uv, const uint4* wv) {
#pragma unroll
    for (int i = 0; i < PER_ALL; ++i) {
      const uint4 g = gate8(uv[i], wv[i]);
      st_shared_v4(chunk_dst(i), g.x, g.y, g.z, g.w);
    }
  };

  // Epilogue-4 geometry.  Output lane m holds G_AI row (n2 half, c', n2 mod
  // 32) (plan.cpp).  Causal: two M = 64 MMAs put column half hh in lanes
  // 16 hh .. 16 hh + 15 of every quadrant, rows q*16 + lane%16 (n2 < 32).
  // (TMEM stage A^-1, causal: half h in lane quadrants 2h, 2h + 1, row
  // (c' = quad & 1, n2 = lane), columns [64 h, 64 h + 64))
  constexpr int OUT_COLS = M64 ? 32 : 64;  // output columns per thread (this slice)
  const int o_hh = M64 ? (AI_TS ? quad >> 1 : lane >> 4) : slice;
  const int o_row = M64 ? (AI_TS ? (quad & 1) * 32 + lane : quad * 16 + (lane & 15)) : m;
  const int o_cp = (o_row >> 5) & 1, o_n2 = (o_row >> 6) * 32 + (o_row & 31);
  const int o_col0 = M64 ? o_hh * 64 + slice * 32 : slice * 64;  // first (p, n1) column of this thread
  const uint32_t o_tcol = M64 ? (AI_TS ? o_hh * 64 : 0) + slice * 32 : slice * 64;  // its TMEM column

  int64_t hh = (t0 + (CPL ? 0 : wg)) / nbt, bt = (t0 + (CPL ? 0 : wg)) % nbt;
  bool loaded = false;  // the tile's operand was stored by the previous tile's epilogue 4
  bool ys_pending = false;  // (wtid 0) a TMA store of y from sYS is in flight
  for (int64_t t = t0 + (CPL ? 0 : wg); t < t1; t += TSTEP, bt += TSTEP) {
    while (bt >= nbt) { bt -= nbt; ++hh; }
    stage_no = 0;
    stamp(0);
    const int64_t h = phys_head(hh);
    const int64_t tile_base = (bt * RR * H + h) * N;  // element offset of row (bt*R, h)
    const int rows_left = int(B - bt * RR < RR ? B - bt * RR : RR);
    const bool new_h = !DIT && h != cur_h;
    if (new_h) {  // refresh this warpgroup's k_f copy (previous tile's epi2 is long done)
      const uint8_t* src = gkf + h * int64_t(C::KF_BYTES);
      for (uint32_t o = wtid * 16; o < C::KF_BYTES; o += kWGThreads * 16) cp_async16(sKF + o, src + o, true);
      cp_async_commit();
      cur_h = h;
    }
    if constexpr (DIT) {
      stg_wait(0);
      build_dit(rows_left);
    } else if constexpr (STG_IN) {
      stg_wait(0);
      build_from_staging(rows_left);
    } else if (!loaded) {
      uint4 uv[PER_ALL], wv[PER_ALL];
      load_chunks(tile_base, rows_left, uv, wv);
      store_chunks(uv, wv);
    }
    stamp(1);

    // the previous tile's y rows leave from bufX's second half by bulk
    // stores; epilogue 1 rewrites it, so they must have been read by then
    // (the stage-A barrier below publishes this wait to the warpgroup)
    if (STG && filler()) bulk_wait_read0();
    // circular TMA-y tiles: hand the shared y staging to the next user once
    // this warpgroup's previous tensor store has read it
    if (ys_pending) {
      bulk_wait_read0();
      mbar_arrive(&ys_bar);
      ys_pending = false;
    }
    // ---------------- stage A: D[(p,n1)][(re|im|-im, k2)] = X[(p,n1)][(c,n2)] * G_A
    // TMEM column of (block, k2): (k2 / 32) * NA/2 + 32 * block + k2 % 32
    sync_and_issue([&](int h2) {  // half h2: k2 in [32 h2, 32 h2 + 32) of every block, one MMA per K step
      if constexpr (A_FULL) {
        // one N = NA MMA per K step (the G_A rows of both halves are
        // contiguous): the data operand is read from shared memory once
        // instead of once per half (a K = 16 MMA costs ~47 + N/2 cycles,
        // tools/microbench.py); half 1 commits nothing new
        if (h2 == 0) {
          constexpr uint32_t idesc = idesc_f16(128, C::NA, true, false);
#pragma unroll
          for (int s = 0; s < 2 * C::KA / 16; ++s)
            mma_f16_ss(tmem, dadd(dXA, 256 * s), dadd(dGA, 256 * s), idesc, s > 0);
        }
      } else {
        constexpr uint32_t idesc = idesc_f16(128, C::NA / 2, true, false);
#pragma unroll
        for (int s = 0; s < 2 * C::KA / 16; ++s)
          mma_f16_ss(tmem + h2 * (C::NA / 2), dadd(dXA, 256 * s),
                     dadd(dGA, h2 * (C::NA / 16) * C::SBO_GA + 256 * s), idesc, s > 0);
      }
    });
    // this warpgroup's u|w slot has been read by all of it: stage its next tile
    if constexpr (F::SLOT_WG) {
      if (STG_IN && t + kWG < t1 && filler()) fill(0, t + kWG, (t + kWG) / nbt, (t + kWG) % nbt);
    } else if constexpr (CPL) {  // both warpgroups read the slot: the second one past stage A refills it
      if (STG_IN && t + 1 < t1 && filler()) {
        __threadfence_block();
        if (atomicAdd(&bb.uw_cnt, 1u) & 1u) fill(0, t + 1, bt + 1 < nbt ? hh : hh + 1, bt + 1 < nbt ? bt + 1 : 0);
      }
    } else {  // the shared slot goes to tile t + 1 (the other warpgroup's)
      if (STG_IN && t + 1 < t1 && filler()) fill(0, t + 1, bt + 1 < nbt ? hh : hh + 1, bt + 1 < nbt ? bt + 1 : 0);
    }

    // ---------------- epilogue 1: twiddle W^{n1 k2}, transpose -> stage B operand (MN-major)
    // Every stage's operand aliases bufX, so stores wait for BOTH halves of
    // the stage (the other half's MMAs may still read bufX); math on the
    // first item only needs this warp's half.
    if constexpr (EPI1_PIPE) {
      // the second 16-k2 item's TMEM loads are issued right after the first
      // item's wait, so they overlap its math
      wait_half(slice);
      float bre[2][16], bim[2][16];
      const uint32_t cb = slice * (C::NA / 2);
      tmem_ld16(tq + cb, bre[0]);
      tmem_ld16(tq + cb + 32, bim[0]);
#pragma unroll
      for (int sub = 0; sub < 2; ++sub) {
        const int k20 = slice * 32 + sub * 16;
        float4 w[8];
        {
          const float2 a = tw_at(e1A, k20), b = tw_at(e1A, k20 + 1);
          w[0] = make_float4(a.x, b.x, a.y, b.y);
#pragma unroll
          for (int jj = 1; jj < 8; ++jj) w[jj] = cstep(w[jj - 1], tw1_c2);
        }
        tmem_ld_wait();
        if (sub == 0) {
          tmem_ld16(tq + cb + 16, bre[1]);
          tmem_ld16(tq + cb + 16 + 32, bim[1]);
        }
        float* re = bre[sub];
        float* im = bim[sub];
        float ni[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) ni[e] = -im[e];
        cmul8(re, im, ni, w);
        cmul8(re + 8, im + 8, ni + 8, w + 4);
        if (sub == 0) wait_half(slice ^ 1);
#pragma unroll
        for (int hh2 = 0; hh2 < 2; ++hh2) {
          const int mg = grpB(pA, k20 + 8 * hh2);
          st_half8(bufX + mg * 128 + (n1A >> 3) * C::LBO_B + (n1A & 7) * 16, re + 8 * hh2);
          st_half8(bufX + mg * 128 + ((L1 + n1A) >> 3) * C::LBO_B + (n1A & 7) * 16, im + 8 * hh2);
        }
      }
    } else {
      wait_half(slice);
      // both 16-k2 items unrolled (more ILP, 122 registers) measured 1-2 %
      // faster for gated causal and circular tiles and ~1 % slower for plain
      // causal ones on B200
      // (gated order 3 with L0 = 2: 1 -- with the in-place epilogue 4 below
      // 9 % faster; L0 = 4 keeps 2 and the two-pass epilogue 4: 4-7 % faster)
      // (order 3, measured with the fragment epilogue 2: plain L0 = 2 -3.6 %
      // and L0 = 4 -0.8 % with 2; gated L0 = 8 -1.3 % with 1)
      constexpr int kEpi1Unroll = (DIT && FC_EPI1_UNROLL_DIT) ? FC_EPI1_UNROLL_DIT
                                  : DIT ? (GATED ? (L0I == 4 ? 2 : 1) : (L0I <= 4 ? 2 : 1))
                                        : ((GATED && L0I != 2) || !CAUSAL) ? 2 : 1;
#pragma unroll kEpi1Unroll
      for (int sub = 0; sub < 2; ++sub) {
        const int k20 = slice * 32 + sub * 16;  // 16 k2 per item
        const uint32_t c0 = slice * (C::NA / 2) + sub * 16;
        float re[16], im[16], ni[16];
        tmem_ld16(tq + c0, re);
        tmem_ld16(tq + c0 + 32, im);
        if constexpr (C::NEG_A) tmem_ld16(tq + c0 + 64, ni);
        // W^{n1 k2}, k2 = k20 .. k20 + 15: the table pair at k20, then fp32
        // steps by W^{2 n1} (register recurrence instead of 8 table loads)
        float4 w[8];
        {
          const float2 a = tw_at(e1A, k20), b = tw_at(e1A, k20 + 1);
          w[0] = make_float4(a.x, b.x, a.y, b.y);
#pragma unroll
          for (int jj = 1; jj < 8; ++jj) w[jj] = cstep(w[jj - 1], tw1_c2);
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
          const int mg = grpB(pA, k20 + 8 * hh2);
          st_half8(bufX + mg * 128 + (n1A >> 3) * C::LBO_B + (n1A & 7) * 16, re + 8 * hh2);
          st_half8(bufX + mg * 128 + ((L1 + n1A) >> 3) * C::LBO_B + (n1A & 7) * 16, im + 8 * hh2);
        }
      }
    }
    stamp(4);

    // the new head's k_f copy is first read in epilogue 2: wait for this
    // thread's copies here, the warpgroup barrier of stage B publishes them
    if (new_h) cp_async_wait_all();
    // ---------------- stage B: per group of 128 rows (p,k2), contract n1 -> k1
    sync_and_issue([&](int h2) {
      const uint32_t idesc = kc == JC ? idesc_f16(128, NBF, true, false) : idesc_f16(128, 2 * kk, true, false);
#pragma unroll
      for (int gi = h2 * (C::P / 4); gi < (h2 + 1) * (C::P / 4); ++gi) {
#pragma unroll
        for (int s = 0; s < 2 * L1 / 16; ++s)
          mma_f16_ss(tmem + gi * NBF, dadd(dXB, gi * 2048 + 2 * s * C::LBO_B), dadd(dGB, 256 * s), idesc, s > 0);
      }
    }, true, false, CPL ? &bb.bdone[wg] : nullptr);

    // ---------------- epilogue 2: pointwise * k_f -> stage B^-1 operand (own row: TMEM, else K-major smem)
    if constexpr (CPL) {
      // Coupled tiles (L0 = 8): X[f' + 2048 k0] = sum_n0 W_8^{n0 k0}
      // W_256^{n0 k1} Y_n0[f'], n0 = slot + 2 xb + 4 g: the thread reads its
      // (k2, k1 pair) fragment (rows r, r + 8 = xb) from both column blocks
      // (slot) of BOTH warpgroups' TMEM (g) and writes the B^-1 operand of
      // both; warpgroup wg handles k1 chunks 2 wg, 2 wg + 1.  The other
      // warpgroup's stage B is awaited on its once-per-tile barrier (its
      // per-stage barriers may be a stage behind or ahead: parity aliases).
      static_assert(TS && !FC_NEG_B && L1 == 32, "coupled epilogue 2");
      const int fr = lane >> 2, fq = lane & 3;
      const int k2 = fr + 8 * quad + 32 * slice;
      const uint32_t tl0 = tq - uint32_t(wg * C::TMEM_COLS) + (uint32_t(16 * slice) << 16);
      const uint8_t* kfh = gkf + h * int64_t(L0I) * C::KF_BYTES;
      // k_f of the first k1 chunk from L2 before the waits; the second
      // chunk's loads are issued once the first's have been used
      float4 kf[8];
      auto load_kf8 = [&](int k1c) {
#pragma unroll
        for (int k0 = 0; k0 < 8; ++k0)
          kf[k0] = __ldg(reinterpret_cast<const float4*>(kfh + k0 * C::KF_BYTES + dit_kf_off(k2, 4 * k1c + fq)));
      };
      load_kf8(2 * wg);
      mbar_wait_warp(&bb.bdone[wg ^ 1], uint32_t(t - t0) & 1u);
      wait_half(0);
      wait_half(1);
      constexpr float R2 = 0.70710678118654752f;
      constexpr int kCplUnroll = FC_CPL_UNROLL;  // both chunks unrolled: no spills, 2 % faster than 1
#pragma unroll kCplUnroll
      for (int c = 0; c < 2; ++c) {
        const int k1c = 2 * wg + c;
        float yv[2][2][2][4];  // [g][slot][re|im]: {(xb 0, k1), (xb 0, k1 + 1), (xb 1, k1), (xb 1, k1 + 1)}
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int slot = 0; slot < 2; ++slot) {
            const uint32_t col = g * C::TMEM_COLS + slot * NBF + 8 * k1c;
            tmem_ld_16x256b(tl0 + col, yv[g][slot][0]);
            tmem_ld_16x256b(tl0 + col + L1, yv[g][slot][1]);
          }
        // W_256^{n0 k1}, k1 = 8 k1c + 2 fq + e, as f32x2 pairs over e: n0 = 1
        // from MUFU, the others as products W^{i1 k1} W^{i2 k1}, i1 + i2 = n0
        float2 wr[8], wi[8];
        {
          const float2 a = wroot<256>(8 * k1c + 2 * fq), b = wroot<256>(8 * k1c + 2 * fq + 1);
          wr[1] = make_float2(a.x, b.x);
          wi[1] = make_float2(a.y, b.y);
#pragma unroll
          for (int n0 = 2; n0 < 8; ++n0) {
            const int i1 = n0 / 2, i2 = n0 - n0 / 2;
            wr[n0] = fma2(wr[i1], wr[i2], mul2(wi[i1], make_float2(-wi[i2].x, -wi[i2].y)));
            wi[n0] = fma2(wr[i1], wi[i2], mul2(wi[i1], wr[i2]));
          }
        }
        tmem_ld_wait();
        float2 xr[8], xi[8];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int xb = 0; xb < 2; ++xb)
#pragma unroll
            for (int slot = 0; slot < 2; ++slot) {
              const int n0 = slot + 2 * xb + 4 * g;
              const float2 yr = make_float2(yv[g][slot][0][2 * xb], yv[g][slot][0][2 * xb + 1]);
              const float2 yi = make_float2(yv[g][slot][1][2 * xb], yv[g][slot][1][2 * xb + 1]);
              if (n0 == 0) {
                xr[0] = yr; xi[0] = yi;
              } else {  // T = W Y
                xr[n0] = fma2(yr, wr[n0], mul2(yi, make_float2(-wi[n0].x, -wi[n0].y)));
                xi[n0] = fma2(yr, wi[n0], mul2(yi, wr[n0]));
              }
            }
        // DFT_8 (W_8 = e^{-i pi / 4}): radix-2 over n0's high bit, DFT_4 of
        // the even / odd n0, X[k] = E[k] + W_8^k O[k], X[k + 4] = E[k] - W_8^k O[k]
        auto dft4 = [](float2* r, float2* i, int a0, int a1, int a2, int a3, bool inv, float2* orr, float2* oi) {
          const float2 Ar = add2(r[a0], r[a2]), Ai = add2(i[a0], i[a2]);
          const float2 Br = sub2(r[a0], r[a2]), Bi = sub2(i[a0], i[a2]);
          const float2 Cr = add2(r[a1], r[a3]), Ci = add2(i[a1], i[a3]);
          const float2 Dr = sub2(r[a1], r[a3]), Di = sub2(i[a1], i[a3]);
          orr[0] = add2(Ar, Cr); oi[0] = add2(Ai, Ci);
          orr[2] = sub2(Ar, Cr); oi[2] = sub2(Ai, Ci);
          if (!inv) {  // B -+ i D
            orr[1] = add2(Br, Di); oi[1] = sub2(Bi, Dr);
            orr[3] = sub2(Br, Di); oi[3] = add2(Bi, Dr);
          } else {     // B +- i D
            orr[1] = sub2(Br, Di); oi[1] = add2(Bi, Dr);
            orr[3] = add2(Br, Di); oi[3] = sub2(Bi, Dr);
          }
        };
        auto dft8 = [&](float2* r, float2* i, bool inv) {
          float2 er[4], ei[4], odr[4], odi[4];
          dft4(r, i, 0, 2, 4, 6, inv, er, ei);
          dft4(r, i, 1, 3, 5, 7, inv, odr, odi);
          // odd * W_8^{+-k}: k = 1: (1 -+ i) R2, k = 2: -+ i, k = 3: (-1 -+ i) R2
          const float s = inv ? 1.f : -1.f;
          {
            const float2 a = odr[1], b = odi[1];  // (a + i b)(1 + i s) R2
            odr[1] = make_float2(R2 * (a.x - s * b.x), R2 * (a.y - s * b.y));
            odi[1] = make_float2(R2 * (b.x + s * a.x), R2 * (b.y + s * a.y));
          }
          {
            const float2 a = odr[2], b = odi[2];  // (a + i b)(i s)
            odr[2] = make_float2(-s * b.x, -s * b.y);
            odi[2] = make_float2(s * a.x, s * a.y);
          }
          {
            const float2 a = odr[3], b = odi[3];  // (a + i b)(-1 + i s) R2
            odr[3] = make_float2(R2 * (-a.x - s * b.x), R2 * (-a.y - s * b.y));
            odi[3] = make_float2(R2 * (-b.x + s * a.x), R2 * (-b.y + s * a.y));
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            r[k] = add2(er[k], odr[k]); i[k] = add2(ei[k], odi[k]);
            r[k + 4] = sub2(er[k], odr[k]); i[k + 4] = sub2(ei[k], odi[k]);
          }
        };
        dft8(xr, xi, false);
#pragma unroll
        for (int k0 = 0; k0 < 8; ++k0) {  // * k_f[f' + 2048 k0] / 8: kf = {kr_e0, kr_e1, ki_e0, ki_e1}
          const float4 qv = kf[k0];
          const float2 kr = make_float2(qv.x, qv.y), ki = make_float2(qv.z, qv.w);  // (1/8 folded into k_f)
          const float2 zr = fma2(xr[k0], kr, mul2(xi[k0], make_float2(-ki.x, -ki.y)));
          const float2 zi = fma2(xr[k0], ki, mul2(xi[k0], kr));
          xr[k0] = zr; xi[k0] = zi;
        }
        if (c == 0) load_kf8(2 * wg + 1);  // the next chunk's k_f (L2 latency under the rest of this one)
        dft8(xr, xi, true);
#pragma unroll
        for (int n0 = 1; n0 < 8; ++n0) {  // conj twiddle
          const float2 o_r = fma2(xr[n0], wr[n0], mul2(xi[n0], wi[n0]));
          const float2 o_i = fma2(xi[n0], wr[n0], mul2(xr[n0], make_float2(-wi[n0].x, -wi[n0].y)));
          xr[n0] = o_r; xi[n0] = o_i;
        }
        // B^-1 operands of both warpgroups: rows r (xb 0) and r + 8 (xb 1), column kp
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int slot = 0; slot < 2; ++slot) {
            const int na = slot + 4 * g, nb2 = na + 2;
            const uint32_t ca = tl0 + g * C::TMEM_COLS + C::CA + slot * L1 + 4 * k1c;
            tmem_st_16x128b(ca, pack_half2(xr[na].x, xr[na].y), pack_half2(xr[nb2].x, xr[nb2].y));
            tmem_st_16x128b(ca + L1 / 2, pack_half2(xi[na].x, xi[na].y), pack_half2(xi[nb2].x, xi[nb2].y));
          }
      }
      tmem_st_wait();
    } else if constexpr (DIT && FC_O3_FRAG) {
      // Order 3 with no lane shuffles: a 16x256b TMEM fragment gives a
      // thread rows r and r + 8 of its 16-lane block (lane bit 3 = xb: n0's
      // high bit for L0 = 4, the row pair q for L0 = 2) at one (k2, k1 pair),
      // and the two column blocks hold n0's low bit, so every n0 of X[f' +
      // 2048 k0] = sum_n0 W_L0^{n0 k0} W_{32 L0}^{n0 k1} Y_n0[f'] is in the
      // thread: the outer DFT_L0, * k_f / L0, the inverse DFT_L0 and the
      // conjugate twiddle run in registers on f32x2 pairs (k1, k1 + 1), and
      // (L0 = 2) the two rows share each k_f load.  Thread: 16-lane block =
      // slice, r = lane / 4 (k2 = r + 8 quad + 32 slice), kp % 4 = lane % 4
      // (k1 = 8 k1c + 2 (lane % 4) + e, k1c = 0..3, e = 0, 1).
      // (Round 2 before: one row per thread, n0's high bit by shuffles, k_f
      // by 16 B loads from 32 lines per instruction; epilogue 2 took 8.5k of
      // a 17k-cycle L0 = 4 tile, now ~3k.)
      static_assert(TS && !FC_NEG_B && L1 == 32, "order-3 epilogue 2");
      const int fr = lane >> 2, fq = lane & 3;
      const int k2 = fr + 8 * quad + 32 * slice;
      const uint32_t tl = tq + (uint32_t(16 * slice) << 16);  // lane base of the 16-lane block
      const uint8_t* kfh = gkf + h * int64_t(L0I) * C::KF_BYTES;
      auto kf_at = [&](int k0, int k1c) -> float4 {
        const uint32_t off = dit_kf_off(uint32_t(k2), uint32_t(4 * k1c + fq));
        if constexpr (F::KFS) {
          const uint4 v4 = ld_shared_u4(sKFD + k0 * F::KFD_BLOCK + off);
          return make_float4(__uint_as_float(v4.x), __uint_as_float(v4.y), __uint_as_float(v4.z), __uint_as_float(v4.w));
        } else {
          return __ldg(reinterpret_cast<const float4*>(kfh + k0 * C::KF_BYTES + off));
        }
      };
      if constexpr (F::KFS) mbar_wait(&bb.kff, uint32_t(hh - t0 / nbt) & 1u);  // this head's refill landed
      wait_half(0);
      wait_half(1);
#pragma unroll
      for (int bh = 0; bh < 2; ++bh) {  // two k1 chunks per batch of TMEM loads
        // yv[c][slot][re|im] = {(xb 0, k1), (xb 0, k1 + 1), (xb 1, k1), (xb 1, k1 + 1)}
        float yv[2][2][2][4];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int slot = 0; slot < 2; ++slot) {
            const uint32_t col = slot * NBF + 8 * (2 * bh + c);
            tmem_ld_16x256b(tl + col, yv[c][slot][0]);
            tmem_ld_16x256b(tl + col + L1, yv[c][slot][1]);
          }
        float4 kf[2][4];
        float2 wb[2][2];  // W_128^{k1 + e}
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int k0 = 0; k0 < L0I; ++k0) kf[c][k0] = kf_at(k0, 2 * bh + c);
#pragma unroll
          for (int e = 0; e < 2; ++e) wb[c][e] = wroot<32 * L0I>(8 * (2 * bh + c) + 2 * fq + e);
        }
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int k1c = 2 * bh + c;
          if constexpr (L0I == 4) {
            float2 xr[4], xi[4];  // Y_n0, n0 = 2 xb + slot
#pragma unroll
            for (int slot = 0; slot < 2; ++slot)
#pragma unroll
              for (int xb = 0; xb < 2; ++xb) {
                xr[2 * xb + slot] = make_float2(yv[c][slot][0][2 * xb], yv[c][slot][0][2 * xb + 1]);
                xi[2 * xb + slot] = make_float2(yv[c][slot][1][2 * xb], yv[c][slot][1][2 * xb + 1]);
              }
            // W_128^{n0 k1}: n0 = 1 from MUFU, 2 = its square, 3 = 1 * 2
            float2 wr[4], wi[4];
            wr[1] = make_float2(wb[c][0].x, wb[c][1].x);
            wi[1] = make_float2(wb[c][0].y, wb[c][1].y);
            wr[2] = fma2(wr[1], wr[1], mul2(wi[1], make_float2(-wi[1].x, -wi[1].y)));
            wi[2] = mul2(make_float2(2.f * wr[1].x, 2.f * wr[1].y), wi[1]);
            wr[3] = fma2(wr[1], wr[2], mul2(wi[1], make_float2(-wi[2].x, -wi[2].y)));
            wi[3] = fma2(wr[1], wi[2], mul2(wi[1], wr[2]));
            float2 tr[4], ti[4];
            tr[0] = xr[0]; ti[0] = xi[0];
#pragma unroll
            for (int n0 = 1; n0 < 4; ++n0) {  // T = W Y
              tr[n0] = fma2(xr[n0], wr[n0], mul2(xi[n0], make_float2(-wi[n0].x, -wi[n0].y)));
              ti[n0] = fma2(xr[n0], wi[n0], mul2(xi[n0], wr[n0]));
            }
            // S[k0] = sum_n0 W_4^{n0 k0} T[n0], W_4 = -i
            const float2 ar = add2(tr[0], tr[2]), ai = add2(ti[0], ti[2]);
            const float2 br = sub2(tr[0], tr[2]), bi = sub2(ti[0], ti[2]);
            const float2 cr = add2(tr[1], tr[3]), ci = add2(ti[1], ti[3]);
            const float2 dr = sub2(tr[1], tr[3]), di = sub2(ti[1], ti[3]);
            float2 sr[4], si[4];
            sr[0] = add2(ar, cr); si[0] = add2(ai, ci);
            sr[2] = sub2(ar, cr); si[2] = sub2(ai, ci);
            sr[1] = add2(br, di); si[1] = sub2(bi, dr);  // B - i D
            sr[3] = sub2(br, di); si[3] = add2(bi, dr);  // B + i D
            // * k_f[f' + 2048 k0] / 4: kf = {kr_e0, kr_e1, ki_e0, ki_e1}
#pragma unroll
            for (int k0 = 0; k0 < 4; ++k0) {
              const float4 qv = kf[c][k0];
              const float2 kr = make_float2(qv.x, qv.y), ki = make_float2(qv.z, qv.w);  // (1/4 folded into k_f)
              const float2 zr = fma2(sr[k0], kr, mul2(si[k0], make_float2(-ki.x, -ki.y)));
              const float2 zi = fma2(sr[k0], ki, mul2(si[k0], kr));
              sr[k0] = zr; si[k0] = zi;
            }
            // R[n0] = sum_k0 W_4^{-n0 k0} Z[k0]
            const float2 a2r = add2(sr[0], sr[2]), a2i = add2(si[0], si[2]);
            const float2 b2r = sub2(sr[0], sr[2]), b2i = sub2(si[0], si[2]);
            const float2 c2r = add2(sr[1], sr[3]), c2i = add2(si[1], si[3]);
            const float2 d2r = sub2(sr[1], sr[3]), d2i = sub2(si[1], si[3]);
            float2 rr[4], ri[4];
            rr[0] = add2(a2r, c2r); ri[0] = add2(a2i, c2i);
            rr[2] = sub2(a2r, c2r); ri[2] = sub2(a2i, c2i);
            rr[1] = sub2(b2r, d2i); ri[1] = add2(b2i, d2r);  // B' + i D'
            rr[3] = add2(b2r, d2i); ri[3] = sub2(b2i, d2r);  // B' - i D'
#pragma unroll
            for (int n0 = 1; n0 < 4; ++n0) {  // conj twiddle
              const float2 o_r = fma2(rr[n0], wr[n0], mul2(ri[n0], wi[n0]));
              const float2 o_i = fma2(ri[n0], wr[n0], mul2(rr[n0], make_float2(-wi[n0].x, -wi[n0].y)));
              rr[n0] = o_r; ri[n0] = o_i;
            }
            // B^-1 operand (K index c*L1 + k1 -> column (c*L1 + k1) / 2): rows
            // r (xb 0: n0 = slot) and r + 8 (xb 1: n0 = 2 + slot), column kp
#pragma unroll
            for (int slot = 0; slot < 2; ++slot) {
              const uint32_t ca = tl + C::CA + slot * L1 + 4 * k1c;
              tmem_st_16x128b(ca, pack_half2(rr[slot].x, rr[slot].y), pack_half2(rr[2 + slot].x, rr[2 + slot].y));
              tmem_st_16x128b(ca + L1 / 2, pack_half2(ri[slot].x, ri[slot].y), pack_half2(ri[2 + slot].x, ri[2 + slot].y));
            }
          } else {
          // L0 = 2: per row pair xb, n0 = slot; X[k0] = Y_0 + (-1)^k0 W_64^{k1} Y_1
          const float2 wr = make_float2(wb[c][0].x, wb[c][1].x), wi = make_float2(wb[c][0].y, wb[c][1].y);
          const float2 nwi = make_float2(-wi.x, -wi.y);
          float2 orr[2][2], oii[2][2];  // [xb][n0]
#pragma unroll
          for (int xb = 0; xb < 2; ++xb) {
            const float2 y0r = make_float2(yv[c][0][0][2 * xb], yv[c][0][0][2 * xb + 1]);
            const float2 y0i = make_float2(yv[c][0][1][2 * xb], yv[c][0][1][2 * xb + 1]);
            const float2 y1r = make_float2(yv[c][1][0][2 * xb], yv[c][1][0][2 * xb + 1]);
            const float2 y1i = make_float2(yv[c][1][1][2 * xb], yv[c][1][1][2 * xb + 1]);
            const float2 t1r = fma2(y1r, wr, mul2(y1i, nwi)), t1i = fma2(y1r, wi, mul2(y1i, wr));
            float2 sr[2], si[2];
            sr[0] = add2(y0r, t1r); si[0] = add2(y0i, t1i);
            sr[1] = sub2(y0r, t1r); si[1] = sub2(y0i, t1i);
#pragma unroll
            for (int k0 = 0; k0 < 2; ++k0) {  // * k_f / 2
              const float4 qv = kf[c][k0];
              const float2 kr = make_float2(qv.x, qv.y), ki = make_float2(qv.z, qv.w);  // (1/2 folded into k_f)
              const float2 zr = fma2(sr[k0], kr, mul2(si[k0], make_float2(-ki.x, -ki.y)));
              const float2 zi = fma2(sr[k0], ki, mul2(si[k0], kr));
              sr[k0] = zr; si[k0] = zi;
            }
            orr[xb][0] = add2(sr[0], sr[1]); oii[xb][0] = add2(si[0], si[1]);
            const float2 r1r = sub2(sr[0], sr[1]), r1i = sub2(si[0], si[1]);
            orr[xb][1] = fma2(r1r, wr, mul2(r1i, wi));  // * conj W
            oii[xb][1] = fma2(r1i, wr, mul2(r1r, nwi));
          }
#pragma unroll
          for (int slot = 0; slot < 2; ++slot) {  // rows r (xb 0), r + 8 (xb 1); n0 = slot
            const uint32_t ca = tl + C::CA + slot * L1 + 4 * k1c;
            tmem_st_16x128b(ca, pack_half2(orr[0][slot].x, orr[0][slot].y), pack_half2(orr[1][slot].x, orr[1][slot].y));
            tmem_st_16x128b(ca + L1 / 2, pack_half2(oii[0][slot].x, oii[0][slot].y),
                            pack_half2(oii[1][slot].x, oii[1][slot].y));
          }
          }
        }
      }
      tmem_st_wait();
    } else if constexpr (DIT) {
      // Order 3: for each f' = k2 + 64 k1 the L0I inner rows n0 hold
      // Y_n0[f']; X[f' + 2048 k0] = sum_n0 W_L0I^{n0 k0} W_{32 L0I}^{n0 k1}
      // Y_n0[f'] (the W_LF^{n0 k2} part of the twiddle was applied in
      // epilogue 1), * k_f, the inverse DFT_L0I back to n0, conj twiddle,
      // 1 / L0I.  n0 low bit = group (this thread's two TMEM column blocks),
      // n0 high bit (L0I = 4) = lane bit 3 (shuffles).  k_f blocks are read
      // from global memory (L2-resident, 16 B per load).
      static_assert(TS && !FC_NEG_B, "order-3 epilogue 2");
      const int k2 = rowB_k2(0);
      const int xb = (m >> 3) & 1;
      const uint8_t* kfh = gkf + h * int64_t(L0I) * C::KF_BYTES;
      auto k0_of = [&](int slot) { return L0I == 2 ? slot : xb + 2 * slot; };
      auto n0_of = [&](int slot) { return L0I == 2 ? slot : 2 * xb + slot; };
      auto load_kf = [&](int k1c, float4 (&dst)[2][4]) {
#pragma unroll
        for (int slot = 0; slot < 2; ++slot)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            if constexpr (F::KFS) {  // shared buffer: 8 lanes read 128 contiguous bytes per phase
              const uint4 q = ld_shared_u4(sKFD + k0_of(slot) * F::KFD_BLOCK + dit_kf_off(k2, k1c * 4 + jj));
              dst[slot][jj] = make_float4(__uint_as_float(q.x), __uint_as_float(q.y), __uint_as_float(q.z),
                                          __uint_as_float(q.w));
            } else {
              dst[slot][jj] = __ldg(reinterpret_cast<const float4*>(kfh + k0_of(slot) * C::KF_BYTES +
                                                                    dit_kf_off(k2, k1c * 4 + jj)));
            }
          }
      };
      // all complex math on f32x2 pairs of consecutive k1 (FMUL2/FFMA2/FADD2)
      auto process = [&](int k1c, const float4 (&kf)[2][4]) {
        float re[2][8], im[2][8];
#pragma unroll
        for (int slot = 0; slot < 2; ++slot) {
          tmem_ld8(tq + slot * NBF + k1c * 8, re[slot]);
          tmem_ld8(tq + slot * NBF + k1c * 8 + L1, im[slot]);
        }
        // W_{32 L0I}^{n0 k1}, k1 = 8 k1c + e, per slot (n0), as pairs (e, e+1)
        float2 wr[2][4], wi[2][4];
#pragma unroll
        for (int slot = 0; slot < 2; ++slot) {
          const int n0 = n0_of(slot);
          const float2 b0 = wroot<32 * L0I>(n0 * 8 * k1c), b1 = wroot<32 * L0I>(n0 * (8 * k1c + 1));
          const float2 st2 = wroot<32 * L0I>(2 * n0);
          float2 pr = make_float2(b0.x, b1.x), pi = make_float2(b0.y, b1.y);
#pragma unroll
          for (int ee = 0; ee < 4; ++ee) {
            wr[slot][ee] = pr; wi[slot][ee] = pi;
            const float2 nr = fma2(pr, make_float2(st2.x, st2.x), mul2(pi, make_float2(-st2.y, -st2.y)));
            pi = fma2(pr, make_float2(st2.y, st2.y), mul2(pi, make_float2(st2.x, st2.x)));
            pr = nr;
          }
        }
        tmem_ld_wait();
#pragma unroll
        for (int ee = 0; ee < 4; ++ee) {
          const int e = 2 * ee;
          float2 xr[2], xi[2];
#pragma unroll
          for (int slot = 0; slot < 2; ++slot) {  // T = W^{n0 k1} Y
            const float2 r2 = make_float2(re[slot][e], re[slot][e + 1]), i2 = make_float2(im[slot][e], im[slot][e + 1]);
            xr[slot] = sub2(mul2(r2, wr[slot][ee]), mul2(i2, wi[slot][ee]));
            xi[slot] = fma2(i2, wr[slot][ee], mul2(r2, wi[slot][ee]));
          }
          float2 sr[2], si[2];
          if constexpr (L0I == 2) {
            sr[0] = add2(xr[0], xr[1]); si[0] = add2(xi[0], xi[1]);
            sr[1] = sub2(xr[0], xr[1]); si[1] = sub2(xi[0], xi[1]);
          } else {
            float2 tr[2], ti[2];  // S_b[n0lo] = T[0][n0lo] + (-1)^b T[1][n0lo]
#pragma unroll
            for (int slot = 0; slot < 2; ++slot) {
              const float2 pr = make_float2(__shfl_xor_sync(0xffffffffu, xr[slot].x, 8),
                                            __shfl_xor_sync(0xffffffffu, xr[slot].y, 8));
              const float2 pi = make_float2(__shfl_xor_sync(0xffffffffu, xi[slot].x, 8),
                                            __shfl_xor_sync(0xffffffffu, xi[slot].y, 8));
              tr[slot] = xb ? sub2(pr, xr[slot]) : add2(xr[slot], pr);
              ti[slot] = xb ? sub2(pi, xi[slot]) : add2(xi[slot], pi);
            }
            // X[b + 2 kk] = S0 +- W_4^b S1, W_4^1 = -i
            const float2 ur = xb ? ti[1] : tr[1], ui = xb ? make_float2(-tr[1].x, -tr[1].y) : ti[1];
            sr[0] = add2(tr[0], ur); si[0] = add2(ti[0], ui);
            sr[1] = sub2(tr[0], ur); si[1] = sub2(ti[0], ui);
          }
          // * k_f[f' + 2048 k0] / L0I: kf[slot][ee] = {kr_e, kr_e+1, ki_e, ki_e+1}
#pragma unroll
          for (int slot = 0; slot < 2; ++slot) {
            const float4 q = kf[slot][ee];
            const float2 kr = make_float2(q.x, q.y), ki = make_float2(q.z, q.w);  // (1/L0 folded into k_f)
            const float2 nki = make_float2(-ki.x, -ki.y);
            const float2 zr = fma2(si[slot], nki, mul2(sr[slot], kr));
            const float2 zi = fma2(si[slot], kr, mul2(sr[slot], ki));
            sr[slot] = zr; si[slot] = zi;
          }
          float2 ar[2], ai[2];
          if constexpr (L0I == 2) {
            ar[0] = add2(sr[0], sr[1]); ai[0] = add2(si[0], si[1]);
            ar[1] = sub2(sr[0], sr[1]); ai[1] = sub2(si[0], si[1]);
          } else {
            // R[0] = Z0 + Z1, R[1] = W_4^{-b} (Z0 - Z1), W_4^{-1} = +i
            const float2 dr = sub2(sr[0], sr[1]), di = sub2(si[0], si[1]);
            float2 rr[2], ri[2];
            rr[0] = add2(sr[0], sr[1]); ri[0] = add2(si[0], si[1]);
            rr[1] = xb ? make_float2(-di.x, -di.y) : dr; ri[1] = xb ? dr : di;
#pragma unroll
            for (int slot = 0; slot < 2; ++slot) {
              const float2 qr = make_float2(__shfl_xor_sync(0xffffffffu, rr[slot].x, 8),
                                            __shfl_xor_sync(0xffffffffu, rr[slot].y, 8));
              const float2 qi = make_float2(__shfl_xor_sync(0xffffffffu, ri[slot].x, 8),
                                            __shfl_xor_sync(0xffffffffu, ri[slot].y, 8));
              ar[slot] = xb ? sub2(qr, rr[slot]) : add2(rr[slot], qr);
              ai[slot] = xb ? sub2(qi, ri[slot]) : add2(ri[slot], qi);
            }
          }
#pragma unroll
          for (int slot = 0; slot < 2; ++slot) {  // conj twiddle
            const float2 o_r = fma2(ai[slot], wi[slot][ee], mul2(ar[slot], wr[slot][ee]));
            const float2 o_i = sub2(mul2(ai[slot], wr[slot][ee]), mul2(ar[slot], wi[slot][ee]));
            re[slot][e] = o_r.x; re[slot][e + 1] = o_r.y;
            im[slot][e] = o_i.x; im[slot][e + 1] = o_i.y;
          }
        }
#pragma unroll
        for (int slot = 0; slot < 2; ++slot) {  // K index c*L1 + k1 -> column (c*L1 + k1) / 2
          const uint32_t ca = tq + C::CA + slot * L1 + k1c * 4;
          tmem_st4(ca, pack_half2(re[slot][0], re[slot][1]), pack_half2(re[slot][2], re[slot][3]),
                   pack_half2(re[slot][4], re[slot][5]), pack_half2(re[slot][6], re[slot][7]));
          tmem_st4(ca + L1 / 2, pack_half2(im[slot][0], im[slot][1]), pack_half2(im[slot][2], im[slot][3]),
                   pack_half2(im[slot][4], im[slot][5]), pack_half2(im[slot][6], im[slot][7]));
        }
      };
      float4 kfa[2][4];
      if constexpr (F::KFS) mbar_wait(&bb.kff, uint32_t(hh - t0 / nbt) & 1u);  // this head's refill landed
      load_kf(slice, kfa);
      wait_half(0);
      wait_half(1);
      {
        float4 kfb[2][4];
        load_kf(slice + 2, kfb);
        process(slice, kfa);
        process(slice + 2, kfb);
      }
      tmem_st_wait();
    } else if constexpr (EPI_PIPE) {
      // items it = slice + 2 i < (P/2) kc: group gi = it / kc, kept chunk
      // j = it % kc (half 0: groups < P/4).  The TMEM load of item i + 1 is
      // issued right after item i's wait, so its latency overlaps item i's
      // math (tcgen05.wait::ld waits for every earlier load).
      const int nit = (C::P / 2) * kc, it_h1 = (C::P / 4) * kc;
      auto col_of = [&](int i) { const int it = slice + 2 * i; return uint32_t((it / kc) * NBF + (it % kc) * 8); };
      float buf[2][16];  // re[8] | im[8], double-buffered
      bool h1 = false;
      wait_half(0);
      if (slice >= it_h1) { wait_half(1); h1 = true; }
      tmem_ld8(tq + col_of(0), buf[0]);
      tmem_ld8(tq + col_of(0) + kk, buf[0] + 8);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;
        if (it >= nit) break;
        const int gi = it / kc, j = it % kc, k1c = k1c_of(j);
        const int k2 = rowB_k2(gi);
        float4 kf[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kf[jj] = ld_shared_f4(sKF + tab_off<L1 / 2>(k2, k1c * 4 + jj));
        tmem_ld_wait();
        if (it + 2 < nit) {
          if (TS && !h1 && it + 2 >= it_h1) { wait_half(1); h1 = true; }
          tmem_ld8(tq + col_of(i + 1), buf[(i + 1) & 1]);
          tmem_ld8(tq + col_of(i + 1) + kk, buf[(i + 1) & 1] + 8);
        }
        float* re = buf[i & 1];
        float* im = buf[i & 1] + 8;
        float ni[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) ni[e] = -im[e];
        cmul8(re, im, ni, kf);
        if constexpr (TS) {  // K index c*kk + k1' -> column (c*kk + k1') / 2
          const uint32_t ca = tq + C::CA + gi * L1 + j * 4;
          tmem_st4(ca, pack_half2(re[0], re[1]), pack_half2(re[2], re[3]), pack_half2(re[4], re[5]),
                   pack_half2(re[6], re[7]));
          tmem_st4(ca + kk / 2, pack_half2(im[0], im[1]), pack_half2(im[2], im[3]), pack_half2(im[4], im[5]),
                   pack_half2(im[6], im[7]));
        } else {
          if (!h1) { wait_half(1); h1 = true; }  // stores may overwrite operands of the second half
          const int row = gi * 128 + m;
          st_half8(bufX + (row >> 3) * C::SBO_BP + k1c * 128 + (row & 7) * 16, re);
          st_half8(bufX + (row >> 3) * C::SBO_BP + (L1 / 8 + k1c) * 128 + (row & 7) * 16, im);
        }
      }
      if (!h1) wait_half(1);  // (the stage-B barrier phase is tracked per stage)
    } else {
      // items it = slice + 2 i (dense: 0..3 in half 0, 4..7 in half 1; the
      // slow-digit-skip variant: (P/2) kc items, group it / kc, kept chunk
      // it % kc, half 1 from item (P/4) kc)
      const int nit = (C::P / 2) * kc, it_h1 = (C::P / 4) * kc;
      bool h1 = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;
        if (SKP && it >= nit) break;
        const int gi = it / kc, j = it % kc, k1c = SKP ? k1c_of(j) : j;
        const int k2 = rowB_k2(gi);
        if (i == 0) wait_half(0);
        if (TS && (SKP ? (!h1 && it >= it_h1) : i == 2)) { wait_half(1); h1 = true; }
        const uint32_t col = gi * NBF + j * 8;
        float re[8], im[8], ni[8];
        tmem_ld8(tq + col, re);
        tmem_ld8(tq + col + kk, im);
        if constexpr (FC_NEG_B) tmem_ld8(tq + col + 2 * L1, ni);
        float4 kf[4];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) kf[jj] = ld_shared_f4(sKF + tab_off<L1 / 2>(k2, k1c * 4 + jj));
        tmem_ld_wait();
        if constexpr (!FC_NEG_B) {
#pragma unroll
          for (int e = 0; e < 8; ++e) ni[e] = -im[e];
        }
        cmul8(re, im, ni, kf);
        if constexpr (TS) {  // K index c*kk + k1' -> column (c*kk + k1') / 2
          const uint32_t ca = tq + C::CA + gi * L1 + j * 4;
          tmem_st4(ca, pack_half2(re[0], re[1]), pack_half2(re[2], re[3]), pack_half2(re[4], re[5]),
                   pack_half2(re[6], re[7]));
          tmem_st4(ca + kk / 2, pack_half2(im[0], im[1]), pack_half2(im[2], im[3]), pack_half2(im[4], im[5]),
                   pack_half2(im[6], im[7]));
        } else {
          if (i == 0) wait_half(1);  // stores may overwrite operands of the second half
          const int row = gi * 128 + m;
          st_half8(bufX + (row >> 3) * C::SBO_BP + k1c * 128 + (row & 7) * 16, re);
          st_half8(bufX + (row >> 3) * C::SBO_BP + (L1 / 8 + k1c) * 128 + (row & 7) * 16, im);
        }
      }
      if (SKP && TS && !h1) wait_half(1);  // every thread waits each stage's barriers (phase tracking)
      if constexpr (TS) tmem_st_wait();
    }
    stamp(7);

    // ---------------- stage B^-1: contract k1 -> n1
    sync_and_issue([&](int h2) {
      constexpr uint32_t idesc = idesc_f16(128, NBF, false, false);
#pragma unroll
      for (int gi = h2 * (C::P / 4); gi < (h2 + 1) * (C::P / 4); ++gi) {
#pragma unroll
        for (int s = 0; s < 2 * L1 / 16; ++s) {
          if (TS && s >= kc) break;  // slow-digit skip: K = 2 kk
          if constexpr (TS)
            mma_f16_ts(tmem + gi * NBF, tmem + C::CA + gi * L1 + 8 * s, dadd(dGBI, 256 * s), idesc, s > 0);
          else
            mma_f16_ss(tmem + gi * NBF, dadd(dXBP, gi * 16 * C::SBO_BP + 256 * s), dadd(dGBI, 256 * s), idesc,
                       s > 0);
        }
      }
    }, true, CPL);
    // order 3: the whole warpgroup is past epilogue 2 of tile t (the barrier
    // above): signal it, and when the next tile starts a new head, refill
    // the shared k_f buffer once the other warpgroup's tile t - 1 (the last
    // other reader of the old head) is past its epilogue 2 as well
    if constexpr (F::KFS) {
      if (filler()) {
        mbar_arrive(&bb.e2d[wg]);
        if (t + 1 < t1 && (t + 1) / nbt != hh) {
          if (kWG == 2 && t - 1 >= t0) mbar_wait(&bb.e2d[wg ^ 1], uint32_t((t - 1 - t0) / 2) & 1u);
          kf_fill((t + 1) / nbt);
        }
      }
    }

    // ---------------- epilogue 3: conj twiddle, transpose -> stage A^-1 operand (MN-major B)
    if constexpr (EPI_PIPE) {  // item i + 1's TMEM load overlaps item i's math (as epilogue 2)
      auto col_of = [&](int i) { const int it = slice + 2 * i; return uint32_t((it / JC) * NBF + (it % JC) * 8); };
      float buf[2][16];
      wait_half(0);
      tmem_ld8(tq + col_of(0), buf[0]);
      tmem_ld8(tq + col_of(0) + L1, buf[0] + 8);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;
        const int gi = it / JC, n1c = it % JC;
        const int p = rowB_p(gi), k2 = rowB_k2(gi);
        float4 w[4];
        {
          const float2 a = tw_at(n0_of_p(p) + L0I * 8 * n1c, k2);
          const float br = a.x, bi = a.y;
          const float4 c = tw3_c[gi & 1];  // {Re W^{k2}, Im W^{k2}, Re W^{2k2}, Im W^{2k2}}
          w[0] = make_float4(br, br * c.x - bi * c.y, bi, br * c.y + bi * c.x);
#pragma unroll
          for (int jj = 1; jj < 4; ++jj) w[jj] = cstep(w[jj - 1], make_float2(c.z, c.w));
        }
        tmem_ld_wait();
        if (i + 1 < 4) {
          if (TS && i + 1 == 2) wait_half(1);  // bufX is not an operand of stage B^-1 here
          tmem_ld8(tq + col_of(i + 1), buf[(i + 1) & 1]);
          tmem_ld8(tq + col_of(i + 1) + L1, buf[(i + 1) & 1] + 8);
        }
        float* re = buf[i & 1];
        float* im = buf[i & 1] + 8;
        float nr[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) nr[e] = -re[e];
        cmulc8(re, im, nr, w);
        if (!TS && i == 0) wait_half(1);  // stores may overwrite operands of the second half
        const int ng = DIT ? n1c * C::P + p : (p * L1) / 8 + n1c;
        st_half8(bufX + ng * C::SBO_XA + (k2 >> 3) * 128 + (k2 & 7) * 16, re);
        st_half8(bufX + ng * C::SBO_XA + ((L2 + k2) >> 3) * 128 + (k2 & 7) * 16, im);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int it = slice + 2 * i;
        const int gi = it / JC, n1c = it % JC;
        const int p = rowB_p(gi), k2 = rowB_k2(gi);
        if (i == 0) wait_half(0);
        if (TS && i == 2) wait_half(1);  // bufX is not an operand of stage B^-1 here
        const uint32_t col = gi * NBF + n1c * 8;
        float re[8], im[8], nr[8];
        tmem_ld8(tq + col, re);
        tmem_ld8(tq + col + L1, im);
        if constexpr (FC_NEG_B) tmem_ld8(tq + col + 2 * L1, nr);
        // W^{n1 k2}, n1 = 8 n1c .. 8 n1c + 7 at this k2: the table value at
        // 8 n1c (k2 parity picked from the pair), * W^{k2}, then fp32 steps
        // by W^{2 k2}
        float4 w[4];
        {
          const float2 a = tw_at(n0_of_p(p) + L0I * 8 * n1c, k2);
          const float br = a.x, bi = a.y;
          const float4 c = tw3_c[gi & 1];  // {Re W^{k2}, Im W^{k2}, Re W^{2k2}, Im W^{2k2}}
          w[0] = make_float4(br, br * c.x - bi * c.y, bi, br * c.y + bi * c.x);
#pragma unroll
          for (int jj = 1; jj < 4; ++jj) w[jj] = cstep(w[jj - 1], make_float2(c.z, c.w));
        }
        tmem_ld_wait();
        if constexpr (!FC_NEG_B) {
#pragma unroll
          for (int e = 0; e < 8; ++e) nr[e] = -re[e];
        }
        cmulc8(re, im, nr, w);
        if (!TS && i == 0) wait_half(1);  // stores may overwrite operands of the second half
        // A^-1 output column groups: (p, n1c) in natural order; order 3:
        // (n1c, p) so that epilogue 4 finds every n0 of 8 samples together
        const int ng = DIT ? n1c * C::P + p : (p * L1) / 8 + n1c;
        st_half8(bufX + ng * C::SBO_XA + (k2 >> 3) * 128 + (k2 & 7) * 16, re);
        st_half8(bufX + ng * C::SBO_XA + ((L2 + k2) >> 3) * 128 + (k2 & 7) * 16, im);
      }
    }
    stamp(10);

    // ---------------- stage A^-1: D[(c',n2)][(p,n1)] = G_A^-1 * X[(c,k2)][(p,n1)]
    sync_and_issue([&](int h2) {  // half h2: output columns (p, n1) in [64 h2, 64 h2 + 64)
      if constexpr (AI_TS) {  // half h2 against the G_A^-1 copy in TMEM (causal: copy h2), N = 64
        constexpr uint32_t idesc = idesc_f16(128, 64, false, true);
        const uint32_t ga = tmem - wg * C::TMEM_COLS + (M64 ? h2 * C::TMEM_COLS : 0) + GAI_COL;
#pragma unroll
        for (int s = 0; s < 2 * L2 / 16; ++s)
          mma_f16_ts(tmem + h2 * 64, ga + 8 * s, dadd(dXAI, h2 * 8 * C::SBO_XA + 256 * s), idesc, s > 0);
      } else {
        constexpr uint32_t idesc = idesc_f16(M64 ? 64 : 128, 64, false, true);
        const uint32_t dcol = M64 ? tmem + (uint32_t(16 * h2) << 16) : tmem + h2 * 64;
#pragma unroll
        for (int s = 0; s < 2 * L2 / 16; ++s)
          mma_f16_ss(dcol, dadd(dGAI, 256 * s), dadd(dXAI, h2 * 8 * C::SBO_XA + 256 * s), idesc, s > 0);
      }
    }, true);

    // ---------------- epilogue 4: (gate), convert, store y; load the next tile
    // v (output gate) and the next tile's input are read with coalesced 16 B
    // loads issued before the wait.  y leaves TMEM transposed (lane = n2), so
    // it is staged in natural order through bufX (free once stage A^-1 has
    // completed; 128 B XOR swizzle, conflict-free both ways) and written back
    // coalesced.  Gated tiles stage the conv output in fp16 (the operand
    // precision of every stage; finer than bf16 output) before * v.
    // (Circular gated tiles store directly.)
    {
#ifndef FC_CIRC_DIRECT
#define FC_CIRC_DIRECT 0
#endif
      // circular tiles (the multipass inner pass) may store straight from
      // TMEM registers (16 B per item, 64 B apart within a warp) instead of
      // staging through bufX for fully coalesced rows (FC_CIRC_DIRECT)
      constexpr bool STAGE = CAUSAL || (!GATED && !FC_CIRC_DIRECT);
      using S = typename std::conditional<GATED, __half, T>::type;
      constexpr int OCH = RR * NROW / 8 / kWGThreads;  // coalesced output chunks per thread
      static_assert(!STAGE || RR * NROW * sizeof(S) <= C::BUFX_BYTES, "y staging fits in bufX");
      static_assert(!STG || CPL || (RR * NROW * sizeof(S) <= C::BUFX_BYTES / 2 && RR * F::ROW_BYTES <= C::BUFX_BYTES / 2 &&
                             128 * 2 * C::KA * 2 <= C::BUFX_BYTES / 2),
                    "causal: staged conv output, next stage-A operand and y rows share bufX by halves");
      constexpr int PER = OUT_COLS / 8;  // transposed 8-column items per thread
      constexpr int NV = STAGE ? OCH : PER;
      const bool has_next = t + kWG < t1;
      uint4 nu[PER_ALL], nw[PER_ALL], vv[NV];
      auto och_r = [&](int i) { return (i * kWGThreads + wtid) / (NROW / 8); };
      auto och_n = [&](int i) { return ((i * kWGThreads + wtid) % (NROW / 8)) * 8; };
      auto item_rn = [&](int i, int& r, int& n) {  // transposed item -> (tile row, position)
        const int gc = o_col0 + 8 * i;
        r = 2 * (gc / L1) + o_cp;
        n = ((gc % L1) / 8) * 8 + L1 * o_n2;
      };
      if (GATED && !STG) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          int r, n;
          if (STAGE) { r = och_r(i); n = och_n(i); } else item_rn(i, r, n);
          if (r < rows_left) vv[i] = *reinterpret_cast<const uint4*>(gv + tile_base + int64_t(r) * HN + n);
        }
      }
      if (!STG_IN && has_next && (STAGE || !GATED)) {
        int64_t hh2 = hh, bt2 = bt + kWG;
        while (bt2 >= nbt) { bt2 -= nbt; ++hh2; }
        const int64_t base2 = (bt2 * RR * H + phys_head(hh2)) * N;
        const int left2 = int(B - bt2 * RR < RR ? B - bt2 * RR : RR);
        load_chunks(base2, left2, nu, nw);
      }
      wait_half(M64 ? 0 : slice);
      wait_half(M64 ? 1 : slice ^ 1);  // bufX is rewritten below: both halves done
      stamp(15);
      if constexpr (STAGE) {
        // circular plain tiles (the multipass inner pass): the staged tile
        // leaves by one TMA tensor store from the y staging the warpgroups
        // share in tile order (the store's read of it is awaited only before
        // this warpgroup's next stage A); the staging layout is the 128 B
        // swizzle of the {64, Lp/64, 1, R} box
        const bool tma_out = F::YS_BYTES > 0 && prm.tma_y;
        // causal tiles with TMA I/O: v arrives and y leaves in the 128 B
        // swizzled layout of a {64, N/64, 1, R} box, so each thread gates
        // its own 16-byte units in place (v and y at swz128(offset): no bank
        // conflicts) and writes y straight into the store staging -- no
        // intermediate copy of the conv output, no second pass, one barrier
        // (not for gated order-3 tiles with L0 = 4: the extra registers spill
        // there, 14 % slower; their v / y maps stay natural-order, api.cu)
        constexpr bool Y_DIRECT = STG && !(GATED && L0I == 4 && !FC_O3G4_DIRECT);
        const bool direct = Y_DIRECT && prm.tma_io;
        // (coupled tiles: y is staged -- gated: gated in place -- in the v slot)
        const uint32_t sstg = tma_out ? sYS : CPL ? sV : direct ? sY : bufX;
        if (tma_out && t > t0) mbar_wait(&ys_bar, uint32_t((t - t0 - 1) & 1));
        // all of this thread's TMEM loads in flight before one wait (PER <= 8)
        float ob[PER][8];
#pragma unroll
        for (int i = 0; i < PER; ++i) tmem_ld8(tq + o_tcol + 8 * i, ob[i]);
        if (STG && direct) stg_wait(1);  // v has landed in the output slot
        tmem_ld_wait();
        // one 16-byte unit of y (8 samples at byte offset off of the tile's
        // natural layout, conv output already packed in S): gate, store
        auto put16 = [&](uint32_t off, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
          if (!direct || !GATED) {
            st_shared_v4(sstg + swz128(off), w0, w1, w2, w3);
            return;
          }
          uint4 st = make_uint4(w0, w1, w2, w3);
          const uint4 vq = ld_shared_u4(sV + swz128(off));
          if constexpr (std::is_same<T, __half>::value) {
            __half2* a2 = reinterpret_cast<__half2*>(&st);
            const __half2* v2 = reinterpret_cast<const __half2*>(&vq);
#pragma unroll
            for (int e = 0; e < 4; ++e) a2[e] = __hmul2(a2[e], v2[e]);
          } else {
            float a[8], v8[8];
            IO<__half>::to_f32x8(st, a);
            IO<T>::to_f32x8(vq, v8);
            st = make_uint4(IO<T>::pack2(a[0] * v8[0], a[1] * v8[1]), IO<T>::pack2(a[2] * v8[2], a[3] * v8[3]),
                            IO<T>::pack2(a[4] * v8[4], a[5] * v8[5]), IO<T>::pack2(a[6] * v8[6], a[7] * v8[7]));
          }
          st_shared_v4(sstg + swz128(off), st.x, st.y, st.z, st.w);
        };
        // 8 bytes (4 samples) of y at byte offset off: gate, store (coupled tiles)
        auto put8 = [&](uint32_t off, uint32_t w0, uint32_t w1) {  // (off: final SMEM offset)
          const uint32_t a = sstg + off;
          if constexpr (!GATED) {
            st_shared_v2(a, w0, w1);
          } else {
            uint2 st = make_uint2(w0, w1);
            const uint2 vq = ld_shared_u2(sV + off);
            if constexpr (std::is_same<T, __half>::value) {
              __half2* a2 = reinterpret_cast<__half2*>(&st);
              const __half2* v2 = reinterpret_cast<const __half2*>(&vq);
              a2[0] = __hmul2(a2[0], v2[0]);
              a2[1] = __hmul2(a2[1], v2[1]);
            } else {
              const __half2* a2 = reinterpret_cast<const __half2*>(&st);
              const __nv_bfloat162* v2 = reinterpret_cast<const __nv_bfloat162*>(&vq);
              const float2 a0 = __half22float2(a2[0]), a1 = __half22float2(a2[1]);
              const float2 v0 = __bfloat1622float2(v2[0]), v1 = __bfloat1622float2(v2[1]);
              st = make_uint2(IO<T>::pack2(a0.x * v0.x, a0.y * v0.y), IO<T>::pack2(a1.x * v1.x, a1.y * v1.y));
            }
            st_shared_v2(a, st.x, st.y);
          }
        };
        if constexpr (CPL) {
          // coupled tiles: inner rows n0 = 4 wg + p (items p) at n1 = 8 n1c + e:
          // samples 4 wg + p + 8 (n1 + 32 n2) of real row c' -- 4 consecutive
          // samples per e, the other warpgroup's 4 beside them; the staging
          // box is ordered (n0, n2, n1) (api.cu make_tmap_cpl), so the lanes'
          // consecutive n2 are consecutive 16 B units (the natural order put
          // them 512 B apart: 16-way bank conflicts, 47 M excess wavefronts)
          const int n1c = 2 * o_hh + slice;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t off = uint32_t(o_cp) * F::ROW_BYTES + uint32_t(8 * n1c + e) * (NROW / 16) +
                                 uint32_t(o_n2) * 16 + 8 * wg;
            put8(off, IO<S>::pack2(ob[0][e], ob[1][e]), IO<S>::pack2(ob[2][e], ob[3][e]));
          }
        } else if constexpr (DIT) {
          // items i = inner rows p = q L0I + n0 at 8 n1 of column group n1c:
          // samples n0 + L0I (n1 + 32 n2) of real row 2q + c', interleaved
          const int n1c = 2 * o_hh + slice;
          static_assert(PER == C::P, "order-3 epilogue 4 items");
#pragma unroll
          for (int q = 0; q < C::P / L0I; ++q) {
            const int r = 2 * q + o_cp;
            const int nb = L0I * (8 * n1c + 32 * o_n2);
            uint32_t wd[4 * L0I];
#pragma unroll
            for (int t2 = 0; t2 < 4 * L0I; ++t2) {
              const int a = 2 * t2, b = 2 * t2 + 1;  // samples nb + a, nb + b
              wd[t2] = IO<S>::pack2(ob[q * L0I + a % L0I][a / L0I], ob[q * L0I + b % L0I][b / L0I]);
            }
#pragma unroll
            for (int v4 = 0; v4 < L0I; ++v4)
              put16(uint32_t(r * NROW + nb + 8 * v4) * sizeof(S), wd[4 * v4], wd[4 * v4 + 1], wd[4 * v4 + 2],
                    wd[4 * v4 + 3]);
          }
        } else {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const float* o = ob[i];
          int r, n;
          item_rn(i, r, n);
          put16(uint32_t(r * NROW + n) * sizeof(S), IO<S>::pack2(o[0], o[1]), IO<S>::pack2(o[2], o[3]),
                IO<S>::pack2(o[4], o[5]), IO<S>::pack2(o[6], o[7]));
        }
        }
        stamp(16);
        if (STG && direct) {
          fence_async_smem();  // y -> the tensor store (async proxy)
          if (CPL) named_sync(3, kThreads);  // both warpgroups' samples written
          else wg_sync();      // all of y written, all of v read
          if ((!CPL || wg == 0) && filler()) {
            if (CPL) {  // one (n0, n2, n1)-ordered box per row
              tma_store_4d(&prm.tmap_yo, sV, 0, 0, 0, int(bt * RR * H + h));
              tma_store_4d(&prm.tmap_yo, sV + F::ROW_BYTES, 0, 0, 0, int((bt * RR + 1) * H + h));
            } else {
              tma_store_4d(&prm.tmap_yo, sY, 0, 0, int(h), int(bt * RR));  // rows past B are clipped
            }
            bulk_commit();
            if (CPL) bulk_wait_read0();  // the v slot (y staging) is refilled next
            // v has been read: the output slot goes to tile t + 1 at once
            if (t + 1 < t1) release_out(t + 1, bt + 1 < nbt ? hh : hh + 1, bt + 1 < nbt ? bt + 1 : 0);
          }
        } else if (tma_out) {
          fence_async_smem();
          tc_fence_before();
          wg_sync();
          if (wtid == 0) {
            tma_store_4d(&prm.tmap_y, sYS, 0, 0, int(h), int(bt * RR));
            bulk_commit();
            ys_pending = true;
            if (t + kWG >= t1) {  // no further tile of this warpgroup: hand over now
              bulk_wait_read0();
              mbar_arrive(&ys_bar);
              ys_pending = false;
            }
          }
        } else {
        tc_fence_before();
        if (STG) stg_wait(1);
        stamp(17);
        wg_sync();
        stamp(18);
#pragma unroll
        for (int i = 0; i < OCH; ++i) {
          const int r = och_r(i), n = och_n(i);
          const uint32_t off = uint32_t(r * NROW + n) * sizeof(S);
          uint4 st;
          if constexpr (GATED && std::is_same<T, __half>::value) {
            // fp16 y * fp16 v: HMUL2 rounds the exact product once, the same
            // value as the fp32 product rounded to fp16
            st = ld_shared_u4(bufX + swz128(off));
            if (STG) vv[i] = ld_shared_u4(sV + r * F::ROW_BYTES + n * 2);  // the output slot holds v
            __half2* a2 = reinterpret_cast<__half2*>(&st);
            const __half2* v2 = reinterpret_cast<const __half2*>(&vv[i]);
#pragma unroll
            for (int e = 0; e < 4; ++e) a2[e] = __hmul2(a2[e], v2[e]);
          } else if constexpr (GATED) {
            float a[8], v8[8];
            IO<__half>::to_f32x8(ld_shared_u4(bufX + swz128(off)), a);
            if (STG) vv[i] = ld_shared_u4(sV + r * F::ROW_BYTES + n * 2);  // the output slot holds v
            IO<T>::to_f32x8(vv[i], v8);
            st = make_uint4(IO<T>::pack2(a[0] * v8[0], a[1] * v8[1]), IO<T>::pack2(a[2] * v8[2], a[3] * v8[3]),
                            IO<T>::pack2(a[4] * v8[4], a[5] * v8[5]), IO<T>::pack2(a[6] * v8[6], a[7] * v8[7]));
          } else {
            st = ld_shared_u4(bufX + swz128(off));
          }
          // y in natural order in bufX's second half (the staged conv output
          // and the next tile's stage-A operand use only the first half)
          if (STG) st_shared_v4(sY + r * F::ROW_BYTES + n * 2, st.x, st.y, st.z, st.w);
          else if (r < rows_left) *reinterpret_cast<uint4*>(gy + tile_base + int64_t(r) * HN + n) = st;
        }
        stamp(19);
        if (STG) fence_async_smem();  // y rows -> bulk stores (async proxy)
        wg_sync();  // staging reads done before bufX takes the next tile's operand
        if (STG && filler()) {
          if (prm.tma_io)  // one tensor store (rows past B are clipped)
            tma_store_4d(&prm.tmap_yo, sY, 0, 0, int(h), int(bt * RR));
          else
            for (int r = 0; r < rows_left; ++r) bulk_s2g(gy + tile_base + int64_t(r) * HN, sY + r * F::ROW_BYTES, F::ROW_BYTES);
          bulk_commit();
          // v has been read: the output slot goes to tile t + 1 at once
          if (t + 1 < t1) release_out(t + 1, bt + 1 < nbt ? hh : hh + 1, bt + 1 < nbt ? bt + 1 : 0);
        }
        }  // !tma_out
      } else {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          float o[8];
          tmem_ld8(tq + o_tcol + 8 * i, o);
          tmem_ld_wait();
          int r, n;
          item_rn(i, r, n);
          if constexpr (GATED) {
            float v8[8];
            IO<T>::to_f32x8(vv[i], v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] *= v8[e];
          }
          if (r < rows_left)
            *reinterpret_cast<uint4*>(gy + tile_base + int64_t(r) * HN + n) =
                make_uint4(IO<T>::pack2(o[0], o[1]), IO<T>::pack2(o[2], o[3]), IO<T>::pack2(o[4], o[5]),
                           IO<T>::pack2(o[6], o[7]));
        }
        if (GATED && has_next) {  // (plain tiles prefetched these before the wait)
          int64_t hh2 = hh, bt2 = bt + kWG;
          while (bt2 >= nbt) { bt2 -= nbt; ++hh2; }
          const int64_t base2 = (bt2 * RR * H + phys_head(hh2)) * N;
          const int left2 = int(B - bt2 * RR < RR ? B - bt2 * RR : RR);
          load_chunks(base2, left2, nu, nw);
        }
        tc_fence_before();
        wg_sync();
      }
      if (!STG_IN && has_next) store_chunks(nu, nw);
      loaded = !STG_IN && has_next;
    }
    stamp(13);
    stamp(14);
    ++trace_tile;
  }
  if (STG || prm.tma_y) bulk_wait0();  // this thread's bulk stores complete
  __syncthreads();
  if (warp == 0) tmem_dealloc<(kWG * C::TMEM_COLS > 512 ? 512 : kWG * C::TMEM_COLS)>(tmem_slot);
}

// ------------------------------------------------------------------ launch
template <int L1, bool CAUSAL, bool GATED, typename T, int L0I = 1, bool SKP = false>
static cudaError_t launch_o2(const FwdParams& prm, cudaStream_t stream) {
  using F = FwdCfg<L1, CAUSAL, GATED, L0I>;
  auto kern = fftconv_fwd_o2_kernel<L1, CAUSAL, GATED, T, L0I, SKP>;
  static int attr[64] = {0};
  if (cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(F::SMEM), attr)) return e;
  const int64_t nbt = (prm.B + F::RR - 1) / F::RR;
  const int64_t tiles = (prm.row_map ? (prm.H / prm.row_L0) * prm.nrow : prm.H) * nbt;
  int grid = int(tiles < prm.num_sms ? tiles : prm.num_sms);
  if (grid < 1) return cudaSuccess;
  return launch_pdl(PDL_CONV, kern, dim3(grid), dim3(F::THREADS), F::SMEM, stream, prm);
}

template <bool CAUSAL, bool GATED, typename T>
static cudaError_t dispatch_l1(const FwdParams& prm, cudaStream_t s) {
  if constexpr (CAUSAL) {  // single-pass order 3 (fft_size 4096 / 8192 / 16384)
    if (prm.L0I == 2) return prm.L1 == 32 ? launch_o2<32, true, GATED, T, 2>(prm, s) : cudaErrorInvalidValue;
    if (prm.L0I == 4) return prm.L1 == 32 ? launch_o2<32, true, GATED, T, 4>(prm, s) : cudaErrorInvalidValue;
    if (prm.L0I == 8)  // coupled warpgroups: tensor-map I/O only
      return prm.L1 == 32 && prm.tma_io ? launch_o2<32, true, GATED, T, 8>(prm, s) : cudaErrorInvalidValue;
  }
  if (prm.L0I > 1) return cudaErrorInvalidValue;
  if (prm.kcn > 0)  // frequency-sparse slow-digit skip (kept k1 chunks only)
    return prm.L1 == 32 && prm.kcn < 4 ? launch_o2<32, CAUSAL, GATED, T, 1, true>(prm, s) : cudaErrorInvalidValue;
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
