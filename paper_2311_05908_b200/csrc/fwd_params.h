// fwd_params.h -- launch parameters of the fused forward kernels (internal).
#pragma once
// Gated order-3 L0 = 4 tiles: y gated in place in the swizzled v slot (1)
// or natural-order v / y and a second pass (0).  Kernel and host agree on it.
#ifndef FC_O3G4_DIRECT
#define FC_O3G4_DIRECT 0
#endif
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#if defined(__CUDACC__)
#define FC_HD_PARAMS __host__ __device__ __forceinline__
#else
#define FC_HD_PARAMS inline
#endif

namespace fc {
struct FwdParams {
  const void* u;
  const void* w;   // gated only
  const void* v;   // gated only
  void* y;
  const void* kf;      // H * L complex fp32, [k2][k1], 128B-swizzled per head
  const void* tables;  // plan table image
  int64_t B, H, N;
  int32_t L1;
  int32_t causal;
  int32_t gated;
  int32_t dtype;  // 0 fp16, 1 bf16, 2 fp32 (validation build)
  int32_t num_sms;
  // sparse multipass: iterate over Hi = (H / row_L0) * nrow heads only; head
  // hh maps to tensor head (hh / nrow) * row_L0 + row_map[hh % nrow]
  const int32_t* row_map;
  int32_t nrow, row_L0;
  const void* wl;  // fp32 validation build: W_L^e, e < L (plan table)
  // circular (multipass inner) tiles: y leaves the SMEM staging buffer by one
  // TMA tensor store (4-D box {64, Lp/64, 1 head, R rows}, 128 B swizzle)
  int32_t tma_y;
  CUtensorMap tmap_y;
  // causal fused tiles: u, w, v rows of a tile arrive by one TMA tensor load
  // per tensor and y leaves by one tensor store (4-D box {256, N/256, 1
  // head, R rows}); 0 = per-row bulk copies
  int32_t tma_io;
  CUtensorMap tmap_u, tmap_w, tmap_v, tmap_yo;
  // single-pass order 3 (causal fft_size = L0I * 2048, L0I in {2, 4}): k_f
  // holds L0I blocks per head, block k0 = K_f[f' + 2048 k0]; 1 = order 2
  int32_t L0I;
  // frequency-sparse slow-digit skip: only kcn chunks of 8 k1 columns
  // (original chunk of kept chunk j = (k1map >> 2 j) & 3) run through stage
  // B, the pointwise step and stage B^-1, with the compacted G_B / G_B^-1 at
  // image offsets off_gb / off_gbi; kcn = 0: dense
  int32_t kcn;
  uint32_t k1map;
  uint32_t off_gb, off_gbi;
};
// Encode a map of 16-bit signal rows (B, H, N), box of R rows of one head.
cudaError_t make_tmap_sig(CUtensorMap* map, const void* base, int64_t B, int64_t H, int64_t N, int R);
// Encode tmap_y for fp16 rows (rows, heads, n) of length n = Lp (in elements),
// row stride heads * Lp; box of R rows of one head.
cudaError_t make_tmap_rows(CUtensorMap* map, void* base, int64_t rows, int64_t heads, int64_t Lp, int R);
cudaError_t launch_fwd_fused(const FwdParams& prm, cudaStream_t s);
// fp32 validation build of the same decomposition on CUDA cores (kernels_f32.cu)
cudaError_t launch_fwd_f32(const FwdParams& prm, cudaStream_t s);

struct KfParams {
  const float* k;     // (H, K)
  void* kf;           // H * L complex fp32
  const float* mask;  // length L or nullptr
  const float2* twiddle;  // W_L^e, e < L (plan table)
  int64_t H, K, L;
  int32_t L1, L2;
  // multipass sparse plans: inner rows k0 with row_keep[k0] == 0 are never
  // read by the inner pass, so their k_f blocks are not computed
  const uint8_t* row_keep;
  // recursive plans: outer level sizes (inner row r -> frequency digit k0(r))
  int32_t nlev;
  int32_t lev[4];
  // bidirectional filters (reading B1): k_bwd (H, K) acts at lags -t; the
  // two-sided filter of the length-Lk transform is k[t] + k_bwd[Lk - t]
  // (t > Lk - K) with lag 0 = k[0] + k_bwd[0]; nullptr = causal filter only
  const float* kb;
  int64_t Lk;
};
// tap t (0 <= t < Lk) of head h's (two-sided) filter, zero-padded
FC_HD_PARAMS float filter_tap(const KfParams& p, int64_t h, int64_t t) {
  float v = t < p.K ? p.k[h * p.K + t] : 0.f;
  if (p.kb) {
    if (t == 0) v += p.kb[h * p.K];
    else if (t > p.Lk - p.K) v = p.kb[h * p.K + (p.Lk - t)];
  }
  return v;
}
// frequency digit k0 + L0 f' of inner row r of a recursive plan: rows nest
// level 0 outermost, frequencies have level 0 fastest
FC_HD_PARAMS int32_t row_freq_digit(int32_t r, int32_t nlev, const int32_t* lev) {
  if (nlev <= 1) return r;
  int32_t d[4] = {0, 0, 0, 0};
  for (int l = nlev - 1; l >= 0; --l) { d[l] = r % lev[l]; r /= lev[l]; }
  int32_t k = 0, m = 1;
  for (int l = 0; l < nlev; ++l) { k += d[l] * m; m *= lev[l]; }
  return k;
}
cudaError_t launch_precompute_kf(const KfParams& prm, cudaStream_t s);
// single-pass order-3 plans: k_f in L0 blocks per head, block k0 = K_f[f' + 2048 k0]
cudaError_t launch_precompute_kf_dit(const KfParams& prm, int L0, cudaStream_t s);
// ... and its multipass (DIF) layout for the backward
cudaError_t launch_kf_dit_to_dif(const void* src, void* dst, int64_t H, int L0, cudaStream_t s);

// multipass regime (kernels_mp.cu)
struct MpParams {
  const void* u;
  const void* w;
  const void* v;
  void* y;
  void* ws;             // T: fp16 rows (2 * pairs, H * L0, Lp)
  const float2* wbase;  // W_L^{n'}, n' < Lp
  const float2* wtab;   // W_L^{n' k0}, [k0][n'] (L0 * Lp entries)
  const void* v2;       // pass 3 only: optional second gate (y2 = x * v2)
  void* y2;
  int64_t B, H, N;
  int32_t L0, Lp;
  int32_t gated;
  int32_t dtype;
  // partial (overlap-save) mode: virtual row b_v = b * NC + j is the window
  // u[b, h, (j-1) C : (j+1) C] (zero before 0); its output is the second half
  // of the circular result, y[b, h, j C : (j+1) C].  B above is then B * NC.
  int32_t partial;
  int64_t NC, C;
  const uint8_t* row_keep;  // sparse: L0 flags, rows with 0 are never written/read
  const int32_t* row_map;   // sparse one-level plans: the kept rows k0 (nrow of them)
  int32_t nrow;
  // recursive levels (N > 16384): complex circular rows of an intermediate in
  // and out (all n0, no gating, fp16); twiddles W_Llev^{n' k0} computed on
  // the fly when wtab == nullptr
  int32_t circ;
  int64_t Llev;
  // chunked execution (L2-resident T): this launch covers pairs
  // [pair0, pair0 + (B+1)/2) and heads [h0, h0 + H) of a signal with Hg
  // heads; T is indexed by the chunk-local (pair, head), u/w/v/y by the
  // global ones.  Hg = 0 means Hg = H (unchunked).
  int64_t pair0, h0, Hg;
  // backward of the partial conv: pass 1 loads only the second half of each
  // window (dc blocks); pass 3 overlap-adds neighbouring windows (dg)
  int32_t win_hi_only, ola;
  // fp16 headroom of the intermediates (top level only): pass 1 scales its
  // output by 2^-shift, pass 3 its result by 2^+shift (exact; 0 = none)
  int32_t shift;
};
cudaError_t launch_mp_pass(const MpParams& prm, int pass, cudaStream_t s);

// backward (kernels_bwd.cu)
struct BwdParams {
  const void* u;   // g source (or T_g rows)
  const void* w;   // gate of u (gated)
  const void* v;   // gate of dy (gated)
  const void* dy;  // dc source (or T_dc rows)
  void* du;        // dg * w (gated), dg (plain / inner)
  void* dw;        // dg * u (gated)
  void* dv;        // dy * c (gated), c (inner)
  const void* kf;
  const void* tables;
  void* acc;       // per-tile partial spectra [tile][L] complex fp32
  int64_t B, H, N;
  int32_t L1;
  int32_t causal;
  int32_t gate_io;
  int32_t need_c;
  int32_t dtype;
  int32_t num_sms;
};
cudaError_t launch_bwd_fused(const BwdParams& prm, cudaStream_t s);
// fp32 validation build of the backward (kernels_f32.cu): per (pair, head)
// partial spectra [h][pair][L]; wl = W_L^e (plan table)
cudaError_t launch_bwd_f32(const BwdParams& prm, const void* wl, cudaStream_t s);
int64_t bwd_f32_units_per_head(int64_t B);
int64_t bwd_tiles_per_head(int64_t B, int L1);

// dk = Re IFFT(mask * sum of partial spectra)[:K] (kernels_kf.cu)
struct DkParams {
  const float2* part;   // [H * L0][nbt][Lp] partial spectra
  float2* scratch;      // multipass: H * L0 * Lp complex fp32 (may alias part)
  float* dk;            // (H, K)
  const float* mask;    // length L or nullptr
  const float2* twiddle;  // W_Lp^e, e < Lp
  const float2* wbase;    // multipass: W_L^{n'}, n' < Lp
  int64_t H, K, nbt;
  int32_t L0, Lp;
  // recursive plans (nlev > 1): L0 above is the product of the levels; the
  // deeper levels are inverted in place on scratch, then level 0 (twiddles
  // W_Lfull^{n'} on the fly when wbase is null)
  const int32_t* lev_L0;
  int32_t nlev;
  int64_t Lfull;
  int32_t lev[4];  // device copy of lev_L0 (mask digit mapping)
  int32_t shift2;  // dk *= 2^shift2 (undoes the headroom pre-scale of G and DC)
  // bidirectional backward (reading B1): dk_bwd[t] = lag -t of the inverse
  // transform, i.e. index (Lfull - t) mod Lfull; nullptr = not written
  float* dkb;
};
// lag index t (0 <= t < Lfull) of the inverse transform of head h -> dk / dkb
FC_HD_PARAMS void dk_emit(const DkParams& p, int64_t h, int64_t t, int64_t Lfull, float x) {
  if (t < p.K) p.dk[h * p.K + t] = x;
  if (p.dkb) {
    if (t == 0) p.dkb[h * p.K] = x;
    else if (t > Lfull - p.K) p.dkb[h * p.K + (Lfull - t)] = x;
  }
}
cudaError_t launch_dk_finalize(const DkParams& prm, cudaStream_t s);
cudaError_t launch_mp_precompute_kf(const KfParams& prm, const int32_t* lev_L0, int nlev, int64_t Lfull,
                                    size_t block_bytes, cudaStream_t s);
cudaError_t launch_mp_cols_inverse(float2* data, int L0, int64_t rows, int64_t Lrow, cudaStream_t s);
}  // namespace fc
