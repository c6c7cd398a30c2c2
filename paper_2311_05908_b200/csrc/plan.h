// plan.h -- internal plan structure shared by the host planner (plan.cpp)
// and the launch code (api.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "fftconv.h"

namespace fc {

enum Regime : int32_t { REGIME_FUSED = 1, REGIME_PARTIAL = 2, REGIME_MULTIPASS = 3 };

// Byte offsets of the constant tables inside the uploaded device image.
// Each table is stored exactly as the fused kernel wants it in shared memory
// (SWIZZLE_NONE canonical UMMA layouts for the DFT matrices, 128-byte XOR
// swizzle for the fp32 twiddle table), so the kernel copies it linearly.
struct TableLayout {
  size_t ga = 0, ga_bytes = 0;    // stage A  : B operand, K-major, rows (c',k2) 2*L2, K (c,n2) 2*KA
  size_t gb = 0, gb_bytes = 0;    // stage B  : B operand, K-major, rows (c',k1) 2*L1, K (c,n1) 2*L1
  size_t gbi = 0, gbi_bytes = 0;  // stage B^-1
  size_t gai = 0, gai_bytes = 0;  // stage A^-1: A operand, K-major, rows (c',n2) 2*L2, K (c,k2) 2*L2
  size_t tw = 0, tw_bytes = 0;    // W_L^{n1 k2}, [n1][k2/2] float4 pairs, swizzled
  size_t twt = 0, twt_bytes = 0;  // same values, [k2][n1/2]
  size_t wl = 0, wl_bytes = 0;    // W_L^e, e < L, float2 (k_f precompute)
  size_t wbase = 0, wbase_bytes = 0;  // multipass: W_L^{n'}, n' < L', float2
  size_t wtab = 0, wtab_bytes = 0;    // multipass: W_L^{n' k0}, [k0][n'], float2
  size_t total = 0;
};

}  // namespace fc

struct fftconv_plan_s {
  int64_t N = 0;         // input length per row
  int64_t L = 0;         // fft_size
  int32_t causal = 1;
  fftconv_dtype_t dtype = FFTCONV_F16;
  int32_t regime = fc::REGIME_FUSED;
  int32_t order = 2;
  int32_t L1 = 0, L2 = 0;  // L = L1 * L2 ; n = n1 + L1*n2 ; f = k2 + L2*k1
  int32_t KA = 0;          // contracted length of stage A (L2/2 causal, L2 circular)
  int32_t P = 0;           // row pairs per tile (two-row real packing)
  int64_t chunk = 0;       // partial regime: chunk length (= L/2)
  int32_t L0 = 1;          // multipass: total outer factor, L = L0 * Lp
  int32_t nlev = 0;        // multipass: outer levels (L0 = prod lev_L0)
  int32_t lev_L0[4] = {1, 1, 1, 1};
  int32_t Lp = 0;          // multipass: inner (fused) transform length
  // single-pass order 3 (causal fft_size = dit * 2048, dit in {2, 4, 8}): the
  // forward runs one fused kernel (DIT outer DFT in its pointwise step) with
  // the causal 2048-point tables at image offset dit_tab_off, and k_f holds
  // dit blocks per head, block k0 = K_f[f' + 2048 k0]; the backward runs the
  // multipass path on k_f re-laid out in its workspace.  1 = not used.
  int32_t dit = 1;
  // fp16 headroom: multipass / partial plans pre-scale the first
  // outer pass's output by 2^-headroom_shift (undone exactly by the last), so
  // every fp16 intermediate stays finite for rows with max|g| <= 256
  int32_t headroom_shift = 0;
  size_t dit_tab_off = 0;
  fc::TableLayout tl;
  std::vector<uint8_t> image;  // host copy of the table image
  void* d_tables = nullptr;    // bound by fftconv_plan_upload
  // frequency sparsity (A13)
  bool sparse = false;
  std::vector<float> mask;     // length L, 0/1, Hermitian-symmetric
  std::vector<int32_t> row_map;  // multipass: kept outer rows k0 (empty = all)
  size_t row_keep_off = 0, row_map_off = 0;  // image offsets (sparse multipass)
  double mask_fraction = 0.0;
  double skip_fraction = 0.0;
  // slow-digit skip: chunks of 8 stage-B output columns k1
  // whose frequencies are masked for every k2 and every inner row are left
  // out of stage B, the pointwise step and stage B^-1 (0 = dense); the
  // forward reads compacted G_B / G_B^-1 copies at gb_sp / gbi_sp
  int32_t k1_chunks = 0;
  uint32_t k1_map = 0;   // 2 bits per kept chunk: its original chunk index
  size_t gb_sp = 0, gbi_sp = 0;
  size_t kf_bytes_per_head = 0;
  size_t ws_bytes_per_head = 0;
  int32_t sram_smem_bytes = 0;  // dynamic shared memory of the fused kernel
};

namespace fc {
// Eq. 2 cost model -- host planner utilities, exported for tests.
struct CostConstants {
  double mu, sigma_h, sigma_s, tau_m, tau_g, sram_bytes;
};
double cost_eq2(int64_t N, const std::vector<int64_t>& factors, const CostConstants& c, double BH);
int select_order(int64_t N, const CostConstants& c, std::vector<int64_t>* factors_out);
std::vector<int64_t> factorize(int64_t n, int p);
void set_last_error(const std::string& msg);
}  // namespace fc
