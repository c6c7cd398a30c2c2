// plan.cpp -- host planner of the B200 FlashFFTConv library.
//
//  * validates (N, fft_size, dtype, causal, sparsity) and picks the regime;
//  * factorises the complex transform length (Monarch order-2, P:124-126,
//    Alg. 1) and builds every constant table in fp64, rounded once
//    to the storage precision (real-pair fp16 DFT matrices with unitary
//    1/sqrt(L_i) scaling, fp32 twiddles with the exponent reduced mod L in
//    integers);
//  * builds the Hermitian-symmetric frequency mask of A13;
//  * implements the Eq. 2 cost model and order selection.
//
// No CUDA calls happen here except in fftconv_plan_upload (api.cu).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "plan.h"
#include "layout.h"

// B200 tier cost model coefficients (seconds per feature unit), fitted by
// tools/cost_model.py on the bench sweep (profiles/r02c/cost_model.md).
#define COST_B200_0 1.005051e-08
#define COST_B200_1 7.413649e-09
#define COST_B200_2 1.279446e-08
#define COST_B200_3 1.558044e-08
#define COST_B200_4 3.572859e-12
#define COST_B200_5 9.231505e-12
#define COST_B200_6 1.237435e-05
#define COST_B200_7 0.000000e+00
#define COST_B200_8 4.945092e-12
#define COST_B200_9 3.467309e-11
#define COST_B200_10 0.000000e+00
#define COST_B200_11 1.197651e-13

namespace fc {

static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }

static bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
static int ilog2(int64_t x) {
  int r = 0;
  while ((int64_t(1) << r) < x) ++r;
  return r;
}

// Balanced power-of-two split, larger factors first.
std::vector<int64_t> factorize(int64_t n, int p) {
  std::vector<int64_t> f;
  if (!is_pow2(n) || p < 1) return f;
  int e = ilog2(n);
  if (e < p) return f;
  for (int i = 0; i < p; ++i) {
    int ei = e / p + (i < e % p ? 1 : 0);
    f.push_back(int64_t(1) << ei);
  }
  return f;
}

// Eq. 2: C = BH * sum_i [ 16 N N_i / gamma(N_i) + 4 N / omega(i) ]  (A10)
// gamma(N_i) = tau_G if N_i < mu else tau_M; omega(i) = sigma_S if
// the stage-i working set 4N / prod_{j<i} N_j fits the SRAM budget, else
// sigma_H (A11).
double cost_eq2(int64_t N, const std::vector<int64_t>& factors, const CostConstants& c, double BH) {
  double total = 0.0, prefix = 1.0;
  for (size_t i = 0; i < factors.size(); ++i) {
    const double Ni = double(factors[i]);
    const double gamma = Ni < c.mu ? c.tau_g : c.tau_m;
    const double ws = 4.0 * double(N) / prefix;
    const double omega = ws <= c.sram_bytes ? c.sigma_s : c.sigma_h;
    total += 16.0 * double(N) * Ni / gamma + 4.0 * double(N) / omega;
    prefix *= Ni;
  }
  return BH * total;
}

int select_order(int64_t N, const CostConstants& c, std::vector<int64_t>* factors_out) {
  int best_p = 0;
  double best = 0.0;
  for (int p = 2; p <= 4; ++p) {
    auto f = factorize(N, p);
    if (f.empty()) continue;
    double cst = cost_eq2(N, f, c, 1.0);
    if (best_p == 0 || cst < best) {  // ties -> smaller p
      best = cst;
      best_p = p;
      if (factors_out) *factors_out = f;
    }
  }
  return best_p;
}

// ---------------------------------------------------------------- tables
static inline uint16_t to_half_bits(double x) {
  // round-to-nearest-even fp64 -> fp16 (values here are |x| <= 1, normal or 0)
  float f = float(x);  // fp64->fp32 rounding is far below fp16 resolution
  uint32_t u;
  std::memcpy(&u, &f, 4);
  uint32_t sign = (u >> 16) & 0x8000u;
  int32_t exp = int32_t((u >> 23) & 0xFF) - 127 + 15;
  uint32_t mant = u & 0x7FFFFFu;
  if ((u & 0x7FFFFFFFu) == 0) return uint16_t(sign);
  if (exp <= 0) {  // subnormal half
    if (exp < -10) return uint16_t(sign);
    mant |= 0x800000u;
    uint32_t shift = uint32_t(14 - exp);
    uint32_t half_m = mant >> shift;
    uint32_t rem = mant & ((1u << shift) - 1), halfway = 1u << (shift - 1);
    if (rem > halfway || (rem == halfway && (half_m & 1))) half_m++;
    return uint16_t(sign | half_m);
  }
  uint32_t half_m = mant >> 13, rem = mant & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (half_m & 1))) {
    half_m++;
    if (half_m == 0x400u) { half_m = 0; exp++; }
  }
  if (exp >= 31) return uint16_t(sign | 0x7C00u);
  return uint16_t(sign | (uint32_t(exp) << 10) | half_m);
}

static void put_half(std::vector<uint8_t>& img, size_t off, double x) {
  uint16_t h = to_half_bits(x);
  std::memcpy(img.data() + off, &h, 2);
}

// W_n^{e} = exp(-2 pi i e / n) with e reduced mod n in integers (H3).
static void root(int64_t e, int64_t n, double* re, double* im) {
  e %= n;
  if (e < 0) e += n;
  const double ang = -2.0 * M_PI * double(e) / double(n);
  *re = std::cos(ang);
  *im = std::sin(ang);
}

// Real-pair matrix entry for input (c, a) -> output (c', b) of the complex
// map out_b = sum_a F[a][b] in_a:  [[Fr, Fi], [-Fi, Fr]] arrangement.
static double realpair(double fr, double fi, int c_in, int c_out) {
  if (c_in == 0 && c_out == 0) return fr;
  if (c_in == 1 && c_out == 0) return -fi;
  if (c_in == 0 && c_out == 1) return fi;
  return fr;
}

// K-major canonical (SWIZZLE_NONE) byte offset of element (row r, k).
static size_t kmajor_off(int r, int k, int Ktot) {
  const size_t sbo = size_t(Ktot / 8) * 128;
  return size_t(r / 8) * sbo + size_t(k / 8) * 128 + size_t(r % 8) * 16 + size_t(k % 8) * 2;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static void put_float(std::vector<uint8_t>& img, size_t off, double x) {
  float f = float(x);
  std::memcpy(img.data() + off, &f, 4);
}

// Table image of the fused order-2 kernel (kernels_fwd.cu, O2Cfg):
//  GA  : stage A B-operand, K-major rows (k2 half, re|im, k2 mod 32) = 2*L2, K (c,n2) = 2*KA
//  GB  : stage B B-operand, rows (re|im|-im|pad, k1) = NB, K (c,n1) = 2*L1
//  GBI : stage B^-1, rows (re|im|-re|pad, n1) = NB, K (c,k1) = 2*L1
//  GAI : stage A^-1 A-operand, rows (n2 half, c', n2 mod 32) = 2*L2, K (c,k2) = 2*L2
//  TW  : [n1][k2/2] {wr(k2), wr(k2+1), wi(k2), wi(k2+1)} fp32, W = W_L^{n1 k2}
//  TWT : [k2][n1/2] {wr(n1), wr(n1+1), wi(n1), wi(n1+1)} fp32
// DFT matrices carry the unitary 1/sqrt(L_i) scale, so the whole forward +
// inverse pair scales by 1/L and k_f is used unscaled.
static void build_fused_tables(fftconv_plan_s* p, int64_t L) {
  const int L1 = p->L1, L2 = p->L2, KA = p->KA;
  const int NA = 2 * L2, NB = (3 * L1 + 15) / 16 * 16;  // O2Cfg::NA, NB
  TableLayout& t = p->tl;
  size_t off = 0;  // order GA | GB | GBI | TW | GAI | TWT (O2Cfg)
  t.ga = off;  t.ga_bytes = size_t(NA) * (2 * KA) * 2;      off = align_up(off + t.ga_bytes, 1024);
  t.gb = off;  t.gb_bytes = size_t(NB) * (2 * L1) * 2;      off = align_up(off + t.gb_bytes, 1024);
  t.gbi = off; t.gbi_bytes = t.gb_bytes;                    off = align_up(off + t.gbi_bytes, 1024);
  t.tw = off;  t.tw_bytes = size_t(L1) * tab_stride(L2 / 2); off = align_up(off + t.tw_bytes, 1024);
  t.gai = off; t.gai_bytes = size_t(2 * L2) * (2 * L2) * 2; off = align_up(off + t.gai_bytes, 1024);
  t.twt = off; t.twt_bytes = size_t(L2) * tab_stride(L1 / 2); off = align_up(off + t.twt_bytes, 1024);
  t.wl = off;  t.wl_bytes = size_t(L) * 8;                  off = align_up(off + t.wl_bytes, 1024);
  const int64_t Lfull = p->L;  // the whole transform (== L unless multipass)
  t.wbase = off; t.wbase_bytes = Lfull != L ? size_t(L) * 8 : 0; off = align_up(off + t.wbase_bytes, 1024);
  t.wtab = off;  t.wtab_bytes = (Lfull != L && Lfull <= 32768) ? size_t(Lfull) * 8 : 0;
  off = align_up(off + t.wtab_bytes, 1024);
  t.total = off;
  p->image.assign(t.total, 0);
  std::vector<uint8_t>& img = p->image;
  const double sA = 1.0 / std::sqrt(double(L2)), sB = 1.0 / std::sqrt(double(L1));
  // stage A (forward, contracts n2 -> k2): B^T[(blk,k2)][(c,n2)], n2 < KA
  for (int blk = 0; blk < NA / L2; ++blk)
    for (int k2 = 0; k2 < L2; ++k2)
      for (int ci = 0; ci < 2; ++ci)
        for (int n2 = 0; n2 < KA; ++n2) {
          double fr, fi;
          root(int64_t(n2) * k2, L2, &fr, &fi);
          const int co = blk == 0 ? 0 : 1;
          const double sgn = blk == 2 ? -1.0 : 1.0;
          // rows ordered (k2 half, blk, k2 mod 32): each stage-A half is one MMA
          const int row = (k2 / 32) * (NA / 2) + blk * 32 + k2 % 32;
          put_half(img, t.ga + kmajor_off(row, ci * KA + n2, 2 * KA),
                   sgn * realpair(fr * sA, fi * sA, ci, co));
        }
  // stage B (forward, contracts n1 -> k1; blocks re | im | -im) and
  // B^-1 (contracts k1 -> n1; blocks re | im | -re)
  for (int blk = 0; blk < 3; ++blk)
    for (int b = 0; b < L1; ++b)
      for (int ci = 0; ci < 2; ++ci)
        for (int a = 0; a < L1; ++a) {
          double fr, fi;
          root(int64_t(a) * b, L1, &fr, &fi);
          const int co_f = blk == 0 ? 0 : 1;
          const double sg_f = blk == 2 ? -1.0 : 1.0;
          put_half(img, t.gb + kmajor_off(blk * L1 + b, ci * L1 + a, 2 * L1),
                   sg_f * realpair(fr * sB, fi * sB, ci, co_f));
          root(-int64_t(a) * b, L1, &fr, &fi);
          const int co_i = blk == 1 ? 1 : 0;
          const double sg_i = blk == 2 ? -1.0 : 1.0;
          put_half(img, t.gbi + kmajor_off(blk * L1 + b, ci * L1 + a, 2 * L1),
                   sg_i * realpair(fr * sB, fi * sB, ci, co_i));
        }
  // stage A^-1 (contracts k2 -> n2), as the A operand: rows (c',n2), K (c,k2)
  for (int co = 0; co < 2; ++co)
    for (int n2 = 0; n2 < L2; ++n2)
      for (int ci = 0; ci < 2; ++ci)
        for (int k2 = 0; k2 < L2; ++k2) {
          double fr, fi;
          root(-int64_t(k2) * n2, L2, &fr, &fi);
          // rows ordered (n2 half, c', n2 mod 32): the causal forward keeps
          // only n2 < L2/2, i.e. the first 64 rows (one M = 64 MMA)
          const int row = (n2 / 32) * 64 + co * 32 + n2 % 32;
          put_half(img, t.gai + kmajor_off(row, ci * L2 + k2, 2 * L2), realpair(fr * sA, fi * sA, ci, co));
        }
  // twiddles W_L^{n1 k2} as element pairs, padded rows (tab_off_rt)
  for (int n1 = 0; n1 < L1; ++n1)
    for (int k2 = 0; k2 < L2; ++k2) {
      double wr, wi;
      root(int64_t(n1) * k2, L, &wr, &wi);
      const uint32_t q = tab_off_rt(uint32_t(L2 / 2), uint32_t(n1), uint32_t(k2 / 2));
      put_float(img, t.tw + q + (k2 & 1) * 4, wr);
      put_float(img, t.tw + q + 8 + (k2 & 1) * 4, wi);
      const uint32_t r = tab_off_rt(uint32_t(L1 / 2), uint32_t(k2), uint32_t(n1 / 2));
      put_float(img, t.twt + r + (n1 & 1) * 4, wr);
      put_float(img, t.twt + r + 8 + (n1 & 1) * 4, wi);
    }
  // full-length twiddles of the (inner) transform for the k_f precompute;
  // multipass outer twiddles only for a single outer level (deeper levels
  // compute them on the fly)
  for (int64_t e = 0; e < L; ++e) {
    double wr, wi;
    root(e, L, &wr, &wi);
    put_float(img, t.wl + size_t(e) * 8, wr);
    put_float(img, t.wl + size_t(e) * 8 + 4, wi);
  }
  // multipass outer twiddle bases W_Lfull^{n'} ("Twiddle factors")
  if (t.wbase_bytes)
    for (int64_t e = 0; e < L; ++e) {
      double wr, wi;
      root(e, Lfull, &wr, &wi);
      put_float(img, t.wbase + size_t(e) * 8, wr);
      put_float(img, t.wbase + size_t(e) * 8 + 4, wi);
    }
  if (t.wtab_bytes)
    for (int64_t k0 = 0; k0 < Lfull / L; ++k0)
      for (int64_t n = 0; n < L; ++n) {
        double wr, wi;
        root(n * k0, Lfull, &wr, &wi);
        put_float(img, t.wtab + size_t(k0 * L + n) * 8, wr);
        put_float(img, t.wtab + size_t(k0 * L + n) * 8 + 4, wi);
      }
}

// A13: keep(f) = prod_j keep_j[digit_j(f)], digits of f on the row-major
// grid dims (slowest first); m[f] = keep(f) | keep((L - f) mod L).
static fftconv_status_t build_mask(fftconv_plan_s* p, const fftconv_sparsity_t* s) {
  if (s->ndims < 1 || s->ndims > 4) return FFTCONV_ERR_BAD_SPARSITY;
  int64_t prod = 1;
  for (int j = 0; j < s->ndims; ++j) {
    if (s->dims[j] < 1 || !s->keep[j]) return FFTCONV_ERR_BAD_SPARSITY;
    prod *= s->dims[j];
  }
  if (prod != p->L) return FFTCONV_ERR_BAD_SPARSITY;
  const int64_t L = p->L;
  auto keep = [&](int64_t f) {
    int64_t rem = f;
    for (int j = s->ndims - 1; j >= 0; --j) {
      int64_t d = rem % s->dims[j];
      rem /= s->dims[j];
      if (!s->keep[j][d]) return false;
    }
    return true;
  };
  p->mask.assign(size_t(L), 0.0f);
  int64_t zeros = 0;
  for (int64_t f = 0; f < L; ++f) {
    bool k = keep(f) || keep((L - f) % L);
    p->mask[size_t(f)] = k ? 1.0f : 0.0f;
    zeros += k ? 0 : 1;
  }
  p->sparse = true;
  p->mask_fraction = double(zeros) / double(L);
  // Skippable work: in the multipass / partial regimes the inner pass runs
  // one row per outer frequency k0 (f = k0 + L0 f'); a row whose whole
  // spectrum is masked contributes nothing and is skipped ("skip one
  // iteration of the outer loop").  The fused regime skips nothing yet.
  p->row_map.clear();
  if (p->L0 > 1 && p->nlev > 1) {
    // recursive plans: the mask acts through k_f only (inner row r holds the
    // frequencies k0(r) + L0 f', k0(r) the level-digit reversal of r); no row
    // is skipped
    for (int k0 = 0; k0 < p->L0; ++k0) p->row_map.push_back(k0);
    p->skip_fraction = 0.0;
  } else if (p->L0 > 1) {
    for (int k0 = 0; k0 < p->L0; ++k0) {
      bool any = false;
      for (int64_t fp = 0; fp < p->Lp && !any; ++fp) any = p->mask[size_t(k0 + int64_t(p->L0) * fp)] != 0.0f;
      if (any) p->row_map.push_back(k0);
    }
    p->skip_fraction = 1.0 - double(p->row_map.size()) / double(p->L0);
  } else {
    p->skip_fraction = 0.0;
  }
  // Slow-digit skip ("sparsity in the first dimension allows us
  // to skip computation in B"): the inner transform's frequency is
  // f = k0 + L0 (k2 + L2 k1) (L0 = 1 fused), so stage-B output column chunk
  // c (k1 in [8c, 8c + 8)) holds exactly the frequencies f in
  // [c L / (L1/8), (c + 1) L / (L1/8)); a chunk masked there for every f is
  // never computed.  Inner transforms with L1 = 32 (fused fft_size 2048 and
  // every multipass inner pass; chunks of 8 = one K = 16 step of re | im).
  p->k1_chunks = 0;
  p->k1_map = 0;
  const int nch = p->L1 / 8;
  if (p->L1 == 32 && p->dit == 1) {
    int kept = 0;
    uint32_t map = 0;
    const int64_t span = L / nch;
    for (int c = 0; c < nch; ++c) {
      bool any = false;
      for (int64_t f = c * span; f < (c + 1) * span && !any; ++f) any = p->mask[size_t(f)] != 0.0f;
      if (any) map |= uint32_t(c) << (2 * kept++);
    }
    if (kept > 0 && kept < nch) {
      p->k1_chunks = kept;
      p->k1_map = map;
      const double rows_kept = p->L0 > 1 ? double(p->row_map.size()) / double(p->L0) : 1.0;
      p->skip_fraction = 1.0 - rows_kept * double(kept) / double(nch);
    }
  }
  return FFTCONV_OK;
}

// Compacted copies of the forward's G_B (output rows re | im, only the kept
// k1 chunks) and G_B^-1 (contraction index (c, k1) -> (c, kept k1)) for the
// slow-digit skip; same K-major canonical layout and strides as the dense
// tables, unused rows / K columns zero.
static void build_k1_compact(fftconv_plan_s* p) {
  if (p->k1_chunks == 0) return;
  const int L1 = p->L1, kk = 8 * p->k1_chunks, Kt = 2 * L1;
  auto k1_of = [&](int k1c) {  // compacted k1 -> original
    return int((p->k1_map >> (2 * (k1c / 8))) & 3u) * 8 + k1c % 8;
  };
  std::vector<uint8_t>& img = p->image;
  p->gb_sp = align_up(img.size(), 1024);
  p->gbi_sp = align_up(p->gb_sp + p->tl.gb_bytes, 1024);
  img.resize(align_up(p->gbi_sp + p->tl.gbi_bytes, 1024), 0);
  for (int blk = 0; blk < 2; ++blk)
    for (int j = 0; j < kk; ++j)
      for (int k = 0; k < Kt; ++k)
        std::memcpy(img.data() + p->gb_sp + kmajor_off(blk * kk + j, k, Kt),
                    img.data() + p->tl.gb + kmajor_off(blk * L1 + k1_of(j), k, Kt), 2);
  for (int row = 0; row < 2 * L1; ++row)  // forward rows re | im (n1)
    for (int c = 0; c < 2; ++c)
      for (int j = 0; j < kk; ++j)
        std::memcpy(img.data() + p->gbi_sp + kmajor_off(row, c * kk + j, Kt),
                    img.data() + p->tl.gbi + kmajor_off(row, c * L1 + k1_of(j), Kt), 2);
}

}  // namespace fc

using namespace fc;

double predict_seconds(const fftconv_plan_s* p, int64_t B, int64_t H, bool bwd, bool gated, const double* coef);

extern "C" fftconv_status_t fftconv_plan(fftconv_plan_t* out, int64_t N, int64_t fft_size, fftconv_dtype_t dtype,
                                         int causal, const fftconv_sparsity_t* sparsity) {
  if (!out) { set_last_error("fftconv_plan: out is NULL"); return FFTCONV_ERR_INVALID_ARG; }
  if (N <= 0 || fft_size <= 0) { set_last_error("fftconv_plan: sizes must be positive"); return FFTCONV_ERR_INVALID_ARG; }
  if (!is_pow2(N) || !is_pow2(fft_size)) {
    set_last_error("fftconv_plan: N and fft_size must be powers of two");
    return FFTCONV_ERR_NOT_POW2;
  }
  if (dtype != FFTCONV_F16 && dtype != FFTCONV_BF16 && dtype != FFTCONV_F32) {
    set_last_error("fftconv_plan: unknown dtype");
    return FFTCONV_ERR_INVALID_ARG;
  }
  if (!causal && fft_size != N) {
    set_last_error("fftconv_plan: circular convolution needs fft_size == N");
    return FFTCONV_ERR_INVALID_ARG;
  }
  fftconv_plan_s* p = new (std::nothrow) fftconv_plan_s();
  if (!p) return FFTCONV_ERR_INVALID_ARG;
  p->N = N;
  p->L = fft_size;
  p->causal = causal ? 1 : 0;
  p->dtype = dtype;
  if (causal && fft_size < 2 * N) {
    p->regime = REGIME_PARTIAL;
    p->chunk = fft_size / 2;
  } else {
    p->regime = REGIME_FUSED;
  }
  // Regimes:
  //  fused     : L = L1 * 64, L1 in {8, 16, 32}; causal L = 2N or circular L = N
  //  multipass : causal, L = L0 * 2048 with L0 in {2, 4, 8, 16} (N = 2048..16384)
  const int64_t L = fft_size;
  const bool io_ok = true;  // fp16 / bf16 I/O, or the fp32 validation build
  if (io_ok && p->regime == REGIME_FUSED && L >= 512 && L <= 2048 && (!causal || fft_size == 2 * N)) {
    p->order = 2;
    p->L2 = 64;
    p->L1 = int32_t(L / 64);
    p->KA = causal ? p->L2 / 2 : p->L2;
    p->P = std::max(128 / p->L1, 2);
    build_fused_tables(p, L);
    p->Lp = int32_t(L);
  } else if (io_ok && L >= 4096 && L <= (int64_t(1) << 23) &&
             ((causal && (fft_size == 2 * N || (p->regime == REGIME_PARTIAL && L <= 32768 && N % (L / 2) == 0))) ||
              (!causal && fft_size == N))) {
    // (circular plans, fft_size == N: the paper's circular benchmark rows,
    // P:1243-1244; the outer passes keep every n0 in and out)
    // multipass; the partial regime (K <= L/2 < N) runs the same passes on
    // overlap-save windows of length L (A12).  L / 2048 is split
    // into outer levels of at most 16 (recursive Alg. 4).
    if (p->regime != REGIME_PARTIAL) p->regime = REGIME_MULTIPASS;
    p->Lp = 2048;
    p->L0 = int32_t(L / 2048);
    int r = ilog2(L / 2048);
    p->nlev = (r + 3) / 4;
    for (int l = 0; l < p->nlev; ++l) {
      const int el = r / p->nlev + (l < r % p->nlev ? 1 : 0);
      p->lev_L0[l] = 1 << el;
    }
    // experiments: FFTCONV_LEVELS="a,b[,c]" overrides the outer split (the
    // product must be L / 2048, each factor in {2, 4, 8, 16})
    if (const char* env = getenv("FFTCONV_LEVELS")) {
      int32_t lv[4] = {1, 1, 1, 1}, n = 0;
      int64_t prod = 1;
      for (const char* c = env; *c && n < 4;) {
        const long v = strtol(c, const_cast<char**>(&c), 10);
        if (v == 2 || v == 4 || v == 8 || v == 16) { lv[n++] = int32_t(v); prod *= v; }
        if (*c == ',') ++c; else break;
      }
      if (n > 0 && prod == L / 2048) {
        p->nlev = n;
        for (int l = 0; l < 4; ++l) p->lev_L0[l] = lv[l];
      }
    }
    p->order = 2 + p->nlev;
    p->L2 = 64;
    p->L1 = 32;
    p->KA = 64;  // the inner transform is circular over complex rows
    p->P = 4;
    build_fused_tables(p, p->Lp);
    // single-pass order 3 for causal fft_size 4096 / 8192 / 16384 (N = 2K, 4K,
    // 8K; 8K: the two warpgroups share each row pair, kernels_fwd.cu): the
    // whole row pair stays on chip (decimated inner rows z[n0 + L0 n'] are
    // the tile's complex rows, the outer DFT_L0 runs in the fused kernel's
    // pointwise step).  Not for partial, sparse (row skipping stays with the
    // multipass passes) or fp32 validation plans; FFTCONV_DIT=0 disables it,
    // FFTCONV_DIT=1 takes it wherever it applies (cost-model measurements).
    const char* dit_env = getenv("FFTCONV_DIT");
    if (p->regime == REGIME_MULTIPASS && causal && fft_size == 2 * N && (L == 4096 || L == 8192 || L == 16384) &&
        dtype != FFTCONV_F32 && !sparsity && !(dit_env && dit_env[0] == '0')) {
      fftconv_plan_s t;
      t.L = 2048;
      t.causal = 1;
      t.L2 = 64;
      t.L1 = 32;
      t.KA = 32;
      t.P = 4;
      // NEXT-1: the B200 tier cost model picks order 3 vs multipass for the
      // paper's benchmark shape (B = 64, H = 768; the choice does not depend
      // on B H beyond tile rounding)
      const double t_mp = predict_seconds(p, 64, 768, false, false, nullptr);
      p->dit = int32_t(L / 2048);
      const double t_dit = predict_seconds(p, 64, 768, false, false, nullptr);
      if (t_dit < t_mp || (dit_env && dit_env[0] == '1')) {  // (FFTCONV_DIT=1: always, for measurements)
        build_fused_tables(&t, 2048);
        p->dit_tab_off = align_up(p->image.size(), 1024);
        p->image.resize(p->dit_tab_off, 0);
        p->image.insert(p->image.end(), t.image.begin(), t.image.end());
        p->order = 3;
      } else {
        p->dit = 1;
      }
    }
    if (dtype == FFTCONV_F32 && p->nlev > 1) {
      delete p;
      set_last_error("fftconv_plan: the fp32 validation build supports fft_size <= 32768");
      return FFTCONV_ERR_UNSUPPORTED;
    }
  } else {
    delete p;
    set_last_error("fftconv_plan: this build supports fft_size 512..2048 (fused; causal "
                   "fft_size == 2N or circular), causal fft_size 4096..32768 == 2N (multipass) and partial "
                   "convolutions with fft_size 4096..32768 < 2N dividing 2N (overlap-save)");
    return FFTCONV_ERR_UNSUPPORTED;
  }
  if (sparsity) {
    fftconv_status_t s = build_mask(p, sparsity);
    if (s != FFTCONV_OK) {
      delete p;
      set_last_error("fftconv_plan: inconsistent sparsity pattern (prod(dims) must equal fft_size)");
      return s;
    }
    // the mask rides at the end of the table image (read by precompute_kf),
    // followed by the row keep flags and the list of kept rows, then the
    // compacted stage-B tables of the slow-digit skip
    const size_t mo = p->image.size();
    p->image.resize(mo + p->mask.size() * sizeof(float));
    std::memcpy(p->image.data() + mo, p->mask.data(), p->mask.size() * sizeof(float));
    if (p->L0 > 1) {
      p->row_keep_off = p->image.size();
      std::vector<uint8_t> keep(size_t(p->L0), 0);
      for (int32_t k0 : p->row_map) keep[size_t(k0)] = 1;
      p->image.insert(p->image.end(), keep.begin(), keep.end());
      p->image.resize(align_up(p->image.size(), 16), 0);
      p->row_map_off = p->image.size();
      const size_t bytes = p->row_map.size() * sizeof(int32_t);
      p->image.resize(p->image.size() + align_up(bytes, 16), 0);
      std::memcpy(p->image.data() + p->row_map_off, p->row_map.data(), bytes);
    }
    if (dtype != FFTCONV_F32) build_k1_compact(p);
    else { p->k1_chunks = 0; p->skip_fraction = p->L0 > 1 ? 1.0 - double(p->row_map.size()) / double(p->L0) : 0.0; }
  }
  // fp16 headroom: with unitary stages the largest intermediate of a row
  // pair z = g_b + i g_{b+1} with |g| <= A is its DC bin, |Z_0| <= |z|_1 /
  // sqrt(L) = A sqrt(L/2) (causal, N = L/2 nonzero samples) or A sqrt(2L)
  // (circular).  Keep it <= 2^15 (half of fp16's range, margin for the
  // k_f product) for A = 256 by an exact power-of-two pre-scale.
  if (p->regime == REGIME_MULTIPASS || p->regime == REGIME_PARTIAL) {
    const double amp = 256.0;
    const double peak = amp * std::sqrt((causal ? 0.5 : 2.0) * double(L));
    int sh = 0;
    while (peak / std::ldexp(1.0, sh) > 32768.0) ++sh;
    p->headroom_shift = p->dit > 1 ? 0 : sh;
  }
  // complex fp32 [k2][k1/2] pairs with padded rows, one block per outer index k0
  p->kf_bytes_per_head = size_t(p->L0) * size_t(p->L2) * tab_stride(uint32_t(p->L1 / 2));
  p->ws_bytes_per_head = size_t(L) * 8;  // fp32 spectral accumulator for dk
  *out = p;
  set_last_error("");
  return FFTCONV_OK;
}

extern "C" fftconv_status_t fftconv_plan_info(fftconv_plan_t p, fftconv_plan_info_t* info) {
  if (!p || !info) { set_last_error("fftconv_plan_info: NULL argument"); return FFTCONV_ERR_INVALID_ARG; }
  std::memset(info, 0, sizeof(*info));
  info->N = p->N;
  info->fft_size = p->L;
  info->causal = p->causal;
  info->dtype = p->dtype;
  info->regime = p->regime;
  info->order = p->order;
  if (p->dit > 1) {  // order 3: L0 (outer, in the pointwise step) * L1 * L2
    info->regime = REGIME_FUSED;
    info->factors[0] = p->dit;
    info->factors[1] = p->L1;
    info->factors[2] = p->L2;
  } else if (p->regime == REGIME_MULTIPASS || p->regime == REGIME_PARTIAL) {
    int i = 0;
    for (int l = 0; l < p->nlev && i < FFTCONV_MAX_ORDER - 2; ++l) info->factors[i++] = p->lev_L0[l];
    info->factors[i++] = p->L1;
    info->factors[i++] = p->L2;
  } else {
    info->factors[0] = p->L1;
    info->factors[1] = p->L2;
  }
  info->rows_per_tile = 2 * p->P / p->dit;
  info->max_kernel_len = p->causal ? p->L / 2 : p->L;
  info->table_bytes = p->image.size();
  info->kf_bytes_per_head = p->kf_bytes_per_head;
  info->workspace_bytes_per_head = p->ws_bytes_per_head;
  info->mask_fraction = p->mask_fraction;
  info->skip_fraction = p->skip_fraction;
  return FFTCONV_OK;
}

extern "C" void fftconv_plan_destroy(fftconv_plan_t p) { delete p; }

extern "C" const char* fftconv_last_error(void) { return fc::g_last_error.c_str(); }

// Host-side cost model hooks (tests pin them to the paper's A100 grouping).
extern "C" double fftconv_cost_eq2(int64_t N, int32_t p, double mu, double sigma_h, double sigma_s, double tau_m,
                                   double tau_g, double sram_bytes) {
  CostConstants c{mu, sigma_h, sigma_s, tau_m, tau_g, sram_bytes};
  auto f = factorize(N, p);
  if (f.empty()) return -1.0;
  return cost_eq2(N, f, c, 1.0);
}
extern "C" int32_t fftconv_select_order(int64_t N, double mu, double sigma_h, double sigma_s, double tau_m,
                                        double tau_g, double sram_bytes) {
  CostConstants c{mu, sigma_h, sigma_s, tau_m, tau_g, sram_bytes};
  return select_order(N, c, nullptr);
}
// ---------------------------------------------------------------- B200 tier cost model (NEXT-1)
// Eq. 2 charges each Monarch stage its flops at tau_M / tau_G and
// its intermediate I/O at sigma_S / sigma_H.  On B200 the fused kernels are
// bound by their tile pipeline's latency, not by any of those rates, so the
// B200 model counts the work units of the plan's actual kernels and charges
// each a measured cost: fused tiles per variant (order 2 causal / circular,
// order 3 with L0 = 2 / 4), outer-pass elements (every multipass level
// moves the fp16 intermediate through HBM: Eq. 2's 4N / sigma_H term),
// k_f precompute elements, launches, and the backward's tiles, T-chain
// elements and dk elements.  t = sum_i coef[i] * feat[i]; the default
// coefficients are a least-squares fit to the bench sweep on one B200
// (tools/cost_model.py, profiles/r02c/cost_model.md).
static double cdiv(double a, double b) { return std::ceil(a / b); }

static void cost_features(const fftconv_plan_s* p, int64_t B, int64_t H, bool bwd, bool gated, double* f) {
  for (int i = 0; i < FFTCONV_COST_NFEAT; ++i) f[i] = 0.0;
  const double L = double(p->L), Hd = double(H);
  const bool mp = p->regime == REGIME_MULTIPASS || p->regime == REGIME_PARTIAL;
  const double Bv = p->regime == REGIME_PARTIAL ? double(B) * double(p->N / (p->L / 2)) : double(B);
  const double pairs = std::ceil(Bv / 2.0);
  f[5] = Hd * L;  // k_f precompute
  if (p->dit == 8) {  // coupled row-pair tiles: ~3 L0 = 4 tiles each (16.2k vs 5.4k cycles per pair, traced)
    f[3] = 3.0 * Hd * cdiv(double(B), 2.0);
    f[6] = 4;
  } else if (p->dit > 1) {
    f[p->dit == 2 ? 2 : 3] = Hd * cdiv(double(B), 8.0 / p->dit);
    f[6] = 2;
  } else if (!mp) {
    f[p->causal ? 0 : 1] = Hd * cdiv(double(B), 2.0 * p->P);
    f[6] = 2;
  } else {
    const double kept = p->row_map.empty() ? double(p->L0) : double(p->row_map.size());
    f[1] = Hd * kept * cdiv(2.0 * pairs, 8.0);
    const double lvl = double(p->nlev - 1) + kept / double(p->L0);
    f[4] = lvl * pairs * Hd * L;
    f[6] = 1 + (1 + p->nlev) + (1 + 2 * p->nlev);
  }
  if (bwd) {
    if (!mp && p->dit == 1) {
      f[7] = Hd * cdiv(double(B), 2.0 * p->P);
      f[6] += 2;
    } else {
      const double L0 = double(p->L0);
      f[7] = Hd * L0 * cdiv(2.0 * pairs, 8.0);
      f[8] = 2.0 * double(p->nlev) * pairs * Hd * L;
      f[6] += 2 + 4 * p->nlev + (p->dit > 1 ? 1 : 0);
    }
    f[9] = Hd * L;
  }
  if (gated) f[10] = f[0] + f[1] + f[2] + f[3];
  // algorithmic HBM bytes: 16-bit u, y (+ w, v) per row, fp32 k_f;
  // backward: dy, u (+ w, v) in, du (+ dw, dv) out, dk
  const double el = double(B) * Hd * double(p->N) * 2.0;
  f[11] = el * (gated ? 4.0 : 2.0) + Hd * L * 8.0;
  if (bwd) f[11] += el * (gated ? 7.0 : 3.0) + Hd * L * 8.0;
}

// Default coefficients (seconds per unit; fitted on B200, 1965 MHz).
static const double kCostB200[FFTCONV_COST_NFEAT] = {
    COST_B200_0, COST_B200_1, COST_B200_2, COST_B200_3, COST_B200_4,
    COST_B200_5, COST_B200_6, COST_B200_7, COST_B200_8, COST_B200_9, COST_B200_10, COST_B200_11};

double predict_seconds(const fftconv_plan_s* p, int64_t B, int64_t H, bool bwd, bool gated, const double* coef) {
  double f[FFTCONV_COST_NFEAT];
  cost_features(p, B, H, bwd, gated, f);
  const double* c = coef ? coef : kCostB200;
  double t = 0.0;
  for (int i = 0; i < FFTCONV_COST_NFEAT; ++i) t += c[i] * f[i];
  return t;
}

extern "C" fftconv_status_t fftconv_cost_features(fftconv_plan_t p, int64_t B, int64_t H, int bwd, int gated,
                                                  double* feat) {
  if (!p || !feat || B < 0 || H < 0) { set_last_error("fftconv_cost_features: bad argument"); return FFTCONV_ERR_INVALID_ARG; }
  cost_features(p, B, H, bwd != 0, gated != 0, feat);
  return FFTCONV_OK;
}
extern "C" fftconv_status_t fftconv_cost_predict(fftconv_plan_t p, int64_t B, int64_t H, int bwd, int gated,
                                                 const double* coef, double* seconds) {
  if (!p || !seconds || B < 0 || H < 0) { set_last_error("fftconv_cost_predict: bad argument"); return FFTCONV_ERR_INVALID_ARG; }
  *seconds = predict_seconds(p, B, H, bwd != 0, gated != 0, coef);
  return FFTCONV_OK;
}

extern "C" int32_t fftconv_factorize(int64_t n, int32_t p, int64_t* out) {
  auto f = factorize(n, p);
  for (size_t i = 0; i < f.size(); ++i) out[i] = f[i];
  return int32_t(f.size());
}
