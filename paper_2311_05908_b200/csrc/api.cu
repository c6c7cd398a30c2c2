// api.cu -- C-ABI entry points (include/fftconv.h): argument validation,
// table upload and kernel launches.  Every device-side step of the path runs
// in this library's own kernels; there is no CPU fallback.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fftconv.h"
#include "fwd_params.h"
#include "plan.h"
#include "layout.h"

using namespace fc;

namespace {
thread_local int64_t g_launches = 0;

// Chunk size of the multipass intermediate kept in L2 (bytes); FFTCONV_CHUNK_MB
// overrides it for experiments (0 = one chunk, the default: measured on B200,
// chunks of 16-96 MB were 3-50% slower -- the passes are not HBM-bound).
size_t chunk_target_bytes() {
  static size_t v = [] {
    const char* e = getenv("FFTCONV_CHUNK_MB");
    const long mb = e ? atol(e) : 0;
    return mb > 0 ? size_t(mb) << 20 : ~size_t(0) >> 1;
  }();
  return v;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeTiledFn(nullptr);
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// The multipass inner pass stores its tiles with TMA tensor stores unless
// FFTCONV_TMA_Y=0 (experiments).
bool tma_y_enabled() {
  static bool v = [] {
    const char* e = getenv("FFTCONV_TMA_Y");
    return !(e && e[0] == '0');
  }();
  return v;
}

// bytes per element of the multipass intermediate T (fp16; fp32 in the
// validation build)
size_t t_elem_bytes(const fftconv_plan_s* p) { return p->dtype == FFTCONV_F32 ? 4 : 2; }

int num_sms_current() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

fftconv_status_t cuda_fail(const char* what, cudaError_t e) {
  set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FFTCONV_ERR_CUDA;
}

fftconv_status_t check_signal_args(fftconv_plan_t p, const char* fn, int64_t B, int64_t H,
                                   std::initializer_list<const void*> ptrs) {
  if (!p) { set_last_error(std::string(fn) + ": plan is NULL"); return FFTCONV_ERR_INVALID_ARG; }
  if (!p->d_tables) { set_last_error(std::string(fn) + ": plan tables not uploaded"); return FFTCONV_ERR_INVALID_ARG; }
  if (B < 0 || H < 0) { set_last_error(std::string(fn) + ": negative B or H"); return FFTCONV_ERR_INVALID_ARG; }
  for (const void* q : ptrs) {
    if (!q && B * H > 0) { set_last_error(std::string(fn) + ": NULL device pointer"); return FFTCONV_ERR_INVALID_ARG; }
    if (q && !aligned16(q)) { set_last_error(std::string(fn) + ": device pointer not 16-byte aligned"); return FFTCONV_ERR_MISALIGNED; }
  }
  return FFTCONV_OK;
}
}  // namespace

extern "C" fftconv_status_t fftconv_plan_upload(fftconv_plan_t p, void* d_tables, fftconv_stream_t stream) {
  if (!p || !d_tables) { set_last_error("fftconv_plan_upload: NULL argument"); return FFTCONV_ERR_INVALID_ARG; }
  if ((reinterpret_cast<uintptr_t>(d_tables) & 1023u) != 0) {
    set_last_error("fftconv_plan_upload: table buffer must be 1024-byte aligned");
    return FFTCONV_ERR_MISALIGNED;
  }
  cudaError_t e = cudaMemcpyAsync(d_tables, p->image.data(), p->image.size(), cudaMemcpyHostToDevice,
                                  reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("fftconv_plan_upload", e);
  // the host image must stay valid until the copy completes (pageable copy is
  // staged synchronously by the driver, but be explicit)
  e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("fftconv_plan_upload", e);
  p->d_tables = d_tables;
  return FFTCONV_OK;
}

namespace fc {
cudaError_t make_tmap_rows(CUtensorMap* map, void* base, int64_t rows, int64_t heads, int64_t Lp, int R) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return cudaErrorNotSupported;
  // dims by increasing stride: element in a 128 B segment, segment, head, row
  const cuuint64_t dim[4] = {64, cuuint64_t(Lp / 64), cuuint64_t(heads), cuuint64_t(rows)};
  const cuuint64_t stride[3] = {128, cuuint64_t(Lp) * 2, cuuint64_t(heads) * cuuint64_t(Lp) * 2};
  const cuuint32_t box[4] = {64, cuuint32_t(Lp / 64), 1, cuuint32_t(R)};
  const cuuint32_t estride[4] = {1, 1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, base, dim, stride, box, estride,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
// Coupled order-3 tiles (L0 = 8): one row's first N samples n = n0 + 8 (n1 +
// 32 n2) as a box ordered (n0, n2, n1) -- SMEM offset (n1 * N/256 + n2) * 16
// + 2 n0 -- so the epilogue-4 threads, which hold consecutive n2, write
// consecutive 16 B units; one box per row (rows = b * H + h; rows past B*H
// are zero-filled on load and clipped on store).
cudaError_t make_tmap_cpl(CUtensorMap* map, const void* base, int64_t B, int64_t H, int64_t N) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dim[4] = {8, cuuint64_t(N / 256), 32, cuuint64_t(B * H)};
  const cuuint64_t stride[3] = {512, 16, cuuint64_t(N) * 2};
  const cuuint32_t box[4] = {8, cuuint32_t(N / 256), 32, 1};
  const cuuint32_t estride[4] = {1, 1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(base), dim, stride, box, estride,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
cudaError_t make_tmap_sig(CUtensorMap* map, const void* base, int64_t B, int64_t H, int64_t N, int R) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc || N % 256 != 0) return cudaErrorNotSupported;
  // dims by increasing stride: element in a 512 B segment, segment, head, batch row
  const cuuint64_t dim[4] = {256, cuuint64_t(N / 256), cuuint64_t(H), cuuint64_t(B)};
  const cuuint64_t stride[3] = {512, cuuint64_t(N) * 2, cuuint64_t(H) * cuuint64_t(N) * 2};
  const cuuint32_t box[4] = {256, cuuint32_t(N / 256), 1, cuuint32_t(R)};
  const cuuint32_t estride[4] = {1, 1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, const_cast<void*>(base), dim, stride, box, estride,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
}  // namespace fc

static fftconv_status_t run_precompute(fftconv_plan_t p, const float* d_k, const float* d_kb, int64_t H, int64_t K,
                                       void* d_kf, fftconv_stream_t stream, bool bidir) {
  if (!p) { set_last_error("fftconv_precompute_kf: plan is NULL"); return FFTCONV_ERR_INVALID_ARG; }
  if (!p->d_tables) { set_last_error("fftconv_precompute_kf: plan tables not uploaded"); return FFTCONV_ERR_INVALID_ARG; }
  if (H < 0 || K < 1) { set_last_error("fftconv_precompute_kf: need H >= 0 and K >= 1"); return FFTCONV_ERR_INVALID_ARG; }
  const int64_t kmax = p->causal ? p->L / 2 : p->L;
  if (K > kmax) { set_last_error("fftconv_precompute_kf: kernel exceeds causal budget"); return FFTCONV_ERR_KERNEL_TOO_LONG; }
  if (H > 0 && (!d_k || !d_kf)) { set_last_error("fftconv_precompute_kf: NULL device pointer"); return FFTCONV_ERR_INVALID_ARG; }
  if (d_kf && !aligned16(d_kf)) { set_last_error("fftconv_precompute_kf: k_f not 16-byte aligned"); return FFTCONV_ERR_MISALIGNED; }
  if (bidir) {  // bidirectional: full causal plans (fft_size = 2N), dense
    if (H > 0 && !d_kb) { set_last_error("fftconv_precompute_kf_bidir: NULL device pointer"); return FFTCONV_ERR_INVALID_ARG; }
    if (!p->causal || p->regime == REGIME_PARTIAL || p->L != 2 * p->N || p->sparse) {
      set_last_error("fftconv_precompute_kf_bidir: needs a dense full causal plan (fft_size == 2N)");
      return FFTCONV_ERR_UNSUPPORTED;
    }
  }
  KfParams prm{};
  prm.k = d_k;
  prm.kb = d_kb;
  prm.Lk = p->L;
  prm.kf = d_kf;
  prm.mask = p->sparse ? reinterpret_cast<const float*>(static_cast<const uint8_t*>(p->d_tables) + p->tl.total)
                       : nullptr;
  prm.twiddle = reinterpret_cast<const float2*>(static_cast<const uint8_t*>(p->d_tables) + p->tl.wl);
  prm.H = H;
  prm.K = K;
  prm.L = p->L;
  prm.L1 = p->L1;
  prm.L2 = p->L2;
  cudaError_t e;
  if (p->dit > 1) {  // single-pass order 3: L0 blocks of K_f[f' + 2048 k0] per head
    e = launch_precompute_kf_dit(prm, p->dit, reinterpret_cast<cudaStream_t>(stream));
    g_launches += H > 0 ? 1 : 0;
  } else if (p->regime == REGIME_MULTIPASS || p->regime == REGIME_PARTIAL) {
    const size_t block = size_t(p->L2) * tab_stride(uint32_t(p->L1 / 2));
    prm.L = p->Lp;
    if (p->sparse && p->row_map.size() < size_t(p->L0))
      prm.row_keep = static_cast<const uint8_t*>(p->d_tables) + p->row_keep_off;
    prm.nlev = p->nlev;
    for (int l = 0; l < 4; ++l) prm.lev[l] = p->lev_L0[l];
    e = launch_mp_precompute_kf(prm, p->lev_L0, p->nlev, p->L, block, reinterpret_cast<cudaStream_t>(stream));
    g_launches += H > 0 ? 2 + p->nlev - 1 : 0;
  } else {
    e = launch_precompute_kf(prm, reinterpret_cast<cudaStream_t>(stream));
    g_launches += H > 0 ? 1 : 0;
  }
  if (e != cudaSuccess) return cuda_fail("fftconv_precompute_kf", e);
  return FFTCONV_OK;
}

extern "C" fftconv_status_t fftconv_precompute_kf(fftconv_plan_t p, const float* d_k, int64_t H, int64_t K,
                                                  void* d_kf, fftconv_stream_t stream) {
  return run_precompute(p, d_k, nullptr, H, K, d_kf, stream, false);
}

extern "C" fftconv_status_t fftconv_precompute_kf_bidir(fftconv_plan_t p, const float* d_k_fwd, const float* d_k_bwd,
                                                        int64_t H, int64_t K, void* d_kf, fftconv_stream_t stream) {
  return run_precompute(p, d_k_fwd, d_k_bwd, H, K, d_kf, stream, true);
}

// frequency-sparse slow-digit skip of the fused kernel (plan.cpp build_mask)
static void set_k1_skip(fftconv_plan_t p, FwdParams& prm) {
  if (p->k1_chunks <= 0) return;
  prm.kcn = p->k1_chunks;
  prm.k1map = p->k1_map;
  prm.off_gb = uint32_t(p->gb_sp);
  prm.off_gbi = uint32_t(p->gbi_sp);
}

static fftconv_status_t run_fwd(fftconv_plan_t p, const void* u, const void* w, const void* v, const void* kf,
                                void* y, int64_t B, int64_t H, void* ws, fftconv_stream_t stream, const char* fn) {
  const bool gated = (w != nullptr);
  fftconv_status_t chk = gated ? check_signal_args(p, fn, B, H, {u, w, v, kf, y}) : check_signal_args(p, fn, B, H, {u, kf, y});
  if (chk != FFTCONV_OK) return chk;
  if (gated && !v) { set_last_error(std::string(fn) + ": v is NULL"); return FFTCONV_ERR_INVALID_ARG; }
  if (B * H == 0) return FFTCONV_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (p->dit > 1) {  // single-pass order 3: one fused launch, no workspace
    FwdParams prm{};
    prm.u = u; prm.w = w; prm.v = v; prm.y = y; prm.kf = kf;
    prm.tables = static_cast<const uint8_t*>(p->d_tables) + p->dit_tab_off;
    prm.B = B; prm.H = H; prm.N = p->N; prm.L1 = 32; prm.causal = 1;
    prm.gated = gated ? 1 : 0;
    prm.dtype = p->dtype == FFTCONV_BF16 ? 1 : 0;
    prm.num_sms = num_sms_current();
    prm.L0I = p->dit;
    const int R = p->dit == 8 ? 2 : 8 / p->dit;  // real rows per tile (L0 = 8: one pair, coupled warpgroups)
    // u, w: natural-order boxes; v, y: 128 B swizzled boxes (epilogue 4
    // gates and stages 16-byte units in place) -- gated L0 = 4 tiles keep
    // natural-order v and y (their epilogue 4 gates in a second pass)
    const bool natural = gated && p->dit == 4 && !FC_O3G4_DIRECT;  // (kernels_fwd.cu: Y_DIRECT)
    // (L0 = 8: u, w arrive 128 B swizzled too -- each thread reads one 128 B
    // line of a row, the swizzle spreads 8 lanes' lines over all banks)
    const bool swz_in = p->dit == 8;
    bool ok = (swz_in ? make_tmap_rows(&prm.tmap_u, const_cast<void*>(u), B, H, p->N, R)
                      : make_tmap_sig(&prm.tmap_u, u, B, H, p->N, R)) == cudaSuccess &&
              (swz_in  ? make_tmap_cpl(&prm.tmap_yo, y, B, H, p->N)
               : natural ? make_tmap_sig(&prm.tmap_yo, y, B, H, p->N, R)
                         : make_tmap_rows(&prm.tmap_yo, y, B, H, p->N, R)) == cudaSuccess;
    if (ok && gated)
      ok = (swz_in ? make_tmap_rows(&prm.tmap_w, const_cast<void*>(w), B, H, p->N, R)
                   : make_tmap_sig(&prm.tmap_w, w, B, H, p->N, R)) == cudaSuccess &&
           (swz_in  ? make_tmap_cpl(&prm.tmap_v, v, B, H, p->N)
            : natural ? make_tmap_sig(&prm.tmap_v, v, B, H, p->N, R)
                      : make_tmap_rows(&prm.tmap_v, const_cast<void*>(v), B, H, p->N, R)) == cudaSuccess;
    prm.tma_io = ok ? 1 : 0;
    cudaError_t e = launch_fwd_fused(prm, st);
    if (e != cudaSuccess) return cuda_fail(fn, e);
    g_launches += 1;
    return FFTCONV_OK;
  }
  if (p->regime == REGIME_MULTIPASS || p->regime == REGIME_PARTIAL) {
    if (!ws) { set_last_error(std::string(fn) + ": multipass regime needs a workspace"); return FFTCONV_ERR_INVALID_ARG; }
    if (!aligned16(ws)) { set_last_error(std::string(fn) + ": workspace not 16-byte aligned"); return FFTCONV_ERR_MISALIGNED; }
    MpParams mp{};
    mp.shift = p->headroom_shift;  // fp16 headroom pre-scale (top-level passes only)
    mp.u = u; mp.w = w; mp.v = v; mp.y = y; mp.ws = ws;
    mp.L0 = p->lev_L0[0];
    mp.wbase = reinterpret_cast<const float2*>(static_cast<const uint8_t*>(p->d_tables) + p->tl.wbase);
    mp.wtab = reinterpret_cast<const float2*>(static_cast<const uint8_t*>(p->d_tables) + p->tl.wtab);
    mp.B = B; mp.H = H; mp.N = p->N; mp.Lp = int32_t(p->L / p->lev_L0[0]);
    mp.gated = gated ? 1 : 0;
    mp.dtype = p->dtype == FFTCONV_BF16 ? 1 : p->dtype == FFTCONV_F32 ? 2 : 0;
    const bool skip = p->sparse && p->row_map.size() < size_t(p->L0);
    if (skip) {
      mp.row_keep = static_cast<const uint8_t*>(p->d_tables) + p->row_keep_off;
      if (p->nlev == 1) {  // outer passes produce / consume only the kept rows
        mp.row_map = reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(p->d_tables) + p->row_map_off);
        mp.nrow = int32_t(p->row_map.size());
      }
    }
    if (p->regime == REGIME_PARTIAL) {  // overlap-save windows as virtual rows
      mp.partial = 1;
      mp.C = p->L / 2;
      mp.NC = p->N / mp.C;
      mp.B = B * mp.NC;
    }
    if (p->nlev > 1) mp.wtab = nullptr;  // deep plans: outer twiddles on the fly
    mp.Llev = p->L;
    mp.circ = p->causal ? 0 : 1;  // circular plan: every n0 in and out
    if (p->nlev == 1) {
      // One outer level: run the three passes chunk by chunk over (pairs,
      // heads) so the chunk's intermediate T stays resident in L2 between
      // pass 1, the inner pass and pass 3 (Alg. 4's extra I/O, then
      // never reaches HBM); chunks reuse the start of the workspace.
      const int64_t Bv = mp.B, pairs = (Bv + 1) / 2;
      const size_t per_pair_head = size_t(4) * size_t(p->L);  // fp16 re + im planes
      const size_t target = chunk_target_bytes();
      int64_t Hc = H, Pc = pairs;
      if (size_t(pairs) * per_pair_head * size_t(H) > target) {
        Hc = int64_t(target / (size_t(pairs) * per_pair_head));
        if (Hc < 1) {
          Hc = 1;
          Pc = int64_t(target / per_pair_head);
          if (Pc < 1) Pc = 1;
        }
      }
      int launches = 0;
      for (int64_t pc0 = 0; pc0 < pairs; pc0 += Pc) {
        const int64_t rows_c = (2 * (pc0 + Pc) < Bv ? 2 * Pc : Bv - 2 * pc0);
        for (int64_t h0 = 0; h0 < H; h0 += Hc) {
          const int64_t hc = H - h0 < Hc ? H - h0 : Hc;
          MpParams c = mp;
          c.B = rows_c; c.H = hc; c.h0 = h0; c.Hg = H; c.pair0 = pc0; c.ws = ws;
          cudaError_t e = launch_mp_pass(c, 1, st);
          if (e != cudaSuccess) return cuda_fail(fn, e);
          FwdParams in{};
          in.u = ws; in.y = ws; in.tables = p->d_tables;
          if (tma_y_enabled() && p->dtype != FFTCONV_F32 &&
              make_tmap_rows(&in.tmap_y, ws, 2 * ((rows_c + 1) / 2), hc * p->L0, p->Lp, 8) == cudaSuccess)
            in.tma_y = 1;
          // the inner tiles' input rows arrive by one TMA tensor load each
          in.tma_io = make_tmap_sig(&in.tmap_u, ws, 2 * ((rows_c + 1) / 2), hc * p->L0, p->Lp, 8) == cudaSuccess;
          in.kf = static_cast<const uint8_t*>(kf) + size_t(h0) * p->kf_bytes_per_head;
          in.B = 2 * ((rows_c + 1) / 2); in.H = hc * p->L0; in.N = p->Lp;
          in.L1 = p->L1; in.causal = 0; in.gated = 0; in.dtype = 0;
          in.num_sms = num_sms_current();
          if (p->dtype == FFTCONV_F32) {  // validation build: fp32 rows, every inner row
            in.dtype = 2;
            in.wl = static_cast<const uint8_t*>(p->d_tables) + p->tl.wl;
            e = launch_fwd_f32(in, st);
          } else {
            if (skip) {
              in.row_map = reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(p->d_tables) + p->row_map_off);
              in.nrow = int32_t(p->row_map.size());
              in.row_L0 = p->L0;
            }
            set_k1_skip(p, in);
            e = launch_fwd_fused(in, st);
          }
          if (e != cudaSuccess) return cuda_fail(fn, e);
          e = launch_mp_pass(c, 3, st);
          if (e != cudaSuccess) return cuda_fail(fn, e);
          launches += 3;
        }
      }
      g_launches += launches;
      return FFTCONV_OK;
    }
    const int64_t rows = 2 * ((mp.B + 1) / 2);
    const size_t tbytes = size_t(rows) * size_t(H) * size_t(p->L) * 2;
    void* Tb[2] = {ws, static_cast<uint8_t*>(ws) + tbytes};
    cudaError_t e = launch_mp_pass(mp, 1, st);
    if (e != cudaSuccess) return cuda_fail(fn, e);
    // deeper outer levels: complex circular rows, ping-pong between T buffers
    auto level = [&](int l) {  // params of level l >= 1 (0-based)
      MpParams q{};
      int64_t Hl = H, Ll = p->L;
      for (int j = 0; j < l; ++j) { Hl *= p->lev_L0[j]; Ll /= p->lev_L0[j]; }
      q.B = rows; q.H = Hl; q.N = Ll; q.L0 = p->lev_L0[l]; q.Lp = int32_t(Ll / p->lev_L0[l]);
      q.Llev = Ll; q.circ = 1; q.dtype = 0; q.gated = 0;
      q.u = Tb[(l - 1) & 1]; q.ws = Tb[l & 1]; q.y = Tb[(l - 1) & 1];
      return q;
    };
    for (int l = 1; l < p->nlev; ++l) {
      e = launch_mp_pass(level(l), 1, st);
      if (e != cudaSuccess) return cuda_fail(fn, e);
    }
    // inner pass: the fused circular kernel over the complex rows, in place
    void* Tin = Tb[(p->nlev - 1) & 1];
    FwdParams in{};
    in.u = Tin; in.y = Tin; in.kf = kf; in.tables = p->d_tables;
    if (tma_y_enabled() && make_tmap_rows(&in.tmap_y, Tin, rows, H * p->L0, p->Lp, 8) == cudaSuccess) in.tma_y = 1;
    in.tma_io = make_tmap_sig(&in.tmap_u, Tin, rows, H * p->L0, p->Lp, 8) == cudaSuccess;
    in.B = rows; in.H = H * p->L0; in.N = p->Lp;
    in.L1 = p->L1; in.causal = 0; in.gated = 0; in.dtype = 0;
    in.num_sms = num_sms_current();
    if (skip) {  // frequency-sparse: only rows k0 with a non-zero mask are transformed
      in.row_map = reinterpret_cast<const int32_t*>(static_cast<const uint8_t*>(p->d_tables) + p->row_map_off);
      in.nrow = int32_t(p->row_map.size());
      in.row_L0 = p->L0;
    }
    set_k1_skip(p, in);
    e = launch_fwd_fused(in, st);
    if (e != cudaSuccess) return cuda_fail(fn, e);
    for (int l = p->nlev - 1; l >= 1; --l) {
      e = launch_mp_pass(level(l), 3, st);
      if (e != cudaSuccess) return cuda_fail(fn, e);
    }
    mp.ws = Tb[0];
    e = launch_mp_pass(mp, 3, st);
    if (e != cudaSuccess) return cuda_fail(fn, e);
    g_launches += 1 + 2 * p->nlev;
    return FFTCONV_OK;
  }
  if (p->regime != REGIME_FUSED) { set_last_error(std::string(fn) + ": regime not supported by this build"); return FFTCONV_ERR_UNSUPPORTED; }
  FwdParams prm{};
  prm.u = u;
  prm.w = w;
  prm.v = v;
  prm.y = y;
  prm.kf = kf;
  prm.tables = p->d_tables;
  prm.B = B;
  prm.H = H;
  prm.N = p->N;
  prm.L1 = p->L1;
  prm.causal = p->causal;
  prm.gated = gated ? 1 : 0;
  prm.dtype = p->dtype == FFTCONV_BF16 ? 1 : p->dtype == FFTCONV_F32 ? 2 : 0;
  prm.num_sms = num_sms_current();
  prm.wl = static_cast<const uint8_t*>(p->d_tables) + p->tl.wl;
  prm.L0I = 1;
  if (p->causal && p->dtype != FFTCONV_F32 && tma_y_enabled()) {  // one tensor copy per tile and tensor
    const int R = 2 * p->P;
    bool ok = make_tmap_sig(&prm.tmap_u, u, B, H, p->N, R) == cudaSuccess &&
              make_tmap_rows(&prm.tmap_yo, y, B, H, p->N, R) == cudaSuccess;
    if (ok && gated)
      ok = make_tmap_sig(&prm.tmap_w, w, B, H, p->N, R) == cudaSuccess &&
           make_tmap_rows(&prm.tmap_v, const_cast<void*>(v), B, H, p->N, R) == cudaSuccess;
    prm.tma_io = ok ? 1 : 0;
  } else if (!p->causal && !gated && p->dtype != FFTCONV_F32) {  // circular plain: input rows by TMA
    prm.tma_io = make_tmap_sig(&prm.tmap_u, u, B, H, p->N, 2 * p->P) == cudaSuccess;
  }
  set_k1_skip(p, prm);
  cudaError_t e = p->dtype == FFTCONV_F32 ? launch_fwd_f32(prm, st) : launch_fwd_fused(prm, st);
  if (e != cudaSuccess) return cuda_fail(fn, e);
  g_launches += 1;
  return FFTCONV_OK;
}

extern "C" fftconv_status_t fftconv_fwd(fftconv_plan_t p, const void* d_u, const void* d_kf, void* d_y, int64_t B,
                                        int64_t H, void* d_workspace, fftconv_stream_t stream) {
  return run_fwd(p, d_u, nullptr, nullptr, d_kf, d_y, B, H, d_workspace, stream, "fftconv_fwd");
}

extern "C" fftconv_status_t fftconv_gated_fwd(fftconv_plan_t p, const void* d_u, const void* d_w, const void* d_v,
                                              const void* d_kf, void* d_y, int64_t B, int64_t H, void* d_workspace,
                                              fftconv_stream_t stream) {
  if (!d_w || !d_v) { set_last_error("fftconv_gated_fwd: w and v are required"); return FFTCONV_ERR_INVALID_ARG; }
  return run_fwd(p, d_u, d_w, d_v, d_kf, d_y, B, H, d_workspace, stream, "fftconv_gated_fwd");
}

// ---------------------------------------------------------------- host streaming
// Device staging slot for `rows` batch rows: u | (w | v) | y | workspace.
static size_t elem_bytes(const fftconv_plan_s* p) { return p->dtype == FFTCONV_F32 ? 4 : 2; }
static size_t slot_bytes(fftconv_plan_t p, int64_t H, int64_t rows, bool gated, size_t* ws_bytes) {
  const size_t t = (size_t(rows) * size_t(H) * size_t(p->N) * elem_bytes(p) + 1023) / 1024 * 1024;
  size_t ws = 0;
  fftconv_workspace_size(p, rows, H, 0, &ws);
  ws = (ws + 1023) / 1024 * 1024;
  if (ws_bytes) *ws_bytes = ws;
  return t * (gated ? 4 : 2) + ws;
}

extern "C" fftconv_status_t fftconv_host_stage_size(fftconv_plan_t p, int64_t H, int64_t rows_per_chunk, int gated,
                                                    size_t* bytes) {
  if (!p || !bytes || H < 0 || rows_per_chunk < 1) {
    set_last_error("fftconv_host_stage_size: bad argument");
    return FFTCONV_ERR_INVALID_ARG;
  }
  const int64_t rc = rows_per_chunk + (rows_per_chunk & 1);  // chunks keep row pairs together
  *bytes = 2 * slot_bytes(p, H, rc, gated != 0, nullptr) + 1024;
  return FFTCONV_OK;
}

namespace {
// Per-device copy-in / copy-out streams and chunk events, created once.
// The pipe's events are re-recorded by every call, so a call holds the
// pipe's mutex for its whole enqueue sequence: a second host thread on the
// same device cannot re-record computed[s] / start between another call's
// record and wait (its copies queue behind the first call's on the same
// copy streams).
struct HostPipe {
  std::mutex mu;
  cudaStream_t in = nullptr, out = nullptr;
  cudaEvent_t start = nullptr, done = nullptr;
  cudaEvent_t loaded[2] = {}, computed[2] = {}, freed[2] = {};
};
std::mutex g_pipe_mu;
HostPipe g_pipes[64];
cudaError_t host_pipe(HostPipe** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  HostPipe& hp = g_pipes[dev];
  if (!hp.in) {
    const unsigned f = cudaStreamNonBlocking, ef = cudaEventDisableTiming;
    if ((e = cudaStreamCreateWithFlags(&hp.in, f)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&hp.out, f)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&hp.start, ef)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&hp.done, ef)) != cudaSuccess) return e;
    for (int i = 0; i < 2; ++i) {
      if ((e = cudaEventCreateWithFlags(&hp.loaded[i], ef)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&hp.computed[i], ef)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&hp.freed[i], ef)) != cudaSuccess) return e;
    }
  }
  *out = &hp;
  return cudaSuccess;
}
// A failed call still orders the caller's stream after every copy it queued,
// so the caller may free its buffers once its stream has drained.
fftconv_status_t drain_pipe(HostPipe* hp, cudaStream_t cs, fftconv_status_t st) {
  if (cudaEventRecord(hp->done, hp->in) == cudaSuccess) cudaStreamWaitEvent(cs, hp->done, 0);
  if (cudaEventRecord(hp->done, hp->out) == cudaSuccess) cudaStreamWaitEvent(cs, hp->done, 0);
  return st;
}
}  // namespace

extern "C" fftconv_status_t fftconv_fwd_host(fftconv_plan_t p, const void* h_u, const void* h_w, const void* h_v,
                                             const void* d_kf, void* h_y, int64_t B, int64_t H,
                                             int64_t rows_per_chunk, void* d_stage, size_t stage_bytes,
                                             fftconv_stream_t stream) {
  const char* fn = "fftconv_fwd_host";
  if (!p) { set_last_error("fftconv_fwd_host: plan is NULL"); return FFTCONV_ERR_INVALID_ARG; }
  const bool gated = h_w != nullptr || h_v != nullptr;
  if (gated && !(h_w && h_v)) { set_last_error("fftconv_fwd_host: gated needs both w and v"); return FFTCONV_ERR_INVALID_ARG; }
  if (B < 0 || H < 0 || rows_per_chunk < 1) { set_last_error("fftconv_fwd_host: bad sizes"); return FFTCONV_ERR_INVALID_ARG; }
  if (B * H == 0) return FFTCONV_OK;
  if (!h_u || !h_y || !d_kf || !d_stage) { set_last_error("fftconv_fwd_host: NULL pointer"); return FFTCONV_ERR_INVALID_ARG; }
  if (!aligned16(d_stage)) { set_last_error("fftconv_fwd_host: stage not 16-byte aligned"); return FFTCONV_ERR_MISALIGNED; }
  // chunks hold an even number of rows so every row keeps its packing
  // partner (two real rows per complex transform): results are bitwise
  // those of one fftconv_fwd / fftconv_gated_fwd call on all B rows
  const int64_t rpc = rows_per_chunk + (rows_per_chunk & 1);
  const int64_t rc = rpc < B ? rpc : B;
  size_t ws_bytes = 0;
  const size_t slot = slot_bytes(p, H, rc, gated, &ws_bytes);
  if (stage_bytes < 2 * slot) { set_last_error("fftconv_fwd_host: staging buffer too small"); return FFTCONV_ERR_INVALID_ARG; }
  {  // every argument run_fwd checks, before any copy is enqueued (the staged pointers stand in for the chunk buffers)
    fftconv_status_t chk = check_signal_args(p, fn, rc, H, {d_stage, d_kf});
    if (chk != FFTCONV_OK) return chk;
  }
  HostPipe* hp = nullptr;
  cudaError_t e = host_pipe(&hp);
  if (e != cudaSuccess) return cuda_fail(fn, e);
  std::lock_guard<std::mutex> pipe_lock(hp->mu);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  // the pipeline starts after earlier work on the caller's stream
  if ((e = cudaEventRecord(hp->start, cs)) != cudaSuccess) return cuda_fail(fn, e);
  if ((e = cudaStreamWaitEvent(hp->in, hp->start, 0)) != cudaSuccess) return cuda_fail(fn, e);
  if ((e = cudaStreamWaitEvent(hp->out, hp->start, 0)) != cudaSuccess) return cuda_fail(fn, e);
  const size_t row_bytes = size_t(H) * size_t(p->N) * elem_bytes(p);
  const size_t t = (size_t(rc) * row_bytes + 1023) / 1024 * 1024;
  uint8_t* base = static_cast<uint8_t*>(d_stage);
  const int64_t nchunks = (B + rc - 1) / rc;
  for (int64_t i = 0; i < nchunks; ++i) {
    const int s = int(i & 1);
    const int64_t b0 = i * rc, rows = (B - b0 < rc ? B - b0 : rc);
    const size_t off = size_t(b0) * row_bytes, nb = size_t(rows) * row_bytes;
    uint8_t* sl = base + size_t(s) * slot;
    uint8_t *du = sl, *dw = sl + t, *dv = sl + 2 * t, *dy = sl + (gated ? 3 : 1) * t, *dws = sl + (gated ? 4 : 2) * t;
    // copy in (slot reusable once the copy-out of chunk i-2 has finished)
    if (i >= 2 && (e = cudaStreamWaitEvent(hp->in, hp->freed[s], 0)) != cudaSuccess) return cuda_fail(fn, e);
    if ((e = cudaMemcpyAsync(du, static_cast<const uint8_t*>(h_u) + off, nb, cudaMemcpyHostToDevice, hp->in)) != cudaSuccess)
      return cuda_fail(fn, e);
    if (gated) {
      if ((e = cudaMemcpyAsync(dw, static_cast<const uint8_t*>(h_w) + off, nb, cudaMemcpyHostToDevice, hp->in)) != cudaSuccess)
        return cuda_fail(fn, e);
      if ((e = cudaMemcpyAsync(dv, static_cast<const uint8_t*>(h_v) + off, nb, cudaMemcpyHostToDevice, hp->in)) != cudaSuccess)
        return cuda_fail(fn, e);
    }
    if ((e = cudaEventRecord(hp->loaded[s], hp->in)) != cudaSuccess) return cuda_fail(fn, e);
    // convolution on the caller's stream
    if ((e = cudaStreamWaitEvent(cs, hp->loaded[s], 0)) != cudaSuccess) return cuda_fail(fn, e);
    fftconv_status_t st = run_fwd(p, du, gated ? dw : nullptr, gated ? dv : nullptr, d_kf, dy, rows, H,
                                  ws_bytes ? dws : nullptr, stream, fn);
    if (st != FFTCONV_OK) return drain_pipe(hp, cs, st);
    if ((e = cudaEventRecord(hp->computed[s], cs)) != cudaSuccess) return cuda_fail(fn, e);
    // copy out
    if ((e = cudaStreamWaitEvent(hp->out, hp->computed[s], 0)) != cudaSuccess) return cuda_fail(fn, e);
    if ((e = cudaMemcpyAsync(static_cast<uint8_t*>(h_y) + off, dy, nb, cudaMemcpyDeviceToHost, hp->out)) != cudaSuccess)
      return cuda_fail(fn, e);
    if ((e = cudaEventRecord(hp->freed[s], hp->out)) != cudaSuccess) return cuda_fail(fn, e);
  }
  // later work on the caller's stream sees every chunk of h_y
  if ((e = cudaEventRecord(hp->done, hp->out)) != cudaSuccess) return cuda_fail(fn, e);
  if ((e = cudaStreamWaitEvent(cs, hp->done, 0)) != cudaSuccess) return cuda_fail(fn, e);
  return FFTCONV_OK;
}

// ---------------------------------------------------------------- sequence streaming (NEXT-4)
// Partial plans only (K <= C = fft_size/2): rows longer than the plan's N are
// streamed from host memory in segments.  Segment i covers outputs
// [i S, (i+1) S) with S = N - C; its device buffer holds u[i S - C, i S + S)
// (zeros before 0 and past the end), so the overlap-save windows of the plan
// see the C-sample history they need and outputs C.. of the buffer are exact.
extern "C" fftconv_status_t fftconv_stream_stage_size(fftconv_plan_t p, int64_t B, int64_t H, int gated,
                                                      size_t* bytes) {
  if (!p || !bytes || B < 1 || H < 1) { set_last_error("fftconv_stream_stage_size: bad argument"); return FFTCONV_ERR_INVALID_ARG; }
  if (p->regime != REGIME_PARTIAL) { set_last_error("fftconv_stream_stage_size: needs a partial plan"); return FFTCONV_ERR_UNSUPPORTED; }
  *bytes = 2 * slot_bytes(p, H, B, gated != 0, nullptr) + 1024;
  return FFTCONV_OK;
}

extern "C" fftconv_status_t fftconv_fwd_stream(fftconv_plan_t p, const void* h_u, const void* h_w, const void* h_v,
                                               const void* d_kf, void* h_y, int64_t B, int64_t H, int64_t N_total,
                                               void* d_stage, size_t stage_bytes, fftconv_stream_t stream) {
  const char* fn = "fftconv_fwd_stream";
  if (!p) { set_last_error("fftconv_fwd_stream: plan is NULL"); return FFTCONV_ERR_INVALID_ARG; }
  if (p->regime != REGIME_PARTIAL) { set_last_error("fftconv_fwd_stream: needs a partial plan (fft_size < 2N)"); return FFTCONV_ERR_UNSUPPORTED; }
  const bool gated = h_w != nullptr || h_v != nullptr;
  if (gated && !(h_w && h_v)) { set_last_error("fftconv_fwd_stream: gated needs both w and v"); return FFTCONV_ERR_INVALID_ARG; }
  if (B < 0 || H < 0 || N_total < 0) { set_last_error("fftconv_fwd_stream: bad sizes"); return FFTCONV_ERR_INVALID_ARG; }
  if (B * H * N_total == 0) return FFTCONV_OK;
  if (!h_u || !h_y || !d_kf || !d_stage) { set_last_error("fftconv_fwd_stream: NULL pointer"); return FFTCONV_ERR_INVALID_ARG; }
  if (!aligned16(d_stage)) { set_last_error("fftconv_fwd_stream: stage not 16-byte aligned"); return FFTCONV_ERR_MISALIGNED; }
  size_t ws_bytes = 0;
  const size_t slot = slot_bytes(p, H, B, gated, &ws_bytes);
  if (stage_bytes < 2 * slot) { set_last_error("fftconv_fwd_stream: staging buffer too small"); return FFTCONV_ERR_INVALID_ARG; }
  {
    fftconv_status_t chk = check_signal_args(p, fn, B, H, {d_stage, d_kf});
    if (chk != FFTCONV_OK) return chk;
  }
  HostPipe* hp = nullptr;
  cudaError_t e = host_pipe(&hp);
  if (e != cudaSuccess) return cuda_fail(fn, e);
  std::lock_guard<std::mutex> pipe_lock(hp->mu);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if ((e = cudaEventRecord(hp->start, cs)) != cudaSuccess) return cuda_fail(fn, e);
  if ((e = cudaStreamWaitEvent(hp->in, hp->start, 0)) != cudaSuccess) return cuda_fail(fn, e);
  if ((e = cudaStreamWaitEvent(hp->out, hp->start, 0)) != cudaSuccess) return cuda_fail(fn, e);
  const int64_t Nseg = p->N, C = p->L / 2, S = Nseg - C, rows = B * H;
  const size_t es = elem_bytes(p);
  const size_t t = (size_t(rows) * size_t(Nseg) * es + 1023) / 1024 * 1024;
  uint8_t* base = static_cast<uint8_t*>(d_stage);
  const int64_t nseg = (N_total + S - 1) / S;
  for (int64_t i = 0; i < nseg; ++i) {
    const int sl_i = int(i & 1);
    uint8_t* sl = base + size_t(sl_i) * slot;
    uint8_t *du = sl, *dw = sl + t, *dv = sl + 2 * t, *dy = sl + (gated ? 3 : 1) * t, *dws = sl + (gated ? 4 : 2) * t;
    const int64_t s0 = i * S;              // first output position of the segment
    const int64_t a = s0 - C;              // first input position in the buffer
    const int64_t lo = a < 0 ? 0 : a;      // first valid input position
    const int64_t hi = s0 + S < N_total ? s0 + S : N_total;  // end of valid input
    const int64_t off = lo - a;            // its column in the buffer
    const int64_t ncols = hi - lo;
    if (i >= 2 && (e = cudaStreamWaitEvent(hp->in, hp->freed[sl_i], 0)) != cudaSuccess) return cuda_fail(fn, e);
    const void* src[3] = {h_u, h_w, h_v};
    uint8_t* dst[3] = {du, dw, dv};
    for (int q = 0; q < (gated ? 3 : 1); ++q) {
      // zero the columns this segment does not fill (history before 0, tail past the end)
      if (off > 0 || off + ncols < Nseg) {
        if ((e = cudaMemsetAsync(dst[q], 0, size_t(rows) * size_t(Nseg) * es, hp->in)) != cudaSuccess)
          return cuda_fail(fn, e);
      }
      if ((e = cudaMemcpy2DAsync(dst[q] + size_t(off) * es, size_t(Nseg) * es,
                                 static_cast<const uint8_t*>(src[q]) + size_t(lo) * es, size_t(N_total) * es,
                                 size_t(ncols) * es, size_t(rows), cudaMemcpyHostToDevice, hp->in)) != cudaSuccess)
        return cuda_fail(fn, e);
    }
    if ((e = cudaEventRecord(hp->loaded[sl_i], hp->in)) != cudaSuccess) return cuda_fail(fn, e);
    if ((e = cudaStreamWaitEvent(cs, hp->loaded[sl_i], 0)) != cudaSuccess) return cuda_fail(fn, e);
    fftconv_status_t st = run_fwd(p, du, gated ? dw : nullptr, gated ? dv : nullptr, d_kf, dy, B, H,
                                  ws_bytes ? dws : nullptr, stream, fn);
    if (st != FFTCONV_OK) return drain_pipe(hp, cs, st);
    if ((e = cudaEventRecord(hp->computed[sl_i], cs)) != cudaSuccess) return cuda_fail(fn, e);
    if ((e = cudaStreamWaitEvent(hp->out, hp->computed[sl_i], 0)) != cudaSuccess) return cuda_fail(fn, e);
    // outputs s0 .. min(s0 + S, N_total) live at buffer columns C ..
    const int64_t nout = (s0 + S < N_total ? s0 + S : N_total) - s0;
    if ((e = cudaMemcpy2DAsync(static_cast<uint8_t*>(h_y) + size_t(s0) * es, size_t(N_total) * es,
                               dy + size_t(C) * es, size_t(Nseg) * es, size_t(nout) * es, size_t(rows),
                               cudaMemcpyDeviceToHost, hp->out)) != cudaSuccess)
      return cuda_fail(fn, e);
    if ((e = cudaEventRecord(hp->freed[sl_i], hp->out)) != cudaSuccess) return cuda_fail(fn, e);
  }
  if ((e = cudaEventRecord(hp->done, hp->out)) != cudaSuccess) return cuda_fail(fn, e);
  if ((e = cudaStreamWaitEvent(cs, hp->done, 0)) != cudaSuccess) return cuda_fail(fn, e);
  return FFTCONV_OK;
}

// Workspace layout of the backward pass (bytes):
//  fused     : [partials: H * nbt * L complex fp32]
//  multipass : [T_g][T_dc] (fp16 rows, 2 * ceil(B/2) * H * L each)
//              [partials: H * L0 * nbt' * Lp complex fp32][scratch: H * L complex fp32]
static size_t bwd_ws_bytes(const fftconv_plan_s* p, int64_t B, int64_t H) {
  if (p->regime == REGIME_MULTIPASS || p->regime == REGIME_PARTIAL) {
    const int64_t Bv = p->regime == REGIME_PARTIAL ? B * (p->N / (p->L / 2)) : B;
    const int64_t rows = 2 * ((Bv + 1) / 2);
    const size_t t = size_t(rows) * size_t(H) * size_t(p->L) * t_elem_bytes(p);
    const int64_t units = p->dtype == FFTCONV_F32 ? bwd_f32_units_per_head(rows) : bwd_tiles_per_head(rows, p->L1);
    const size_t part = size_t(H) * p->L0 * size_t(units) * size_t(p->Lp) * 8;
    // order-3 plans: the multipass-layout copy of k_f at the end
    const size_t kf_copy = p->dit > 1 ? size_t(H) * p->kf_bytes_per_head : 0;
    return (p->nlev > 1 ? 4 : 2) * t + part + size_t(H) * size_t(p->L) * 8 + kf_copy;
  }
  const int64_t units = p->dtype == FFTCONV_F32 ? bwd_f32_units_per_head(B) : bwd_tiles_per_head(B, p->L1);
  return size_t(H) * size_t(units) * size_t(p->L) * 8;
}

static fftconv_status_t run_bwd(fftconv_plan_t p, const void* d_dy, const void* d_u, const void* d_w,
                                const void* d_v, const void* d_kf, void* d_du, void* d_dw, void* d_dv,
                                float* d_dk, float* d_dkb, int64_t B, int64_t H, int64_t K, void* d_workspace,
                                fftconv_stream_t stream, bool bidir) {
  const char* fn = bidir ? "fftconv_bwd_bidir" : "fftconv_bwd";
  const bool gated = d_w != nullptr || d_v != nullptr;
  if (gated && !(d_w && d_v && d_dw && d_dv)) {
    set_last_error("fftconv_bwd: gated backward needs w, v, dw and dv");
    return FFTCONV_ERR_INVALID_ARG;
  }
  fftconv_status_t chk = gated ? check_signal_args(p, fn, B, H, {d_dy, d_u, d_w, d_v, d_kf, d_du, d_dw, d_dv, d_workspace})
                               : check_signal_args(p, fn, B, H, {d_dy, d_u, d_kf, d_du, d_workspace});
  if (chk != FFTCONV_OK) return chk;
  const int64_t kmax = p->causal ? p->L / 2 : p->L;
  if (K < 1 || K > kmax) { set_last_error("fftconv_bwd: K out of range"); return FFTCONV_ERR_KERNEL_TOO_LONG; }
  if (!d_dk && H > 0) { set_last_error("fftconv_bwd: dk is NULL"); return FFTCONV_ERR_INVALID_ARG; }
  if (bidir) {
    if (!d_dkb && H > 0) { set_last_error("fftconv_bwd_bidir: dk_bwd is NULL"); return FFTCONV_ERR_INVALID_ARG; }
    if (!p->causal || p->regime == REGIME_PARTIAL || p->L != 2 * p->N || p->sparse) {
      set_last_error("fftconv_bwd_bidir: needs a dense full causal plan (fft_size == 2N)");
      return FFTCONV_ERR_UNSUPPORTED;
    }
  }
  if (H == 0) return FFTCONV_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (B == 0) {
    cudaError_t e = cudaMemsetAsync(d_dk, 0, size_t(H) * size_t(K) * sizeof(float), st);
    if (e == cudaSuccess && d_dkb) e = cudaMemsetAsync(d_dkb, 0, size_t(H) * size_t(K) * sizeof(float), st);
    return e == cudaSuccess ? FFTCONV_OK : cuda_fail(fn, e);
  }
  const uint8_t* tab = static_cast<const uint8_t*>(p->d_tables);
  DkParams dk{};
  dk.dk = d_dk;
  dk.dkb = d_dkb;
  dk.shift2 = 2 * p->headroom_shift;  // G and DC both carry 2^-shift
  dk.mask = p->sparse ? reinterpret_cast<const float*>(tab + p->tl.total) : nullptr;
  dk.twiddle = reinterpret_cast<const float2*>(tab + p->tl.wl);
  dk.H = H;
  dk.K = K;
  cudaError_t e;
  if (p->regime == REGIME_FUSED) {
    BwdParams b{};
    b.u = d_u; b.w = d_w; b.v = d_v; b.dy = d_dy; b.du = d_du; b.dw = d_dw; b.dv = d_dv;
    b.kf = d_kf; b.tables = p->d_tables; b.acc = d_workspace;
    b.B = B; b.H = H; b.N = p->N; b.L1 = p->L1; b.causal = p->causal;
    b.gate_io = gated ? 1 : 0; b.need_c = gated ? 1 : 0;
    b.dtype = p->dtype == FFTCONV_BF16 ? 1 : 0;
    b.num_sms = num_sms_current();
    const bool f32 = p->dtype == FFTCONV_F32;
    e = f32 ? launch_bwd_f32(b, tab + p->tl.wl, st) : launch_bwd_fused(b, st);
    if (e != cudaSuccess) return cuda_fail(fn, e);
    dk.part = static_cast<const float2*>(d_workspace);
    dk.nbt = f32 ? bwd_f32_units_per_head(B) : bwd_tiles_per_head(B, p->L1);
    dk.L0 = 1;
    dk.Lp = int32_t(p->L);
    e = launch_dk_finalize(dk, st);
    if (e != cudaSuccess) return cuda_fail(fn, e);
    g_launches += 2;
    return FFTCONV_OK;
  }
  if (p->regime != REGIME_MULTIPASS && p->regime != REGIME_PARTIAL) {
    set_last_error("fftconv_bwd: regime not supported by this build");
    return FFTCONV_ERR_UNSUPPORTED;
  }
  // Partial (overlap-save, A12): the rows are the virtual windows b * NC + j.
  // c (for dv) is the second half of each window's circular result as in the
  // forward; dc windows hold only their second half (block j), so the
  // window's correlation with k is block j's contribution to dg over both
  // halves (overlap-add in pass 3) and Sum_windows DC conj(G) is exactly
  // Sum_i dc[i] g[i - t] for t < K <= C (dk).
  if (p->dit > 1) {  // order-3 k_f -> the multipass layout, in the workspace's tail
    uint8_t* kf2 = static_cast<uint8_t*>(d_workspace) + bwd_ws_bytes(p, B, H) - size_t(H) * p->kf_bytes_per_head;
    e = launch_kf_dit_to_dif(d_kf, kf2, H, p->dit, st);
    if (e != cudaSuccess) return cuda_fail(fn, e);
    g_launches += 1;
    d_kf = kf2;
  }
  const bool partial = p->regime == REGIME_PARTIAL;
  const int64_t NCw = partial ? p->N / (p->L / 2) : 1;
  const int64_t Bv = B * NCw;
  const int64_t rows = 2 * ((Bv + 1) / 2);
  const int nlev = p->nlev;
  uint8_t* ws = static_cast<uint8_t*>(d_workspace);
  const bool f32 = p->dtype == FFTCONV_F32;
  if (f32 && nlev > 1) { set_last_error("fftconv_bwd: the fp32 validation build supports fft_size <= 32768"); return FFTCONV_ERR_UNSUPPORTED; }
  const size_t tbytes = size_t(rows) * size_t(H) * size_t(p->L) * t_elem_bytes(p);
  // T buffers of g and dc; recursive plans ping-pong between two of each
  void* Tg[2] = {ws, ws + (nlev > 1 ? 2 : 1) * tbytes};
  void* Tdc[2] = {ws + tbytes, ws + 3 * tbytes};
  if (nlev == 1) { Tg[1] = Tg[0]; Tdc[1] = Tdc[0]; }
  void* part = ws + (nlev > 1 ? 4 : 2) * tbytes;
  const int64_t nbt_in = f32 ? bwd_f32_units_per_head(rows) : bwd_tiles_per_head(rows, p->L1);
  void* scratch = static_cast<uint8_t*>(part) + size_t(H) * p->L0 * size_t(nbt_in) * size_t(p->Lp) * 8;
  MpParams mp{};
  mp.shift = p->headroom_shift;  // fp16 headroom pre-scale (top-level passes only)
  mp.wbase = reinterpret_cast<const float2*>(tab + p->tl.wbase);
  mp.wtab = reinterpret_cast<const float2*>(tab + p->tl.wtab);
  mp.B = Bv; mp.H = H; mp.N = p->N; mp.L0 = p->lev_L0[0]; mp.Lp = int32_t(p->L / p->lev_L0[0]);
  mp.dtype = p->dtype == FFTCONV_BF16 ? 1 : f32 ? 2 : 0;
  mp.Llev = p->L;
  mp.circ = p->causal ? 0 : 1;
  if (nlev > 1) mp.wtab = nullptr;  // outer twiddles on the fly, as in the forward
  if (partial) { mp.partial = 1; mp.C = p->L / 2; mp.NC = NCw; }
  // deeper outer levels (recursive plans): complex circular fp16 rows
  auto level = [&](int l, void* const* T) {
    MpParams q{};
    int64_t Hl = H, Ll = p->L;
    for (int j = 0; j < l; ++j) { Hl *= p->lev_L0[j]; Ll /= p->lev_L0[j]; }
    q.B = rows; q.H = Hl; q.N = Ll; q.L0 = p->lev_L0[l]; q.Lp = int32_t(Ll / p->lev_L0[l]);
    q.Llev = Ll; q.circ = 1; q.dtype = 0; q.gated = 0;
    q.u = T[(l - 1) & 1]; q.ws = T[l & 1]; q.y = T[(l - 1) & 1];
    return q;
  };
  int launches = 0;
  // pass 1 on g = u (* w) and on dc = dy (* v), then the deeper levels
  mp.u = d_u; mp.w = d_w; mp.gated = gated ? 1 : 0; mp.ws = Tg[0];
  e = launch_mp_pass(mp, 1, st);
  if (e != cudaSuccess) return cuda_fail(fn, e);
  mp.u = d_dy; mp.w = d_v; mp.ws = Tdc[0]; mp.win_hi_only = partial ? 1 : 0;
  e = launch_mp_pass(mp, 1, st);
  if (e != cudaSuccess) return cuda_fail(fn, e);
  mp.win_hi_only = 0;
  launches += 2;
  for (int l = 1; l < nlev; ++l) {
    if ((e = launch_mp_pass(level(l, Tg), 1, st)) != cudaSuccess) return cuda_fail(fn, e);
    if ((e = launch_mp_pass(level(l, Tdc), 1, st)) != cudaSuccess) return cuda_fail(fn, e);
    launches += 2;
  }
  // inner backward on the complex rows (circular), in place
  void* Tgi = Tg[(nlev - 1) & 1];
  void* Tdci = Tdc[(nlev - 1) & 1];
  BwdParams b{};
  b.u = Tgi; b.dy = Tdci; b.dv = Tgi; b.du = Tdci;
  b.kf = d_kf; b.tables = p->d_tables; b.acc = part;
  b.B = rows; b.H = H * p->L0; b.N = p->Lp; b.L1 = p->L1; b.causal = 0;
  b.gate_io = 0; b.need_c = gated ? 1 : 0; b.dtype = f32 ? 2 : 0;
  b.num_sms = num_sms_current();
  e = f32 ? launch_bwd_f32(b, tab + p->tl.wl, st) : launch_bwd_fused(b, st);
  if (e != cudaSuccess) return cuda_fail(fn, e);
  launches += 1;
  // deeper levels back (c only when gated: dv needs it)
  for (int l = nlev - 1; l >= 1; --l) {
    if (gated && (e = launch_mp_pass(level(l, Tg), 3, st)) != cudaSuccess) return cuda_fail(fn, e);
    if ((e = launch_mp_pass(level(l, Tdc), 3, st)) != cudaSuccess) return cuda_fail(fn, e);
    launches += gated ? 2 : 1;
  }
  // pass 3: dv = dy * c ; du = dg * w (or dg), dw = dg * u
  if (gated) {
    mp.ws = Tg[0]; mp.gated = 1; mp.v = d_dy; mp.y = d_dv; mp.v2 = nullptr; mp.y2 = nullptr;
    e = launch_mp_pass(mp, 3, st);
    if (e != cudaSuccess) return cuda_fail(fn, e);
    mp.ws = Tdc[0]; mp.v = d_w; mp.y = d_du; mp.v2 = d_u; mp.y2 = d_dw;
    launches += 1;
  } else {
    mp.ws = Tdc[0]; mp.gated = 0; mp.v = nullptr; mp.y = d_du; mp.v2 = nullptr; mp.y2 = nullptr;
  }
  mp.ola = partial ? 1 : 0;  // partial: dg = overlap-add of neighbouring windows
  e = launch_mp_pass(mp, 3, st);
  if (e != cudaSuccess) return cuda_fail(fn, e);
  launches += 1;
  dk.part = static_cast<const float2*>(part);
  dk.scratch = static_cast<float2*>(scratch);
  dk.wbase = nlev > 1 ? nullptr : mp.wbase;
  dk.nbt = nbt_in;
  dk.L0 = p->L0;
  dk.Lp = p->Lp;
  dk.lev_L0 = p->lev_L0;
  dk.nlev = nlev;
  for (int l = 0; l < 4; ++l) dk.lev[l] = p->lev_L0[l];
  dk.Lfull = p->L;
  e = launch_dk_finalize(dk, st);
  if (e != cudaSuccess) return cuda_fail(fn, e);
  g_launches += launches + 1 + nlev;
  return FFTCONV_OK;
}

extern "C" fftconv_status_t fftconv_bwd(fftconv_plan_t p, const void* d_dy, const void* d_u, const void* d_w,
                                        const void* d_v, const void* d_kf, void* d_du, void* d_dw, void* d_dv,
                                        float* d_dk, int64_t B, int64_t H, int64_t K, void* d_workspace,
                                        fftconv_stream_t stream) {
  return run_bwd(p, d_dy, d_u, d_w, d_v, d_kf, d_du, d_dw, d_dv, d_dk, nullptr, B, H, K, d_workspace, stream, false);
}

extern "C" fftconv_status_t fftconv_bwd_bidir(fftconv_plan_t p, const void* d_dy, const void* d_u, const void* d_w,
                                              const void* d_v, const void* d_kf, void* d_du, void* d_dw, void* d_dv,
                                              float* d_dk_fwd, float* d_dk_bwd, int64_t B, int64_t H, int64_t K,
                                              void* d_workspace, fftconv_stream_t stream) {
  return run_bwd(p, d_dy, d_u, d_w, d_v, d_kf, d_du, d_dw, d_dv, d_dk_fwd, d_dk_bwd, B, H, K, d_workspace, stream,
                 true);
}

extern "C" fftconv_status_t fftconv_workspace_size(fftconv_plan_t p, int64_t B, int64_t H, int for_bwd, size_t* bytes) {
  if (!p || !bytes || B < 0 || H < 0) { set_last_error("fftconv_workspace_size: bad argument"); return FFTCONV_ERR_INVALID_ARG; }
  size_t n = 0;
  if (for_bwd) n = bwd_ws_bytes(p, B, H);
  else if (p->regime == REGIME_MULTIPASS && p->dit == 1)  // (order-3 plans need none)
    n = size_t(p->nlev > 1 ? 2 : 1) * size_t(2 * ((B + 1) / 2)) * size_t(H) * size_t(p->L) * t_elem_bytes(p);
  else if (p->regime == REGIME_PARTIAL) {
    const int64_t Bv = B * (p->N / (p->L / 2));
    n = size_t(2 * ((Bv + 1) / 2)) * size_t(H) * size_t(p->L) * t_elem_bytes(p);
  }
  *bytes = n;
  return FFTCONV_OK;
}

extern "C" int64_t fftconv_launch_count_reset(void) {
  int64_t n = g_launches;
  g_launches = 0;
  return n;
}
