/*
 * fftconv.h -- C ABI of the B200-native FlashFFTConv hot path
 * (arXiv 2311.05908, "FlashFFTConv: Efficient Convolutions for Long Sequences
 * with Tensor Cores").
 *
 * Citations: "P:n" = line n of the paper source; "A<n>" = reading
 * n listed in DESIGN.md ("Readings of the paper").
 *
 * The operation (Alg. 1):
 *     y = iFFT( FFT(pad(u)) * k_f )[:N],   k_f = FFT(pad(k))
 * over u of shape (B, H, N) with one real filter k[h, :K] per head h,
 * plus the gated form y = v * ((u * w) conv k) (A17), the
 * partial form K < N (A12), the frequency-sparse form
 * (k_f masked; A13) and the backward pass
 * (recomputation; A15).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All device pointers are CUDA device addresses owned by the caller.  The
 *    library NEVER allocates device memory; sizes come from fftconv_plan_info.
 *  - Signals u, w, v, y, dy, du, dw, dv: contiguous row-major (B, H, N) in the
 *    plan's dtype, 16-byte aligned.  Row (b, h) starts at ((b*H)+h)*N.
 *  - Filters k and gradients dk: contiguous row-major (H, K) fp32.
 *  - k_f: opaque, plan layout, produced only by fftconv_precompute_kf for the
 *    same plan; kf_bytes_per_head bytes per head.
 *  - Calls are asynchronous on `stream`; inputs are never written; outputs
 *    must not alias inputs.  Argument errors are detected before any launch
 *    and leave the outputs untouched.  Launch failures return
 *    FFTCONV_ERR_CUDA; asynchronous device faults surface at the caller's
 *    next synchronisation.  fftconv_last_error() describes the last failure
 *    of the calling thread.
 *  - No atomics: results are bitwise reproducible run to run and do not
 *    depend on how rows are sharded across GPUs.
 *  - A plan is host memory, immutable after fftconv_plan_upload and safe to
 *    share across threads and streams.
 */
#ifndef FFTCONV_H_
#define FFTCONV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t-compatible handle (NULL = legacy default stream). */
typedef struct CUstream_st* fftconv_stream_t;

typedef struct fftconv_plan_s* fftconv_plan_t;

/* I/O element type.  Tensor-core operands are always fp16 with fp32
 * accumulation (A16; bf16 operands would miss the 2e-3 bound).
 * FFTCONV_F32 is the validation build (north star, BASELINE.json: "<= 1e-5
 * relative L2 on an fp32 validation build"): fp32 I/O and the same plan,
 * packing, Monarch decomposition and multipass passes with every stage in
 * fp32 on the CUDA cores (no tensor cores; not a performance path).  It
 * covers the forward and backward calls for fft_size <= 32768. */
typedef enum { FFTCONV_F16 = 0, FFTCONV_BF16 = 1, FFTCONV_F32 = 2 } fftconv_dtype_t;

typedef enum {
  FFTCONV_OK = 0,
  FFTCONV_ERR_INVALID_ARG = 1,     /* null/negative/inconsistent argument       */
  FFTCONV_ERR_NOT_POW2 = 2,        /* N or fft_size not a power of two */
  FFTCONV_ERR_KERNEL_TOO_LONG = 3, /* K exceeds the causal budget fft_size/2    */
  FFTCONV_ERR_BAD_SPARSITY = 4,    /* sparsity dims/masks inconsistent          */
  FFTCONV_ERR_UNSUPPORTED = 5,     /* valid request this build cannot run yet   */
  FFTCONV_ERR_MISALIGNED = 6,      /* device pointer not 16-byte aligned        */
  FFTCONV_ERR_CUDA = 7             /* CUDA launch/runtime error                 */
} fftconv_status_t;

/* Frequency-sparsity pattern (A13).  The length-L spectrum of k
 * (L = fft_size) is viewed as a row-major digit grid dims[0] x ... x
 * dims[ndims-1] (slowest first, product = L).  keep[j][i] != 0 keeps index i
 * of dimension j; frequency f is kept iff every digit is kept.  The mask is
 * applied Hermitian-symmetrically, m[f] = keep(f) | keep(L - f), so y stays
 * real.  The tab:sparsity_fraction patterns (a,b,c,d) zero the last a,b,c,d
 * entries of each dimension.  Pointers are read during fftconv_plan only. */
typedef struct {
  int32_t ndims;          /* 1..4 */
  int32_t dims[4];
  const uint8_t* keep[4]; /* host arrays of dims[j] bytes */
} fftconv_sparsity_t;

#define FFTCONV_MAX_ORDER 6

typedef struct {
  int64_t N;                 /* input/output length per row                   */
  int64_t fft_size;          /* L                                             */
  int32_t causal;            /* 1 causal (zero-padded), 0 circular            */
  int32_t dtype;             /* fftconv_dtype_t                               */
  int32_t regime;            /* 1 fused single pass (order 2 for fft_size
                                <= 2048; causal fft_size 4096 / 8192 / 16384
                                as order 3, the outer L0-point DFT inside the
                                fused kernel, when the B200 cost model
                                predicts it faster -- env FFTCONV_DIT=0 / 1
                                forbids / forces it), 2 partial (chunked),
                                3 multipass (outer L0-point passes + fused
                                inner transform, Alg. 4)                     */
  int32_t order;             /* number of transform levels: order-2 Monarch
                                (L1, L2) plus one per outer multipass level
                                (Alg. 4), order <= FFTCONV_MAX_ORDER         */
  int32_t factors[6];        /* L = prod factors[0..order), slowest level
                                first (outer levels, then L1, L2)            */
  int32_t rows_per_tile;     /* batch rows one CTA work unit processes        */
  int64_t max_kernel_len;    /* largest K accepted by precompute_kf           */
  size_t table_bytes;        /* device bytes for fftconv_plan_upload          */
  size_t kf_bytes_per_head;  /* device bytes of k_f per head                  */
  size_t workspace_bytes_per_head; /* fftconv_bwd workspace, per head         */
  double mask_fraction;      /* fraction of spectrum zeroed by the mask       */
  double skip_fraction;      /* fraction of pointwise blocks the kernel skips */
} fftconv_plan_info_t;

/* Create a plan (host only, no CUDA calls).
 *  N        input length per row, power of two, 256 <= N.
 *  fft_size L, power of two.  causal=1: L == 2N is the full causal conv
 *           (K <= N; N up to 4M); L < 2N selects the partial (overlap-save)
 *           conv with K <= L/2, L <= 32768 (A12).  causal=0:
 *           circular, L == N == K, N = 512 .. 8M (A2).
 *  dtype    FFTCONV_F16 / FFTCONV_BF16 I/O (fp16 tensor-core operands, fp32
 *           accumulation), or FFTCONV_F32 (validation build, L <= 32768).
 *  sparsity NULL for dense; else see fftconv_sparsity_t (prod dims == L).
 * Returns NOT_POW2 / INVALID_ARG / BAD_SPARSITY / UNSUPPORTED on bad input;
 * *out is set only on success. */
fftconv_status_t fftconv_plan(fftconv_plan_t* out, int64_t N, int64_t fft_size, fftconv_dtype_t dtype,
                              int causal, const fftconv_sparsity_t* sparsity);

/* Fill *info (host only). */
fftconv_status_t fftconv_plan_info(fftconv_plan_t plan, fftconv_plan_info_t* info);

/* Copy the plan's constant tables (real-pair DFT matrices of the Monarch
 * factors P:126, twiddles, all built in fp64 on the host) into the
 * caller-owned device buffer d_tables (table_bytes, 1024-byte aligned) and
 * bind it to the plan.  Must precede every other device call.  The buffer
 * must outlive the plan's use. */
fftconv_status_t fftconv_plan_upload(fftconv_plan_t plan, void* d_tables, fftconv_stream_t stream);

/* k_f = FFT_L(pad(k[h, :K])) in plan layout, computed on the
 * GPU in fp32, with the sparsity mask applied.  d_k: (H, K) fp32;
 * d_kf: H * kf_bytes_per_head bytes.  K must be 1..max_kernel_len. */
fftconv_status_t fftconv_precompute_kf(fftconv_plan_t plan, const float* d_k, int64_t H, int64_t K, void* d_kf,
                                       fftconv_stream_t stream);

/* Bidirectional (two-sided) filters (the M2-BERT-style
 * long convolution; the paper names M2-BERT, but prints no
 * formula, so DESIGN.md reading B1 fixes it):
 *     c[i] = sum_{j<=i} g[j] k_fwd[h, i-j] + sum_{j>=i} g[j] k_bwd[h, j-i]
 * (lag 0 carries k_fwd[0] + k_bwd[0]).  With fft_size L = 2N and K <= N the
 * two-sided filter k_fwd[t] + k_bwd[L - t] (t > L - K) is exactly the
 * circular filter whose first N outputs are c, so k_f of it feeds the
 * unchanged fftconv_fwd / fftconv_gated_fwd / fftconv_fwd_host calls.
 * d_k_fwd, d_k_bwd: (H, K) fp32 device; d_kf: H * kf_bytes_per_head bytes.
 * FFTCONV_ERR_UNSUPPORTED unless the plan is dense, causal and full
 * (fft_size == 2N; partial and circular plans have no anti-causal room);
 * other errors as fftconv_precompute_kf. */
fftconv_status_t fftconv_precompute_kf_bidir(fftconv_plan_t plan, const float* d_k_fwd, const float* d_k_bwd,
                                             int64_t H, int64_t K, void* d_kf, fftconv_stream_t stream);

/* Device workspace the forward (for_bwd = 0) or backward (for_bwd = 1) call
 * needs for a (B, H) problem.  The fused regime's forward needs none; the
 * multipass and partial regimes (Alg. 4) keep their fp16
 * intermediate there (2 * ceil(B'/2) * H * fft_size * 2 bytes, B' = B or the
 * number of overlap-save windows; twice that for recursive plans and for the
 * fp32 build); the backward adds the per-tile partial spectra of dk. */
fftconv_status_t fftconv_workspace_size(fftconv_plan_t plan, int64_t B, int64_t H, int for_bwd, size_t* bytes);

/* y = u conv k (Alg. 1; real packing, causal padding and the
 * pointwise k_f product fused).  d_workspace: at least
 * fftconv_workspace_size(plan, B, H, 0) bytes, 16-byte aligned (NULL allowed
 * when that size is 0). */
fftconv_status_t fftconv_fwd(fftconv_plan_t plan, const void* d_u, const void* d_kf, void* d_y, int64_t B,
                             int64_t H, void* d_workspace, fftconv_stream_t stream);

/* y = v * ((u * w) conv k), gating fused into load and store. */
fftconv_status_t fftconv_gated_fwd(fftconv_plan_t plan, const void* d_u, const void* d_w, const void* d_v,
                                   const void* d_kf, void* d_y, int64_t B, int64_t H, void* d_workspace,
                                   fftconv_stream_t stream);

/* End-to-end forward from HOST buffers (plain when h_w == h_v == NULL,
 * gated otherwise).  h_u, h_w, h_v, h_y: (B, H, N) row-major in the plan
 * dtype, preferably pinned (pageable memory makes the copies synchronous).
 * The B batch rows are streamed through the caller-owned device staging
 * buffer d_stage in chunks of rows_per_chunk (rounded up to even, so rows
 * keep their packing partner and the result is bitwise that of the device
 * call; two slots): the host->device
 * copy of chunk i+1, the convolution of chunk i and the device->host copy of
 * chunk i-1 run concurrently on library streams (copy engines beside the
 * SMs).  d_kf: device k_f from fftconv_precompute_kf.  Ordered after earlier
 * work on `stream`; work queued on `stream` after this call sees h_y
 * complete.  stage_bytes >= fftconv_host_stage_size(plan, H, rows_per_chunk,
 * gated).  Errors as fftconv_fwd; FFTCONV_ERR_INVALID_ARG for a short stage.
 * Argument errors are reported before any copy is enqueued; a failure after
 * that still orders `stream` after the copies already queued.  Concurrent
 * calls from several host threads on one device are safe: the library's copy
 * streams and events are per device, and each call holds that device's pipe
 * lock while it enqueues (the calls' copies then run one after another). */
fftconv_status_t fftconv_fwd_host(fftconv_plan_t plan, const void* h_u, const void* h_w, const void* h_v,
                                  const void* d_kf, void* h_y, int64_t B, int64_t H, int64_t rows_per_chunk,
                                  void* d_stage, size_t stage_bytes, fftconv_stream_t stream);
fftconv_status_t fftconv_host_stage_size(fftconv_plan_t plan, int64_t H, int64_t rows_per_chunk, int gated,
                                         size_t* bytes);

/* Sequence streaming for rows longer than device buffers (NEXT-4; partial
 * plans only, K <= C = fft_size/2, plan N = segment length, a multiple of C):
 * (B, H, N_total) host rows are convolved segment by segment.  Segment i
 * produces outputs [i S, (i+1) S), S = N - C, from a device buffer holding
 * u[i S - C, i S + S) (zeros outside the row), so the overlap-save windows see
 * the C samples of history they need; copies of neighbouring segments overlap
 * the convolution as in fftconv_fwd_host.  h_w, h_v NULL = plain.  Result
 * equals the partial convolution of the full rows.  stage_bytes >=
 * fftconv_stream_stage_size(plan, B, H, gated).  FFTCONV_ERR_UNSUPPORTED for
 * non-partial plans.  Thread safety and error ordering as fftconv_fwd_host. */
fftconv_status_t fftconv_fwd_stream(fftconv_plan_t plan, const void* h_u, const void* h_w, const void* h_v,
                                    const void* d_kf, void* h_y, int64_t B, int64_t H, int64_t N_total,
                                    void* d_stage, size_t stage_bytes, fftconv_stream_t stream);
fftconv_status_t fftconv_stream_stage_size(fftconv_plan_t plan, int64_t B, int64_t H, int gated, size_t* bytes);

/* Backward of <y, dy> with recomputation (A15) for every plan the
 * forward accepts (fused, multipass incl. recursive, partial, circular,
 * frequency-sparse, fp32 build).  Plain when d_w == d_v == NULL (then d_dw,
 * d_dv ignored); gated when both are given.  d_dk (H, K) fp32 is OVERWRITTEN
 * with the batch sum (deterministic: fixed-order reductions, no atomics).
 * d_workspace: fftconv_workspace_size(plan, B, H, 1) bytes (required). */
fftconv_status_t fftconv_bwd(fftconv_plan_t plan, const void* d_dy, const void* d_u, const void* d_w,
                             const void* d_v, const void* d_kf, void* d_du, void* d_dw, void* d_dv, float* d_dk,
                             int64_t B, int64_t H, int64_t K, void* d_workspace, fftconv_stream_t stream);

/* Backward of the bidirectional convolution (d_kf from
 * fftconv_precompute_kf_bidir): as fftconv_bwd, with dk split into
 * d_dk_fwd[h, t] = sum_b sum_i dc[i] g[i - t] and d_dk_bwd[h, t] =
 * sum_b sum_i dc[i] g[i + t] (both (H, K) fp32, overwritten; lag 0 appears
 * in both).  Same plans as fftconv_precompute_kf_bidir. */
fftconv_status_t fftconv_bwd_bidir(fftconv_plan_t plan, const void* d_dy, const void* d_u, const void* d_w,
                                   const void* d_v, const void* d_kf, void* d_du, void* d_dw, void* d_dv,
                                   float* d_dk_fwd, float* d_dk_bwd, int64_t B, int64_t H, int64_t K,
                                   void* d_workspace, fftconv_stream_t stream);

void fftconv_plan_destroy(fftconv_plan_t plan);

/* Thread-local description of the last error ("" if none). */
const char* fftconv_last_error(void);

/* ---- cost models (host only, no CUDA calls) --------------------------
 * Eq. 2 of the paper, C = BH sum_i [16 N N_i / gamma(N_i) + 4N /
 * omega(i)] for the balanced order-p factorisation of N,
 * gamma / omega per P:276-279 with the working-set rule of SURVEY A11; and
 * the order p (2..4) it selects (ties -> smaller p).  Pinned by the tests to
 * the paper's A100 grouping. */
double fftconv_cost_eq2(int64_t N, int32_t p, double mu, double sigma_h, double sigma_s, double tau_m,
                        double tau_g, double sram_bytes);
int32_t fftconv_select_order(int64_t N, double mu, double sigma_h, double sigma_s, double tau_m, double tau_g,
                             double sram_bytes);
int32_t fftconv_factorize(int64_t n, int32_t p, int64_t* out);
/* B200 tier cost model: the work units of the kernels a
 * plan launches for one call on (B, H) rows -- feat[0..3] fused tiles
 * (order 2 causal, order 2 circular incl. the multipass inner pass, order 3
 * L0 = 2, L0 = 4), feat[4] outer-pass elements (levels x pairs x H x L),
 * feat[5] k_f precompute elements, feat[6] launches, feat[7..9] (bwd != 0)
 * backward tiles, T-chain elements, dk elements, feat[10] the gated share
 * of the fused tiles (their extra w / v traffic), feat[11] the call's
 * algorithmic HBM bytes -- and the predicted seconds
 * sum coef[i] feat[i] (coef NULL: the library's B200 fit). */
#define FFTCONV_COST_NFEAT 12
fftconv_status_t fftconv_cost_features(fftconv_plan_t plan, int64_t B, int64_t H, int bwd, int gated,
                                       double* feat);
fftconv_status_t fftconv_cost_predict(fftconv_plan_t plan, int64_t B, int64_t H, int bwd, int gated, const double* coef,
                                      double* seconds);

/* Number of kernel launches issued by this thread since the last call
 * (instrumentation for the bench's gpu_launches count). */
int64_t fftconv_launch_count_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* FFTCONV_H_ */
