/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * FlashFFTConv hot path (arXiv 2311.05908).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, headers, tables or constants with the CUDA path
 * (paper_2311_05908_b200/), and never includes anything from it.
 *
 * What it computes (citations are PAPER.md line numbers, "P:n"; SURVEY.md
 * section 8(c) readings are "A<n>"):
 *
 *   causal convolution   c[i] = sum_{j<=i} g[j] k[i-j]            P:105 (A1)
 *   circular convolution c[i] = sum_j g[j] k[(i-j) mod N]          P:109 (A2)
 *   computed through the convolution theorem, P:42-47/P:105-110:
 *       c = Re( IFFT_L( FFT_L(pad g) * m * FFT_L(pad k) ) )[:N]
 *   with an iterative radix-2 Cooley-Tukey FFT of length L (bit reversal +
 *   log2 L butterfly passes), twiddles exp(-2 pi i j / L) evaluated directly
 *   in fp64 per j (no recurrences), forward unnormalised, inverse scaled by
 *   1/L exactly once (A8).  Real inputs are treated as complex with zero
 *   imaginary part: NO real packing, NO Monarch decomposition, NO causal skip.
 *
 *   gating   y = v * ((u*w) conv k)                        P:257, P:439 (A17)
 *   partial  k truncated to K < N taps (zero beyond)       P:300-303 (A12)
 *   frequency-sparse  m = 0/1 Hermitian-symmetric mask on the length-L
 *            spectrum of k                                  P:310-314 (A13)
 *   backward (loss <y, dy>), recomputation semantics       P:245-246 (A15):
 *       dc = dy (plain) or dy*v (gated)
 *       dg = IFFT(FFT(pad dc) * conj(m*KF))[:N]    (correlation with k)
 *       du = dg (plain) or dg*w;   dw = dg*u;   dv = dy*c
 *       dk = Re IFFT( conj(m) * sum_b FFT(pad dc_b) * conj(FFT(pad g_b)) )[:K]
 *
 * Plain direct sums (O(N*K)) are also provided; tests pin the FFT path to
 * them, and to a naive O(L^2) DFT, on small inputs.
 *
 * Layout: u, w, v, y, dy, du, dw, dv are row-major (B, H, N) fp64;
 * k, dk are (H, K) fp64; mask is length L fp64 (or NULL = dense).
 * All functions return 0 on success, a negative value on bad arguments.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const double ORC_PI = 3.14159265358979323846264338327950288;

static int is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

/* Naive O(n^2) DFT, the defining sum X[k] = sum_n x[n] W_n^{nk}
 * (Appendix A.1), W_n = exp(-2 pi i / n).  inverse != 0
 * uses W_n^{-nk} and divides by n.  (n*k) is reduced mod n in integers so the
 * angle stays small and exact. */
int orc_naive_dft(const double* xr, const double* xi, int64_t n, int inverse,
                  double* Xr, double* Xi) {
  if (n <= 0) return -1;
  const double sgn = inverse ? 1.0 : -1.0;
  for (int64_t k = 0; k < n; ++k) {
    double sr = 0.0, si = 0.0;
    for (int64_t t = 0; t < n; ++t) {
      int64_t e = (int64_t)(((__int128)t * k) % n);
      double ang = sgn * 2.0 * ORC_PI * (double)e / (double)n;
      double c = cos(ang), s = sin(ang);
      double a = xr[t], b = xi ? xi[t] : 0.0;
      sr += a * c - b * s;
      si += a * s + b * c;
    }
    if (inverse) { sr /= (double)n; si /= (double)n; }
    Xr[k] = sr;
    Xi[k] = si;
  }
  return 0;
}

/* Iterative radix-2 Cooley-Tukey FFT in place on split re/im arrays.
 * Forward: X[k] = sum x[n] exp(-2 pi i nk/L), unnormalised.
 * Inverse: exp(+2 pi i nk/L) and a single 1/L scale at the end (A8). */
int orc_fft(double* re, double* im, int64_t L, int inverse) {
  if (!is_pow2(L)) return -1;
  /* bit-reversal permutation */
  for (int64_t i = 1, j = 0; i < L; ++i) {
    int64_t bit = L >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      double t = re[i]; re[i] = re[j]; re[j] = t;
      t = im[i]; im[i] = im[j]; im[j] = t;
    }
  }
  const double sgn = inverse ? 1.0 : -1.0;
  for (int64_t len = 2; len <= L; len <<= 1) {
    const int64_t half = len >> 1;
    for (int64_t j = 0; j < half; ++j) {
      /* twiddle exp(sgn 2 pi i j / len), evaluated directly (no recurrence) */
      double ang = sgn * 2.0 * ORC_PI * (double)j / (double)len;
      double wr = cos(ang), wi = sin(ang);
      for (int64_t s = 0; s < L; s += len) {
        int64_t a = s + j, b = s + j + half;
        double tr = re[b] * wr - im[b] * wi;
        double ti = re[b] * wi + im[b] * wr;
        re[b] = re[a] - tr; im[b] = im[a] - ti;
        re[a] += tr;        im[a] += ti;
      }
    }
  }
  if (inverse) {
    const double s = 1.0 / (double)L;
    for (int64_t i = 0; i < L; ++i) { re[i] *= s; im[i] *= s; }
  }
  return 0;
}

/* Spectrum of one filter row: KF = FFT_L(pad(k[:K])) (A15). */
static void filter_spectrum(const double* krow, int64_t K, int64_t L,
                            double* kr, double* ki) {
  memset(kr, 0, sizeof(double) * L);
  memset(ki, 0, sizeof(double) * L);
  for (int64_t t = 0; t < K; ++t) kr[t] = krow[t];
  orc_fft(kr, ki, L, 0);
}

static int check_shapes(int64_t B, int64_t H, int64_t N, int64_t K, int64_t L,
                        int causal) {
  if (B < 0 || H < 0 || N < 0 || K < 0) return -1;
  if (!is_pow2(L)) return -2;
  if (causal) {
    if (N + K - 1 > L) return -3;    /* zero padding must avoid wrap */
  } else {
    if (!(N == L && K == L)) return -4; /* circular: N = fft_size = K */
  }
  if (K > N && causal) return -5;
  return 0;
}

/* Forward convolution.  w, v may be NULL (plain conv); mask may be NULL. */
int orc_conv_fwd(const double* u, const double* w, const double* v,
                 const double* k, const double* mask, int64_t B, int64_t H,
                 int64_t N, int64_t K, int64_t L, int causal, double* y) {
  int rc = check_shapes(B, H, N, K, L, causal);
  if (rc) return rc;
  if (B == 0 || H == 0 || N == 0) return 0;
  double* KFr = (double*)malloc(sizeof(double) * L * H);
  double* KFi = (double*)malloc(sizeof(double) * L * H);
  if (!KFr || !KFi) { free(KFr); free(KFi); return -10; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t h = 0; h < H; ++h) {
    filter_spectrum(k + h * K, K, L, KFr + h * L, KFi + h * L);
    if (mask)
      for (int64_t f = 0; f < L; ++f) { KFr[h * L + f] *= mask[f]; KFi[h * L + f] *= mask[f]; }
  }
#pragma omp parallel
  {
    double* zr = (double*)malloc(sizeof(double) * L);
    double* zi = (double*)malloc(sizeof(double) * L);
#pragma omp for schedule(dynamic, 4)
    for (int64_t row = 0; row < B * H; ++row) {
      const int64_t h = row % H;
      const double* ur = u + row * N;
      memset(zr, 0, sizeof(double) * L);
      memset(zi, 0, sizeof(double) * L);
      for (int64_t n = 0; n < N; ++n) zr[n] = w ? ur[n] * w[row * N + n] : ur[n];
      orc_fft(zr, zi, L, 0);
      const double* kr = KFr + h * L;
      const double* ki = KFi + h * L;
      for (int64_t f = 0; f < L; ++f) {
        double a = zr[f], b = zi[f];
        zr[f] = a * kr[f] - b * ki[f];
        zi[f] = a * ki[f] + b * kr[f];
      }
      orc_fft(zr, zi, L, 1);
      for (int64_t n = 0; n < N; ++n) y[row * N + n] = v ? v[row * N + n] * zr[n] : zr[n];
    }
    free(zr);
    free(zi);
  }
  free(KFr);
  free(KFi);
  return 0;
}

/* Backward pass.  w, v, mask may be NULL.  dw, dv may be NULL when w/v are.
 * dk (H x K) is overwritten with the sum over the batch (A15). */
int orc_conv_bwd(const double* dy, const double* u, const double* w,
                 const double* v, const double* k, const double* mask,
                 int64_t B, int64_t H, int64_t N, int64_t K, int64_t L,
                 int causal, double* du, double* dw, double* dv, double* dk) {
  int rc = check_shapes(B, H, N, K, L, causal);
  if (rc) return rc;
  if (H == 0 || K == 0) return 0;
  if (B == 0 || N == 0) { memset(dk, 0, sizeof(double) * H * K); return 0; }
  int rc2 = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t h = 0; h < H; ++h) {
    double* kr = (double*)malloc(sizeof(double) * L);
    double* ki = (double*)malloc(sizeof(double) * L);
    double* gr = (double*)malloc(sizeof(double) * L);
    double* gi = (double*)malloc(sizeof(double) * L);
    double* cr = (double*)malloc(sizeof(double) * L);
    double* ci = (double*)malloc(sizeof(double) * L);
    double* ar = (double*)calloc(L, sizeof(double)); /* sum_b DC conj(G) */
    double* ai = (double*)calloc(L, sizeof(double));
    if (!kr || !ki || !gr || !gi || !cr || !ci || !ar || !ai) {
#pragma omp atomic write
      rc2 = -10;
    } else {
      filter_spectrum(k + h * K, K, L, kr, ki);
      if (mask) for (int64_t f = 0; f < L; ++f) { kr[f] *= mask[f]; ki[f] *= mask[f]; }
      for (int64_t b = 0; b < B; ++b) {
        const int64_t row = b * H + h;
        const double* urow = u + row * N;
        /* recompute g and its spectrum (recomputation) */
        memset(gr, 0, sizeof(double) * L); memset(gi, 0, sizeof(double) * L);
        for (int64_t n = 0; n < N; ++n) gr[n] = w ? urow[n] * w[row * N + n] : urow[n];
        orc_fft(gr, gi, L, 0);
        /* dv = dy * c needs the forward output c */
        if (v && dv) {
          for (int64_t f = 0; f < L; ++f) {
            cr[f] = gr[f] * kr[f] - gi[f] * ki[f];
            ci[f] = gr[f] * ki[f] + gi[f] * kr[f];
          }
          orc_fft(cr, ci, L, 1);
          for (int64_t n = 0; n < N; ++n) dv[row * N + n] = dy[row * N + n] * cr[n];
        }
        /* dc = dy (plain) or dy * v (gated) */
        memset(cr, 0, sizeof(double) * L); memset(ci, 0, sizeof(double) * L);
        for (int64_t n = 0; n < N; ++n) cr[n] = v ? dy[row * N + n] * v[row * N + n] : dy[row * N + n];
        orc_fft(cr, ci, L, 0);
        /* accumulate DC * conj(G) for dk */
        for (int64_t f = 0; f < L; ++f) {
          ar[f] += cr[f] * gr[f] + ci[f] * gi[f];
          ai[f] += ci[f] * gr[f] - cr[f] * gi[f];
        }
        /* dg = IFFT(DC * conj(KF)) */
        for (int64_t f = 0; f < L; ++f) {
          double a = cr[f], bb = ci[f];
          cr[f] = a * kr[f] + bb * ki[f];
          ci[f] = bb * kr[f] - a * ki[f];
        }
        orc_fft(cr, ci, L, 1);
        for (int64_t n = 0; n < N; ++n) {
          const double dg = cr[n];
          du[row * N + n] = w ? dg * w[row * N + n] : dg;
          if (w && dw) dw[row * N + n] = dg * urow[n];
        }
      }
      if (mask) for (int64_t f = 0; f < L; ++f) { ar[f] *= mask[f]; ai[f] *= mask[f]; }
      orc_fft(ar, ai, L, 1);
      for (int64_t t = 0; t < K; ++t) dk[h * K + t] = ar[t];
    }
    free(kr); free(ki); free(gr); free(gi); free(cr); free(ci); free(ar); free(ai);
  }
  return rc2;
}

/* Direct O(N*K) sums -- the plain definitions (A1, A2). */
int orc_direct_conv(const double* g, const double* k, int64_t N, int64_t K,
                    int causal, double* c) {
  if (N < 0 || K < 0) return -1;
  if (!causal && K != N) return -4;
  for (int64_t i = 0; i < N; ++i) {
    double s = 0.0;
    if (causal) {
      int64_t j0 = i - K + 1 > 0 ? i - K + 1 : 0;
      for (int64_t j = j0; j <= i; ++j) s += g[j] * k[i - j];
    } else {
      for (int64_t j = 0; j < N; ++j) s += g[j] * k[((i - j) % N + N) % N];
    }
    c[i] = s;
  }
  return 0;
}

/* One output element of the (gated) causal conv, by direct sum: used to
 * check sampled outputs at full problem sizes. */
double orc_direct_point(const double* urow, const double* wrow,
                        const double* krow, int64_t K, int64_t i) {
  double s = 0.0;
  int64_t j0 = i - K + 1 > 0 ? i - K + 1 : 0;
  for (int64_t j = j0; j <= i; ++j) s += (wrow ? urow[j] * wrow[j] : urow[j]) * krow[i - j];
  return s;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
