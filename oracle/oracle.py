"""Python wrapper of the fp64 CPU oracle (oracle/oracle.c) plus small numpy
helpers.

TEST INFRASTRUCTURE ONLY -- only tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with the CUDA path (``paper_2311_05908_b200``) and
never imports it.

Citations: ``P:n`` = /root/reference/PAPER.md line n; ``A<n>`` = the reading
listed in SURVEY.md section 8(c).3 and DESIGN.md "Readings of the paper".

Parity status of each function is stated in its docstring; every function
here is pinned by a ``-m "not gpu"`` test in tests/test_oracle_*.py except
where "parity unpinned" is written.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> oracle/liboracle.so with gcc (fp64, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
             "-fno-fast-math", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            d = ctypes.POINTER(ctypes.c_double)
            i64 = ctypes.c_int64
            lib.orc_naive_dft.argtypes = [d, d, i64, ctypes.c_int, d, d]
            lib.orc_fft.argtypes = [d, d, i64, ctypes.c_int]
            lib.orc_conv_fwd.argtypes = [d, d, d, d, d, i64, i64, i64, i64, i64,
                                         ctypes.c_int, d]
            lib.orc_conv_bwd.argtypes = [d, d, d, d, d, d, i64, i64, i64, i64, i64,
                                         ctypes.c_int, d, d, d, d]
            lib.orc_direct_conv.argtypes = [d, d, i64, i64, ctypes.c_int, d]
            lib.orc_direct_point.argtypes = [d, d, d, i64, i64]
            lib.orc_direct_point.restype = ctypes.c_double
            lib.orc_num_threads.restype = ctypes.c_int
            lib.orc_set_num_threads.argtypes = [ctypes.c_int]
            for f in (lib.orc_naive_dft, lib.orc_fft, lib.orc_conv_fwd,
                      lib.orc_conv_bwd, lib.orc_direct_conv):
                f.restype = ctypes.c_int
            _lib = lib
    return _lib


def _f64(a):
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} rejected its arguments (code {rc})")


def num_threads() -> int:
    return int(_load().orc_num_threads())


def set_num_threads(n: int) -> None:
    _load().orc_set_num_threads(int(n))


# --------------------------------------------------------------------------
# transforms
# --------------------------------------------------------------------------
def naive_dft(x, inverse: bool = False) -> np.ndarray:
    """O(n^2) defining sum X[k] = sum_n x[n] W_n^{nk}, W_n = e^{-2 pi i/n}
    (Appendix A.1).  inverse=True uses W^{-nk} and 1/n (A8)."""
    x = np.asarray(x, dtype=np.complex128).ravel()
    xr, xi = _f64(x.real), _f64(x.imag)
    n = x.size
    Xr, Xi = np.empty(n), np.empty(n)
    _check(_load().orc_naive_dft(_ptr(xr), _ptr(xi), n, int(inverse), _ptr(Xr), _ptr(Xi)),
           "naive_dft")
    return Xr + 1j * Xi


def fft(x, inverse: bool = False) -> np.ndarray:
    """Iterative radix-2 Cooley-Tukey FFT (forward unnormalised, inverse 1/L
    once; A8).  Length must be a power of two."""
    x = np.asarray(x, dtype=np.complex128).ravel()
    re, im = _f64(x.real).copy(), _f64(x.imag).copy()
    _check(_load().orc_fft(_ptr(re), _ptr(im), x.size, int(inverse)), "fft")
    return re + 1j * im


# --------------------------------------------------------------------------
# convolution
# --------------------------------------------------------------------------
def conv_fwd(u, k, *, fft_size=None, causal=True, w=None, v=None, mask=None):
    """y = [v *] ((u [* w]) conv k) via the convolution theorem (P:42-47,
    P:105-110, gating P:257/P:439, frequency mask P:310-314 / A13).

    u, w, v: (B, H, N); k: (H, K).  causal: fft_size >= N + K - 1 (default
    2N).  circular: fft_size == N == K.  Returns fp64 (B, H, N)."""
    u = _f64(u)
    k = _f64(k)
    B, H, N = u.shape
    H2, K = k.shape
    if H2 != H:
        raise ValueError("k must be (H, K)")
    L = int(fft_size) if fft_size is not None else (2 * N if causal else N)
    w, v, mask = _f64(w), _f64(v), _f64(mask)
    if mask is not None and mask.size != L:
        raise ValueError("mask must have fft_size entries")
    y = np.empty((B, H, N))
    _check(_load().orc_conv_fwd(_ptr(u), _ptr(w), _ptr(v), _ptr(k), _ptr(mask),
                                B, H, N, K, L, int(causal), _ptr(y)), "conv_fwd")
    return y


def conv_bwd(dy, u, k, *, fft_size=None, causal=True, w=None, v=None, mask=None):
    """Gradients of <y, dy> (A15): returns dict du, dw, dv (None when the
    matching gate is absent) and dk (H, K) summed over the batch."""
    dy, u, k = _f64(dy), _f64(u), _f64(k)
    B, H, N = u.shape
    K = k.shape[1]
    L = int(fft_size) if fft_size is not None else (2 * N if causal else N)
    w, v, mask = _f64(w), _f64(v), _f64(mask)
    du = np.empty((B, H, N))
    dw = np.empty((B, H, N)) if w is not None else None
    dv = np.empty((B, H, N)) if v is not None else None
    dk = np.empty((H, K))
    _check(_load().orc_conv_bwd(_ptr(dy), _ptr(u), _ptr(w), _ptr(v), _ptr(k), _ptr(mask),
                                B, H, N, K, L, int(causal), _ptr(du), _ptr(dw),
                                _ptr(dv), _ptr(dk)), "conv_bwd")
    return {"du": du, "dw": dw, "dv": dv, "dk": dk}


def direct_conv(g, k, causal=True) -> np.ndarray:
    """Plain O(N*K) definition: causal c[i] = sum_{j<=i} g[j] k[i-j] (P:105,
    A1); circular c[i] = sum_j g[j] k[(i-j) mod N] (A2).  1-D."""
    g, k = _f64(g).ravel(), _f64(k).ravel()
    c = np.empty(g.size)
    _check(_load().orc_direct_conv(_ptr(g), _ptr(k), g.size, k.size, int(causal), _ptr(c)),
           "direct_conv")
    return c


def direct_point(urow, krow, i, wrow=None) -> float:
    """One causal output element c[i] = sum_j g[j] k[i-j] by direct sum --
    used for sampled checks at full problem sizes."""
    urow, krow, wrow = _f64(urow), _f64(krow), _f64(wrow)
    return float(_load().orc_direct_point(_ptr(urow), _ptr(wrow), _ptr(krow), krow.size, int(i)))


def direct_conv_py(g, k, causal=True) -> np.ndarray:
    """Pure-Python loop version of the same definition, for tiny inputs; an
    implementation independent of the C code."""
    g = [float(x) for x in np.ravel(g)]
    k = [float(x) for x in np.ravel(k)]
    N, K = len(g), len(k)
    out = []
    for i in range(N):
        s = 0.0
        if causal:
            for j in range(max(0, i - K + 1), i + 1):
                s += g[j] * k[i - j]
        else:
            for j in range(N):
                s += g[j] * k[(i - j) % N]
        out.append(s)
    return np.array(out)


# --------------------------------------------------------------------------
# frequency-sparse masks (A13)
# --------------------------------------------------------------------------
def sparsity_fraction(dims, zeroed) -> float:
    """S = 1 - prod_i (d_i - a_i)/d_i with a_i = number of TRAILING entries of
    dim i set to zero (A13(i), the reading that reproduces every row of
    tab:sparsity_fraction; the printed formula P:1040 lacks the
    normalisation)."""
    keep = 1.0
    for d, a in zip(dims, zeroed):
        if not (0 <= a <= d):
            raise ValueError("zero count out of range")
        keep *= (d - a) / d
    return 1.0 - keep


def keep_masks_from_zero_counts(dims, zeroed):
    """Per-dimension keep masks for the slicing `k_f[..., x:, ...] = 0` of
    P:1036-1038: the zeroed entries of dim j are its TRAILING a_j entries
    (indices >= d_j - a_j), the count reading A13(i) that reproduces
    tab:sparsity_fraction.  Pinned by the hand-enumerated
    golden masks in tests/golden/sparsity_masks.json."""
    return [np.arange(d) < (d - a) for d, a in zip(dims, zeroed)]


def keep_set(dims, keeps) -> np.ndarray:
    """keep(f) before the Hermitian closure: frequency f of the length-L
    spectrum, L = prod(dims), written in the digit grid of the reshape
    `k_f.reshape(d_0, d_1, ...)` (row-major: dim 0 is the SLOWEST
    digit, A13(ii)), is kept iff every digit is kept in its dimension."""
    dims = [int(d) for d in dims]
    L = int(np.prod(dims))
    ok = np.ones(L, dtype=bool)
    rem = np.arange(L)
    for j in range(len(dims) - 1, -1, -1):  # fastest digit first
        digit = rem % dims[j]
        rem = rem // dims[j]
        ok &= np.asarray(keeps[j], dtype=bool)[digit]
    return ok


def frequency_mask(dims, keeps) -> np.ndarray:
    """0/1 mask over the length-L spectrum: keep_set applied
    Hermitian-symmetrically, m[f] = keep(f) or keep((L - f) mod L), so the
    output stays real (A13(iii); the paper is silent on real output)."""
    k = keep_set(dims, keeps)
    L = k.size
    m = k | k[(L - np.arange(L)) % L]
    return m.astype(np.float64)


# --------------------------------------------------------------------------
# bidirectional (two-sided) long convolution -- SURVEY 8(f) NEXT-4, reading
# B1 in DESIGN.md (the paper names M2-BERT, whose long
# convolutions are bidirectional, but prints no formula for them)
# --------------------------------------------------------------------------
def conv_fwd_bidir(u, k_fwd, k_bwd, *, w=None, v=None):
    """Bidirectional convolution, reading B1:

        c[i] = sum_{j<=i} g[j] k_fwd[i-j]  +  sum_{j>=i} g[j] k_bwd[j-i]

    (lag 0 carries k_fwd[0] + k_bwd[0]), g = u [* w], y = [v *] c.  Written
    out as its two halves: the causal convolution of g with k_fwd (the
    pinned conv_fwd) plus the time reverse of the causal convolution of the
    reversed g with k_bwd.  u, w, v: (B, H, N); k_fwd, k_bwd: (H, K), K <= N.
    Returns fp64 (B, H, N)."""
    u = _f64(u)
    g = u * _f64(w) if w is not None else u
    c = conv_fwd(g, k_fwd) + conv_fwd(g[..., ::-1], k_bwd)[..., ::-1]
    return c * _f64(v) if v is not None else c


def conv_bwd_bidir(dy, u, k_fwd, k_bwd, *, w=None, v=None):
    """Gradients of <y, dy> for conv_fwd_bidir: dc = dy [* v]; dg = the
    adjoint of each half (conv_bwd of the causal half, time-reversed conv_bwd
    of the anti-causal half); du = dg [* w]; dw = dg * u; dv = dy * c;
    dk_fwd[t] = sum_b sum_i dc[i] g[i-t], dk_bwd[t] = sum_b sum_i dc[i]
    g[i+t] (t < K).  Returns dict du, dw, dv, dk_fwd, dk_bwd."""
    dy, u = _f64(dy), _f64(u)
    g = u * _f64(w) if w is not None else u
    dc = dy * _f64(v) if v is not None else dy
    a = conv_bwd(dc, g, k_fwd)
    b = conv_bwd(np.ascontiguousarray(dc[..., ::-1]), np.ascontiguousarray(g[..., ::-1]), k_bwd)
    dg = a["du"] + b["du"][..., ::-1]
    out = {"dk_fwd": a["dk"], "dk_bwd": b["dk"], "dw": None, "dv": None}
    out["du"] = dg * _f64(w) if w is not None else dg
    if w is not None:
        out["dw"] = dg * u
    if v is not None:
        out["dv"] = dy * conv_fwd_bidir(u, k_fwd, k_bwd, w=w)
    return out


def direct_conv_bidir_py(g, k_fwd, k_bwd) -> np.ndarray:
    """Pure-Python loops of the B1 definition (both sums written out), for
    tiny inputs: an implementation independent of the FFT path."""
    g = [float(x) for x in np.ravel(g)]
    kf = [float(x) for x in np.ravel(k_fwd)]
    kb = [float(x) for x in np.ravel(k_bwd)]
    N = len(g)
    out = []
    for i in range(N):
        s = 0.0
        for j in range(N):
            if 0 <= i - j < len(kf):
                s += g[j] * kf[i - j]
            if 0 <= j - i < len(kb):
                s += g[j] * kb[j - i]
        out.append(s)
    return np.array(out)
