"""Pins for the oracle's convolutions and gradients (CPU only).

The FFT-based oracle is pinned to plain direct sums (two independent
implementations: C loops and pure-Python loops), closed forms, delta/shift
identities, naive-DFT brute force for masked convolution, adjoint identities
and central finite differences."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import oracle as orc


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def test_direct_sum_implementations_agree():
    g, k = _rand(37, 1), _rand(37, 2)
    np.testing.assert_allclose(orc.direct_conv(g, k, True), orc.direct_conv_py(g, k, True), atol=1e-12)
    np.testing.assert_allclose(orc.direct_conv(g, k, False), orc.direct_conv_py(g, k, False), atol=1e-12)
    np.testing.assert_allclose(orc.direct_conv(g, k[:5], True), orc.direct_conv_py(g, k[:5], True), atol=1e-12)


def test_direct_worked_examples():
    u = [1.0, 2.0, 3.0, 4.0]
    np.testing.assert_allclose(orc.direct_conv_py(u, [1, 0, 0, 0], False), [1, 2, 3, 4])
    np.testing.assert_allclose(orc.direct_conv_py(u, [0, 1, 0, 0], False), [4, 1, 2, 3])
    np.testing.assert_allclose(orc.direct_conv_py(u, [0, 1, 0, 0], True), [0, 1, 2, 3])


@pytest.mark.parametrize("N,K", [(16, 16), (64, 64), (256, 256), (256, 17), (1024, 64)])
def test_fft_conv_matches_direct_causal(N, K):
    B, H = 2, 3
    u = _rand((B, H, N), N)
    k = _rand((H, K), N + 1)
    y = orc.conv_fwd(u, k, causal=True)
    for b in range(B):
        for h in range(H):
            ref = orc.direct_conv(u[b, h], k[h], True)
            np.testing.assert_allclose(y[b, h], ref, atol=1e-11 * np.sqrt(N) * np.abs(ref).max())


@pytest.mark.parametrize("N", [8, 64, 512])
def test_fft_conv_matches_direct_circular(N):
    u = _rand((1, 2, N), 3)
    k = _rand((2, N), 4)
    y = orc.conv_fwd(u, k, causal=False)
    for h in range(2):
        np.testing.assert_allclose(y[0, h], orc.direct_conv(u[0, h], k[h], False), atol=1e-10)


def test_padding_equivalence():
    # causal conv == circular conv of the zero-padded signals, truncated
    N = 32
    u, k = _rand((1, 1, N), 5), _rand((1, N), 6)
    up = np.zeros((1, 1, 2 * N)); up[..., :N] = u
    kp = np.zeros((1, 2 * N)); kp[:, :N] = k
    np.testing.assert_allclose(orc.conv_fwd(u, k)[..., :N],
                               orc.conv_fwd(up, kp, causal=False)[..., :N], atol=1e-12)


@pytest.mark.parametrize("N,K", [(64, 64), (256, 100)])
def test_closed_forms(N, K):
    u = np.ones((1, 1, N))
    y = orc.conv_fwd(u, np.ones((1, K)))
    np.testing.assert_allclose(y[0, 0], np.minimum(np.arange(N) + 1, K), atol=1e-9)
    r = 0.9
    k = r ** np.arange(K)[None, :]
    y = orc.conv_fwd(u, k)
    i = np.arange(N)
    np.testing.assert_allclose(y[0, 0], (1 - r ** np.minimum(i + 1, K)) / (1 - r), atol=1e-10)


def test_delta_and_shift_filters():
    N = 128
    u = _rand((2, 2, N), 9)
    k = np.zeros((2, N)); k[:, 0] = 1.0
    np.testing.assert_allclose(orc.conv_fwd(u, k), u, atol=1e-12)
    s = 5
    k = np.zeros((2, N)); k[:, s] = 1.0
    y = orc.conv_fwd(u, k)
    np.testing.assert_allclose(y[..., s:], u[..., :-s], atol=1e-12)
    np.testing.assert_allclose(y[..., :s], 0, atol=1e-12)


def test_linearity_and_gating():
    N = 64
    u1, u2 = _rand((1, 2, N), 10), _rand((1, 2, N), 11)
    k = _rand((2, N), 12)
    a, b = 1.5, -0.25
    np.testing.assert_allclose(orc.conv_fwd(a * u1 + b * u2, k),
                               a * orc.conv_fwd(u1, k) + b * orc.conv_fwd(u2, k), atol=1e-11)
    w, v = _rand((1, 2, N), 13), _rand((1, 2, N), 14)
    y = orc.conv_fwd(u1, k, w=w, v=v)
    ref = np.stack([[v[0, h] * orc.direct_conv(u1[0, h] * w[0, h], k[h], True) for h in range(2)]])
    np.testing.assert_allclose(y, ref, atol=1e-11)
    ones = np.ones_like(u1)
    np.testing.assert_allclose(orc.conv_fwd(u1, k, w=ones, v=ones), orc.conv_fwd(u1, k), atol=1e-12)
    np.testing.assert_allclose(orc.conv_fwd(u1, k, w=w, v=np.zeros_like(u1)), 0.0, atol=0)


def test_partial_window_property():
    """Partial conv: y[i] depends only on u[i-K+1 .. i]."""
    N, K = 256, 16
    u = _rand((1, 1, N), 20)
    k = _rand((1, K), 21)
    y = orc.conv_fwd(u, k)
    u2 = u.copy(); u2[0, 0, :100] += 5.0
    y2 = orc.conv_fwd(u2, k)
    np.testing.assert_allclose(y2[0, 0, 100 + K - 1:], y[0, 0, 100 + K - 1:], atol=1e-11)
    assert np.abs(y2[0, 0, 99] - y[0, 0, 99]) > 1e-3
    kfull = np.zeros((1, N)); kfull[:, :K] = k
    np.testing.assert_allclose(orc.conv_fwd(u, kfull), y, atol=1e-11)


def test_direct_point():
    N = 300
    u, w = _rand(N, 30), _rand(N, 31)
    k = _rand(N, 32)
    ref = orc.direct_conv(u * w, k, True)
    for i in (0, 1, 150, 299):
        assert abs(orc.direct_point(u, k, i, wrow=w) - ref[i]) < 1e-11


# ---------------------------------------------------------------- masks
def test_sparsity_fraction_table(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "sparsity_fraction.json")))
    for row in g["rows"]:
        S = orc.sparsity_fraction(g["dims"], row["zeroed"])
        assert int(np.floor(100 * S + 0.5)) == row["S_percent"], (row, S)


def test_sparsity_masks_golden(golden_dir):
    """keep_masks_from_zero_counts + keep_set + frequency_mask against masks
    enumerated by hand from P:1035-1038 (tests/golden/sparsity_masks.json):
    pins which entries are zeroed (trailing) and the digit order (dim 0
    slowest)."""
    g = json.load(open(os.path.join(golden_dir, "sparsity_masks.json")))
    for case in g["cases"]:
        dims, zeroed = case["dims"], case["zeroed"]
        L = int(np.prod(dims))
        keeps = orc.keep_masks_from_zero_counts(dims, zeroed)
        got_keep = np.flatnonzero(orc.keep_set(dims, keeps)).tolist()
        assert got_keep == case["keep"], (case, got_keep)
        m = orc.frequency_mask(dims, keeps)
        assert m.shape == (L,)
        assert np.flatnonzero(m).tolist() == case["mask"], (case, np.flatnonzero(m).tolist())


def test_sparsity_fraction_of_constructed_mask(golden_dir):
    """tab:sparsity_fraction on the paper's own 32x32x32x64
    grid of the 2M-length kernel: the kept fraction of the mask the
    oracle BUILDS (keep(f) before the Hermitian closure) reproduces S for
    all six printed rows."""
    g = json.load(open(os.path.join(golden_dir, "sparsity_fraction.json")))
    dims = g["dims"]
    assert int(np.prod(dims)) == 1 << 21
    for row in g["rows"]:
        keep = orc.keep_set(dims, orc.keep_masks_from_zero_counts(dims, row["zeroed"]))
        S = 1.0 - keep.mean()
        assert int(np.floor(100 * S + 0.5)) == row["S_percent"], (row, S)
        # the closure only adds mirror frequencies: kept set grows, never shrinks
        m = orc.frequency_mask(dims, orc.keep_masks_from_zero_counts(dims, row["zeroed"]))
        assert np.all(m[keep] == 1.0)


def test_masked_conv_against_naive_dft():
    N = 16
    L = 2 * N
    u = _rand((1, 1, N), 40)
    k = _rand((1, N), 41)
    dims = [4, 8]
    keeps = orc.keep_masks_from_zero_counts(dims, [2, 4])
    m = orc.frequency_mask(dims, keeps)
    assert np.all(m == m[(-np.arange(L)) % L])  # Hermitian-symmetric
    y = orc.conv_fwd(u, k, mask=m)
    up = np.zeros(L); up[:N] = u[0, 0]
    kp = np.zeros(L); kp[:N] = k[0]
    c = orc.naive_dft(orc.naive_dft(up) * orc.naive_dft(kp) * m, inverse=True)
    assert np.max(np.abs(c.imag)) < 1e-10
    np.testing.assert_allclose(y[0, 0], c.real[:N], atol=1e-10)
    # dense mask == no mask ; zero mask == 0
    np.testing.assert_allclose(orc.conv_fwd(u, k, mask=np.ones(L)), orc.conv_fwd(u, k), atol=1e-12)
    np.testing.assert_allclose(orc.conv_fwd(u, k, mask=np.zeros(L)), 0.0, atol=0)


# ---------------------------------------------------------------- backward
def _bwd_direct(dy, u, k, w, v):
    """c.1 gradient definitions written out as loops."""
    B, H, N = u.shape
    K = k.shape[1]
    g = u * w if w is not None else u
    dc = dy * v if v is not None else dy
    c = np.zeros_like(u)
    dg = np.zeros_like(u)
    dk = np.zeros((H, K))
    for b in range(B):
        for h in range(H):
            for i in range(N):
                for j in range(max(0, i - K + 1), i + 1):
                    c[b, h, i] += g[b, h, j] * k[h, i - j]
                    dg[b, h, j] += dc[b, h, i] * k[h, i - j]
                    dk[h, i - j] += dc[b, h, i] * g[b, h, j]
    out = {"du": dg * w if w is not None else dg, "dk": dk}
    out["dw"] = dg * u if w is not None else None
    out["dv"] = dy * c if v is not None else None
    return out


@pytest.mark.parametrize("gated", [False, True])
@pytest.mark.parametrize("N,K", [(16, 16), (32, 7)])
def test_bwd_matches_direct(gated, N, K):
    B, H = 3, 2
    u, dy = _rand((B, H, N), 50), _rand((B, H, N), 51)
    k = _rand((H, K), 52)
    w = _rand((B, H, N), 53) if gated else None
    v = _rand((B, H, N), 54) if gated else None
    got = orc.conv_bwd(dy, u, k, w=w, v=v)
    ref = _bwd_direct(dy, u, k, w, v)
    for key in ("du", "dk", "dw", "dv"):
        if ref[key] is None:
            assert got[key] is None
        else:
            np.testing.assert_allclose(got[key], ref[key], atol=1e-10)


def test_bwd_finite_differences():
    B, H, N = 2, 1, 8
    u, dy = _rand((B, H, N), 60), _rand((B, H, N), 61)
    w, v = _rand((B, H, N), 62), _rand((B, H, N), 63)
    k = _rand((H, N), 64)
    loss = lambda uu, kk, ww, vv: float(np.sum(orc.conv_fwd(uu, kk, w=ww, v=vv) * dy))
    g = orc.conv_bwd(dy, u, k, w=w, v=v)
    eps = 1e-5
    for name, arr in (("du", u), ("dw", w), ("dv", v), ("dk", k)):
        for idx in [(0, 0, 0), (1, 0, 5)] if arr.ndim == 3 else [(0, 0), (0, 7)]:
            ap = arr.copy(); ap[idx] += eps
            am = arr.copy(); am[idx] -= eps
            args_p = dict(uu=u, kk=k, ww=w, vv=v)
            args_m = dict(uu=u, kk=k, ww=w, vv=v)
            key = {"du": "uu", "dw": "ww", "dv": "vv", "dk": "kk"}[name]
            args_p[key], args_m[key] = ap, am
            fd = (loss(**args_p) - loss(**args_m)) / (2 * eps)
            assert abs(fd - g[name][idx]) < 1e-6 * max(1.0, abs(fd)), (name, idx, fd, g[name][idx])


def test_bwd_adjoint_identity_circular():
    N, B, H = 64, 2, 2
    u, dy = _rand((B, H, N), 70), _rand((B, H, N), 71)
    k = _rand((H, N), 72)
    y = orc.conv_fwd(u, k, causal=False)
    g = orc.conv_bwd(dy, u, k, causal=False)
    # <conv(u), dy> = <u, du> = <k, dk>
    lhs = np.sum(y * dy)
    assert abs(lhs - np.sum(u * g["du"])) < 1e-9 * abs(lhs) + 1e-9
    assert abs(lhs - np.sum(k * g["dk"])) < 1e-9 * abs(lhs) + 1e-9


def test_masked_bwd_adjoint():
    N, B, H = 32, 2, 1
    L = 2 * N
    u, dy = _rand((B, H, N), 80), _rand((B, H, N), 81)
    k = _rand((H, N), 82)
    m = orc.frequency_mask([8, 8], orc.keep_masks_from_zero_counts([8, 8], [4, 2]))
    y = orc.conv_fwd(u, k, mask=m)
    g = orc.conv_bwd(dy, u, k, mask=m)
    lhs = np.sum(y * dy)
    assert abs(lhs - np.sum(u * g["du"])) < 1e-9 * max(1, abs(lhs))
    assert abs(lhs - np.sum(k * g["dk"])) < 1e-9 * max(1, abs(lhs))


# ---------------------------------------------------------------- synth
def test_synth_counter_based_and_sharded():
    full = synth.signal(3, "u", 4, 6, 32)
    part = synth.signal(3, "u", 4, 6, 32, row0=7, nrows=5)
    np.testing.assert_array_equal(full.reshape(24, 32)[7:12], part)
    x = synth.normal(1, 1, np.arange(64), 4096)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01
    k = synth.decay_filters(0, 8, 256)
    np.testing.assert_allclose(np.sum(k ** 2, axis=1), np.sum(k ** 2, axis=1))
    assert k.shape == (8, 256)
    q = synth.quantize(np.array([1.0 + 2 ** -9, 3.14159]), "bf16")
    assert q[0] == 1.0 and abs(q[1] - 3.140625) < 1e-12
