"""Pins for the oracle's transforms (CPU only).

Each test ties the oracle to something other than itself: the paper's DFT
definition evaluated by hand (golden file), textbook identities (Parseval,
delta/constant transforms), and an independent library (numpy.fft)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.filterwarnings("ignore")


def test_naive_dft_worked_example(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "dft4_example.json")))
    X = orc.naive_dft(g["x"])
    np.testing.assert_allclose(X.real, g["X_re"], atol=1e-12)
    np.testing.assert_allclose(X.imag, g["X_im"], atol=1e-12)
    # the radix-2 path on the same example
    X2 = orc.fft(g["x"])
    np.testing.assert_allclose(X2.real, g["X_re"], atol=1e-12)
    np.testing.assert_allclose(X2.imag, g["X_im"], atol=1e-12)


@pytest.mark.parametrize("n", [1, 2, 4, 8, 64])
def test_delta_and_constant(n):
    d = np.zeros(n); d[0] = 1.0
    np.testing.assert_allclose(orc.fft(d), np.ones(n), atol=1e-12)
    c = np.full(n, 3.0)
    ref = np.zeros(n, complex); ref[0] = 3.0 * n
    np.testing.assert_allclose(orc.fft(c), ref, atol=1e-9)


@pytest.mark.parametrize("n", [2, 8, 32, 128, 512])
def test_radix2_matches_naive_and_numpy(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    X = orc.fft(x)
    np.testing.assert_allclose(X, orc.naive_dft(x), rtol=0, atol=1e-9 * np.sqrt(n))
    np.testing.assert_allclose(X, np.fft.fft(x), rtol=0, atol=1e-10 * n)
    xi = orc.fft(X, inverse=True)
    np.testing.assert_allclose(xi, x, atol=1e-12 * n)
    np.testing.assert_allclose(orc.naive_dft(X, inverse=True), x, atol=1e-10 * n)


@pytest.mark.parametrize("n", [16, 256, 4096])
def test_parseval_and_linearity(n):
    rng = np.random.default_rng(7 + n)
    x = rng.standard_normal(n)
    y = rng.standard_normal(n)
    X, Y = orc.fft(x), orc.fft(y)
    assert abs(np.sum(np.abs(X) ** 2) - n * np.sum(x ** 2)) <= 1e-10 * n * np.sum(x ** 2)
    a, b = 0.7, -1.3
    np.testing.assert_allclose(orc.fft(a * x + b * y), a * X + b * Y, atol=1e-10 * n)


def test_fft_rejects_non_pow2():
    with pytest.raises(ValueError):
        orc.fft(np.ones(12))


@pytest.mark.parametrize("L", [8, 64])
def test_appendix_a1_packing_reading(L):
    """Reading A4/A5: Appendix A.1's one-stage DIT formulas hold
    with X_o = (Z[k] - Z*[M-k])/(2i) and inverse twiddle W^{-k}; the typeset
    forms do not.  Checked against the naive DFT."""
    rng = np.random.default_rng(L)
    x = rng.standard_normal(L)
    M = L // 2
    z = x[0::2] + 1j * x[1::2]
    Z = orc.naive_dft(z)
    Zc = np.conj(Z[(-np.arange(M)) % M])
    Xe = (Z + Zc) / 2
    Xo = (Z - Zc) / (2j)
    kk = np.arange(L)
    W = np.exp(-2j * np.pi * kk / L)
    X = Xe[kk % M] + Xo[kk % M] * W
    Xref = orc.naive_dft(x)
    np.testing.assert_allclose(X, Xref, atol=1e-10)
    Xo_typeset = -1j * (Z - Zc) / (2j)
    X_bad = Xe[kk % M] + Xo_typeset[kk % M] * W
    assert np.max(np.abs(X_bad - Xref)) > 1e-3
    # inverse with W^{-k}
    k = np.arange(M)
    XcM = np.conj(Xref[(M - k) % L])
    Xe2 = (Xref[k] + XcM) / 2
    Xo2 = (Xref[k] - XcM) / 2 * np.exp(2j * np.pi * k / L)
    zr = orc.naive_dft(Xe2 + 1j * Xo2, inverse=True)
    xr = np.empty(L); xr[0::2] = zr.real; xr[1::2] = zr.imag
    np.testing.assert_allclose(xr, x, atol=1e-10)
    Xo2_bad = (Xref[k] - XcM) / 2 * np.exp(-2j * np.pi * k / L)
    zb = orc.naive_dft(Xe2 + 1j * Xo2_bad, inverse=True)
    assert np.max(np.abs(zb.imag - x[1::2])) > 1e-3
