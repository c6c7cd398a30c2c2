"""Pins for the oracle's bidirectional convolution (reading B1, DESIGN.md;
SURVEY 8(f) NEXT-4), CPU only: an independent pure-Python two-sided direct
sum, the special cases that reduce to the causal conv or to a shift, a
closed form, central finite differences and the adjoint identity."""
import numpy as np
import pytest

from oracle import oracle as orc


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


@pytest.mark.parametrize("N,K", [(16, 16), (32, 7), (64, 64)])
def test_bidir_matches_two_sided_direct_sum(N, K):
    B, H = 2, 2
    u, w, v = _rand((B, H, N), 1), _rand((B, H, N), 2), _rand((B, H, N), 3)
    kf, kb = _rand((H, K), 4), _rand((H, K), 5)
    y = orc.conv_fwd_bidir(u, kf, kb)
    yg = orc.conv_fwd_bidir(u, kf, kb, w=w, v=v)
    for b in range(B):
        for h in range(H):
            ref = orc.direct_conv_bidir_py(u[b, h], kf[h], kb[h])
            np.testing.assert_allclose(y[b, h], ref, atol=1e-11)
            refg = v[b, h] * orc.direct_conv_bidir_py(u[b, h] * w[b, h], kf[h], kb[h])
            np.testing.assert_allclose(yg[b, h], refg, atol=1e-11)


def test_bidir_special_cases():
    N, K = 32, 32
    u = _rand((1, 2, N), 6)
    kf = _rand((2, K), 7)
    # no anti-causal part: the causal convolution
    np.testing.assert_allclose(orc.conv_fwd_bidir(u, kf, np.zeros((2, K))), orc.conv_fwd(u, kf), atol=1e-12)
    # k_bwd = delta_s, no causal part: y[i] = u[i + s] (zero past the end)
    for s in (0, 1, 5):
        kb = np.zeros((2, K)); kb[:, s] = 1.0
        y = orc.conv_fwd_bidir(u, np.zeros((2, K)), kb)
        ref = np.zeros_like(u); ref[..., :N - s] = u[..., s:]
        np.testing.assert_allclose(y, ref, atol=1e-12)
    # lag 0 counts both k_fwd[0] and k_bwd[0]
    d = np.zeros((2, K)); d[:, 0] = 1.0
    np.testing.assert_allclose(orc.conv_fwd_bidir(u, d, d), 2 * u, atol=1e-12)


@pytest.mark.parametrize("N,K", [(16, 16), (64, 9)])
def test_bidir_closed_form(N, K):
    # u = 1, k_fwd = 1, k_bwd = 1: y[i] = min(i+1, K) + min(N-i, K)
    y = orc.conv_fwd_bidir(np.ones((1, 1, N)), np.ones((1, K)), np.ones((1, K)))
    i = np.arange(N)
    np.testing.assert_allclose(y[0, 0], np.minimum(i + 1, K) + np.minimum(N - i, K), atol=1e-10)


def test_bidir_bwd_finite_differences():
    B, H, N, K = 2, 1, 8, 8
    u, w, v, dy = (_rand((B, H, N), s) for s in (10, 11, 12, 13))
    kf, kb = _rand((H, K), 14), _rand((H, K), 15)
    g = orc.conv_bwd_bidir(dy, u, kf, kb, w=w, v=v)
    loss = lambda uu, ww, vv, a, b: float(np.sum(orc.conv_fwd_bidir(uu, a, b, w=ww, v=vv) * dy))
    eps = 1e-6
    def fd(arr, idx, f):
        p = arr.copy(); p[idx] += eps
        m = arr.copy(); m[idx] -= eps
        return (f(p) - f(m)) / (2 * eps)
    for idx in [(0, 0, 0), (1, 0, 5), (0, 0, 7)]:
        assert abs(fd(u, idx, lambda x: loss(x, w, v, kf, kb)) - g["du"][idx]) < 1e-6
        assert abs(fd(w, idx, lambda x: loss(u, x, v, kf, kb)) - g["dw"][idx]) < 1e-6
        assert abs(fd(v, idx, lambda x: loss(u, w, x, kf, kb)) - g["dv"][idx]) < 1e-6
    for idx in [(0, 0), (0, 3), (0, 7)]:
        assert abs(fd(kf, idx, lambda x: loss(u, w, v, x, kb)) - g["dk_fwd"][idx]) < 1e-6
        assert abs(fd(kb, idx, lambda x: loss(u, w, v, kf, x)) - g["dk_bwd"][idx]) < 1e-6


def test_bidir_bwd_adjoint_and_lag0():
    B, H, N, K = 3, 2, 32, 16
    u, dy = _rand((B, H, N), 20), _rand((B, H, N), 21)
    kf, kb = _rand((H, K), 22), _rand((H, K), 23)
    g = orc.conv_bwd_bidir(dy, u, kf, kb)
    # <conv(u), dy> = <u, du>
    assert abs(np.sum(orc.conv_fwd_bidir(u, kf, kb) * dy) - np.sum(u * g["du"])) < 1e-9
    # <conv(u), dy> is linear in (kf, kb): = <kf, dk_fwd> + <kb, dk_bwd>
    assert abs(np.sum(orc.conv_fwd_bidir(u, kf, kb) * dy)
               - np.sum(kf * g["dk_fwd"]) - np.sum(kb * g["dk_bwd"])) < 1e-9
    # both halves see lag 0: dk_fwd[0] == dk_bwd[0] = sum dc * g
    np.testing.assert_allclose(g["dk_fwd"][:, 0], g["dk_bwd"][:, 0], atol=1e-10)
    np.testing.assert_allclose(g["dk_fwd"][:, 0], np.sum(dy * u, axis=(0, 2)), atol=1e-10)
