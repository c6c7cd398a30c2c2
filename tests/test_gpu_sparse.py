"""GPU parity of frequency-sparse convolutions (k_f masked, P:310-314,
P:1006-1060; mask semantics A13) against the fp64 oracle with the same mask,
and checks that masked rows of the multipass inner pass are skipped."""
import numpy as np
import pytest

import synth
from oracle import oracle as orc
from parity import assert_parity, assert_parity_f32  # noqa: F401

torch = pytest.importorskip("torch")
REL_L2 = 2e-3


def _run(N, dims, keeps, B=4, H=3, gated=False, seed=21):
    from paper_2311_05908_b200 import FFTConvPlan
    plan = FFTConvPlan(N, dtype=torch.float16, causal=True, sparsity=(dims, keeps))
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), "f16")
    u = q("u")
    w, v = (q("w"), q("v")) if gated else (None, None)
    k = synth.decay_filters(seed, H, N).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.gated_fwd(t(u), t(w), t(v), kf) if gated else plan.fwd(t(u), kf)
    m = orc.frequency_mask(dims, keeps)
    ref = orc.conv_fwd(u, k.astype(np.float64), w=w, v=v, mask=m)
    got = y.float().cpu().numpy().astype(np.float64)
    return plan, got, ref, m


@pytest.mark.gpu
def test_sparse_rows_skipped_cfg5_pattern():
    """cfg 5 shape of the mask: N=16384 (fft 32768 = 16 outer rows x 2048);
    keeping outer rows {0, 1, 8, 15} (closed under f -> L - f) skips 75% of the
    inner Monarch rows."""
    N = 16384
    keep_k0 = np.zeros(16, bool)
    keep_k0[[0, 1, 8, 15]] = True
    dims, keeps = [2048, 16], [np.ones(2048, bool), keep_k0]
    plan, got, ref, m = _run(N, dims, keeps)
    assert abs(plan.info.skip_fraction - 0.75) < 1e-12
    assert abs(plan.info.mask_fraction - 0.75) < 1e-12
    assert_parity(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("N,dims,zeroed", [
    (16384, [8, 8, 8, 64], [4, 4, 0, 0]),      # tab:sparsity_fraction-style trailing zeros
    (4096, [32, 256], [16, 0]),                # low-pass half of the slow digit
    (1024, [32, 64], [16, 32]),                # fused regime (no skipping, mask only)
])
@pytest.mark.parametrize("gated", [False, True])
def test_sparse_patterns(N, dims, zeroed, gated):
    keeps = orc.keep_masks_from_zero_counts(dims, zeroed)
    plan, got, ref, m = _run(N, dims, keeps, gated=gated)
    assert abs(plan.info.mask_fraction - (1 - m.mean())) < 1e-12
    assert_parity(got, ref)


@pytest.mark.gpu
def test_sparse_all_masked_is_zero():
    N = 8192
    dims, keeps = [16384], [np.zeros(16384, bool)]
    plan, got, ref, m = _run(N, dims, keeps, B=2, H=2)
    assert np.all(got == 0) and np.all(ref == 0)


@pytest.mark.gpu
@pytest.mark.parametrize("N,dims,zeroed", [
    (16384, [2048, 16], None),                 # cfg 5 row pattern (75% of inner rows skipped forward)
    (1024, [32, 64], [16, 32]),                # fused regime
])
def test_sparse_backward(N, dims, zeroed):
    """Backward of a frequency-sparse conv (NEXT-3): the oracle's gradients
    with the same mask (dg uses conj(K_f) * m, dk = Re IFFT(m * sum DC conj G))."""
    from paper_2311_05908_b200 import FFTConvPlan
    if zeroed is None:
        keep_k0 = np.zeros(16, bool)
        keep_k0[[0, 1, 8, 15]] = True
        keeps = [np.ones(2048, bool), keep_k0]
    else:
        keeps = orc.keep_masks_from_zero_counts(dims, zeroed)
    B, H, seed = 3, 2, 31
    plan = FFTConvPlan(N, dtype=torch.float16, causal=True, sparsity=(dims, keeps))
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), "f16")
    u, w, v, dy = q("u"), q("w"), q("v"), q("dy")
    k = synth.decay_filters(seed, H, N).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    g = plan.bwd(t(dy), t(u), kf, N, w=t(w), v=t(v))
    torch.cuda.synchronize()
    m = orc.frequency_mask(dims, keeps)
    ref = orc.conv_bwd(dy, u, k.astype(np.float64), w=w, v=v, mask=m)
    for key in ("du", "dw", "dv", "dk"):
        got = g[key].float().cpu().numpy().astype(np.float64)
        assert np.all(np.isfinite(got)), key
        assert_parity(got, ref[key], str(key))


@pytest.mark.gpu
def test_sparse_cfg5_full_size_sampled_rows():
    """cfg 5 at full size (B=8, H=768, N=16384, fp16, 75 % of the inner rows
    skipped), bench.py's launch configuration; 16 sampled (b, h) rows compared
    whole against the oracle's masked convolution of those rows."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H, N = 8, 768, 16384
    keep_k0 = np.zeros(16, bool)
    keep_k0[[0, 1, 8, 15]] = True
    dims, keeps = [2048, 16], [np.ones(2048, bool), keep_k0]
    plan = FFTConvPlan(N, dtype=torch.float16, causal=True, sparsity=(dims, keeps))
    u = torch.empty(B, H, N, dtype=torch.float16, device="cuda")
    rows = np.sort(np.random.default_rng(5).choice(B * H, 16, replace=False))
    uh = synth.quantize(synth.signal(6, "u", B, H, N), "f16")
    u.copy_(torch.tensor(uh, dtype=torch.float16))
    k = synth.decay_filters(6, H, N).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.fwd(u, kf).float().cpu().numpy().reshape(B * H, N)
    m = orc.frequency_mask(dims, keeps)
    u2 = uh.reshape(B * H, N)
    for r in rows:
        h = r % H
        ref = orc.conv_fwd(u2[r][None, None, :], k[h:h + 1].astype(np.float64), mask=m)[0, 0]
        assert_parity(y[r], ref, str(r))


@pytest.mark.gpu
@pytest.mark.parametrize("N,dims,zeroed", [
    (32768, [8, 8, 16, 64], [4, 0, 8, 16]),
    (1 << 20, [32, 32, 32, 64], [16, 8, 0, 32]),   # the paper's 2M-length kernel grid
])
def test_sparse_recursive_plans(N, dims, zeroed):
    """Frequency-sparse plans with more than one outer level: the mask acts
    through k_f with inner row r mapped to its frequency digits (level 0
    fastest); forward and, at 32K, backward against the masked oracle."""
    from paper_2311_05908_b200 import FFTConvPlan
    keeps = orc.keep_masks_from_zero_counts(dims, zeroed)
    B, H, seed = 2, 1, 33
    plan = FFTConvPlan(N, dtype=torch.float16, causal=True, sparsity=(dims, keeps))
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), "f16")
    u, dy = q("u"), q("dy")
    k = synth.decay_filters(seed, H, N).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.fwd(t(u), kf).float().cpu().numpy()
    m = orc.frequency_mask(dims, keeps)
    ref = orc.conv_fwd(u, k.astype(np.float64), mask=m)
    assert_parity(y, ref)
    if N <= 32768:
        g = plan.bwd(t(dy), t(u), kf, N)
        torch.cuda.synchronize()
        rb = orc.conv_bwd(dy, u, k.astype(np.float64), mask=m)
        for key in ("du", "dk"):
            got = g[key].float().cpu().numpy()
            assert_parity(got, rb[key], str(key))


def _windows(x, C, NC):
    """overlap-save windows of length 2C: window j = x[(j-1)C : (j+1)C],
    zero before 0 (A12 mechanism); returns (B, H * NC, 2C) ordered (h, j)"""
    B, H, N = x.shape
    pad = np.concatenate([np.zeros((B, H, C)), x], axis=2)
    return np.stack([pad[:, :, j * C:(j + 2) * C] for j in range(NC)], axis=2).reshape(B, H * NC, 2 * C)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,keep_fn", [
    ([256, 16], lambda: [np.ones(256, bool), np.isin(np.arange(16), [0, 1, 15])]),  # inner rows skipped
    ([64, 64], lambda: orc.keep_masks_from_zero_counts([64, 64], [32, 0])),          # slow-digit low-pass
])
def test_sparse_partial_plan(dims, keep_fn):
    """Frequency-sparse PARTIAL plan (N = 16384, fft_size 4096, K = 1500):
    every overlap-save window is a circular fft_size-point convolution with
    the masked K_f (the mask acts on the window spectrum), the output its
    second half.  Oracle: that composition written out window by window with
    the oracle's masked circular convolution (forward) and its gradients
    (backward: dc = dy in the window's second half, dg overlap-added, dk the
    window sum truncated to K)."""
    from paper_2311_05908_b200 import FFTConvPlan
    N, L, K, B, H, seed = 16384, 4096, 1500, 2, 2, 37
    C, NC = L // 2, N // (L // 2)
    keeps = keep_fn()
    plan = FFTConvPlan(N, fft_size=L, dtype=torch.float16, causal=True, sparsity=(dims, keeps))
    assert plan.info.regime == 2
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), "f16")
    u, dy = q("u"), q("dy")
    k = synth.decay_filters(seed, H, K).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.fwd(t(u), kf).float().cpu().numpy()
    g = plan.bwd(t(dy), t(u), kf, K)
    torch.cuda.synchronize()
    m = orc.frequency_mask(dims, keeps)
    kpad = np.zeros((H * NC, L))
    kpad[:, :K] = np.repeat(k.astype(np.float64), NC, axis=0)
    yw = orc.conv_fwd(_windows(u, C, NC), kpad, causal=False, mask=m)          # (B, H*NC, L)
    ref_y = yw[:, :, C:].reshape(B, H, NC * C)
    assert_parity(y, ref_y, "y")
    dyw = np.zeros((B, H * NC, L))
    dyw[:, :, C:] = dy.reshape(B, H * NC, C)
    gb = orc.conv_bwd(dyw, _windows(u, C, NC), kpad, causal=False, mask=m)
    dgw = gb["du"].reshape(B, H, NC, L)
    dg = np.zeros((B, H, N + C))
    for j in range(NC):
        dg[:, :, j * C:(j + 2) * C] += dgw[:, :, j]
    ref_du = dg[:, :, C:]
    ref_dk = gb["dk"].reshape(H, NC, L).sum(axis=1)[:, :K]
    assert_parity(g["du"].float().cpu().numpy(), ref_du, "du")
    assert_parity(g["dk"].cpu().numpy(), ref_dk, "dk")


def _lowpass(L, keep_frac_inv=8):
    """Symmetric low-pass (A13): digit grid [keep_frac_inv * 2, L / (2 keep_frac_inv)]
    (slowest first) with all but the first two slow digits zeroed keeps
    f < L / keep_frac_inv, and the Hermitian closure adds f > L - L / keep_frac_inv."""
    d0 = 2 * keep_frac_inv
    dims = [d0, L // d0]
    return dims, orc.keep_masks_from_zero_counts(dims, [d0 - 2, 0])


@pytest.mark.gpu
@pytest.mark.parametrize("N", [1024, 8192, 16384, 32768])
@pytest.mark.parametrize("gated", [False, True])
def test_sparse_lowpass_slow_digit_skip(N, gated):
    """A genuine symmetric low-pass mask skips the slow digit:
    stage-B column chunks whose frequencies are all masked are left out of
    stage B, the pointwise step and stage B^-1 (here 2 of 4 chunks), in the
    fused (N = 1024), one-level (8192, 16384) and recursive (32768) plans."""
    dims, keeps = _lowpass(2 * N)
    plan, got, ref, m = _run(N, dims, keeps, gated=gated)
    assert abs(plan.info.mask_fraction - (1 - m.mean())) < 1e-12
    assert abs(plan.info.skip_fraction - 0.5) < 1e-12
    assert_parity(got, ref, f"low-pass N={N}")


@pytest.mark.gpu
@pytest.mark.parametrize("N", [1024, 8192])
def test_sparse_lowpass_backward(N):
    """The backward of a slow-digit-skipping plan (dense kernels on the
    masked k_f) against the oracle's masked gradients."""
    from paper_2311_05908_b200 import FFTConvPlan
    dims, keeps = _lowpass(2 * N, 16)
    B, H, seed = 3, 2, 9
    plan = FFTConvPlan(N, dtype=torch.float16, causal=True, sparsity=(dims, keeps))
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), "f16")
    u, w, v, dy = q("u"), q("w"), q("v"), q("dy")
    k = synth.decay_filters(seed, H, N).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    g = plan.bwd(t(dy), t(u), kf, N, w=t(w), v=t(v))
    torch.cuda.synchronize()
    m = orc.frequency_mask(dims, keeps)
    ref = orc.conv_bwd(dy, u, k.astype(np.float64), w=w, v=v, mask=m)
    for key in ("du", "dw", "dv", "dk"):
        assert_parity(g[key].float().cpu().numpy(), ref[key], f"low-pass bwd {key}")
