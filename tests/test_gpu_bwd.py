"""GPU parity of the backward pass (fused and multipass regimes) against the
fp64 oracle's gradients (A15): du, dw, dv per element and dk (batch sum)."""
import numpy as np
import pytest

import synth
from oracle import oracle as orc
from parity import assert_parity, assert_parity_f32  # noqa: F401

torch = pytest.importorskip("torch")

REL_L2 = 2e-3
TDT = {"f16": torch.float16, "bf16": torch.bfloat16}


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _run(N, dtype, gated, B, H, seed=0):
    from paper_2311_05908_b200 import FFTConvPlan
    plan = FFTConvPlan(N, dtype=TDT[dtype], causal=True)
    K = N
    q = lambda name: synth.quantize(synth.signal(seed, name, B, H, N), dtype)
    u, dy = q("u"), q("dy")
    w = q("w") if gated else None
    v = q("v") if gated else None
    k = synth.decay_filters(seed, H, K).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=TDT[dtype], device="cuda") if a is not None else None
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    g = plan.bwd(t(dy), t(u), kf, K, w=t(w), v=t(v))
    torch.cuda.synchronize()
    ref = orc.conv_bwd(dy, u, k.astype(np.float64), w=w, v=v)
    out = {key: (g[key].float().cpu().numpy().astype(np.float64) if g[key] is not None else None) for key in g}
    return out, ref


@pytest.mark.gpu
@pytest.mark.parametrize("N", [256, 1024, 2048, 4096, 8192])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("f16", True), ("bf16", True)])
def test_bwd_parity(N, dtype, gated):
    got, ref = _run(N, dtype, gated, B=5, H=3)
    for key in ("du", "dw", "dv", "dk"):
        if ref[key] is None:
            assert got[key] is None
            continue
        assert np.all(np.isfinite(got[key])), key
        assert_parity(got[key], ref[key], str(key))


@pytest.mark.gpu
def test_bwd_deterministic():
    a, _ = _run(1024, "f16", True, B=9, H=2, seed=3)
    b, _ = _run(1024, "f16", True, B=9, H=2, seed=3)
    for key in a:
        if a[key] is not None:
            assert np.array_equal(a[key], b[key]), key


@pytest.mark.gpu
@pytest.mark.parametrize("N", [32768, 131072])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("bf16", True)])
def test_bwd_multilevel_parity(N, dtype, gated):
    """Backward of recursive multipass plans (two outer levels): both T
    chains through every level, the inner backward, and dk inverted level by
    level (deepest first)."""
    got, ref = _run(N, dtype, gated, B=2, H=1, seed=4)
    for key in ("du", "dw", "dv", "dk"):
        if ref[key] is None:
            continue
        assert np.all(np.isfinite(got[key])), key
        assert_parity(got[key], ref[key], str(key))


@pytest.mark.gpu
def test_bwd_cfg3_full_size_sampled():
    """cfg 3 backward at full size (gated causal bf16, B=16, H=768, N=8192),
    bench.py's launch configuration: du, dw, dv on sampled (b, h) rows and dk of
    sampled heads (batch sums over all 16 rows) against the oracle run on
    just those rows / heads."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H, N = 16, 768, 8192
    plan = FFTConvPlan(N, dtype=torch.bfloat16, causal=True)
    q = lambda name: synth.quantize(synth.signal(8, name, B, H, N), "bf16")
    u, w, v, dy = q("u"), q("w"), q("v"), q("dy")
    k = synth.decay_filters(8, H, N).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.bfloat16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    g = plan.bwd(t(dy), t(u), kf, N, w=t(w), v=t(v))
    torch.cuda.synchronize()
    got = {key: g[key].float().cpu().numpy() for key in ("du", "dw", "dv", "dk")}
    rng = np.random.default_rng(9)
    for h in rng.choice(H, 3, replace=False):
        sl = (slice(None), slice(h, h + 1), slice(None))
        ref = orc.conv_bwd(dy[sl], u[sl], k[h:h + 1].astype(np.float64), w=w[sl], v=v[sl])
        assert_parity(got["dk"][h:h + 1], ref["dk"])
        for b in rng.choice(B, 3, replace=False):
            for key in ("du", "dw", "dv"):
                assert_parity(got[key][b, h], ref[key][b, 0], str((key, b, h)))


@pytest.mark.gpu
@pytest.mark.parametrize("N", [4096, 65536])
def test_bwd_circular_multipass(N):
    from paper_2311_05908_b200 import FFTConvPlan
    B, H = 3, 2
    plan = FFTConvPlan(N, fft_size=N, dtype=torch.float16, causal=False)
    q = lambda name: synth.quantize(synth.signal(12, name, B, H, N), "f16")
    u, w, v, dy = q("u"), q("w"), q("v"), q("dy")
    k = synth.decay_filters(12, H, N).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    g = plan.bwd(t(dy), t(u), kf, N, w=t(w), v=t(v))
    torch.cuda.synchronize()
    ref = orc.conv_bwd(dy, u, k.astype(np.float64), causal=False, w=w, v=v)
    for key in ("du", "dw", "dv", "dk"):
        got = g[key].float().cpu().numpy().astype(np.float64)
        assert np.all(np.isfinite(got)), key
        assert_parity(got, ref[key], str(key))


@pytest.mark.gpu
def test_bwd_range_stress_headroom():
    """Backward at N = 1M with u = const 64 (the g chain's DC bin, 64 *
    sqrt(fft_size / 2) = 65536, exceeds fp16 without the plan's headroom
    pre-scale) and k = delta + noise: du and dk against the oracle."""
    from paper_2311_05908_b200 import FFTConvPlan
    N, B, H = 1 << 20, 2, 1
    plan = FFTConvPlan(N, dtype=torch.float16, causal=True)
    u = synth.quantize(np.full((B, H, N), 64.0), "f16")
    dy = synth.quantize(synth.signal(14, "dy", B, H, N), "f16")
    k = np.zeros((H, N))
    k[0, 0] = 1.0
    k[0, 1:] = 1e-2 * synth.normal(14, 9, np.arange(1), N - 1)[0] / np.sqrt(N)
    k = k.astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    g = plan.bwd(t(dy), t(u), kf, N)
    torch.cuda.synchronize()
    ref = orc.conv_bwd(dy, u, k.astype(np.float64))
    assert_parity(g["du"].float().cpu().numpy(), ref["du"], "du")
    assert_parity(g["dk"].cpu().numpy(), ref["dk"], "dk")
