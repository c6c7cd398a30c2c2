"""GPU parity of the partial convolution (filter truncated to K < N,
P:300-303, A12) computed as overlap-save windows of length fft_size = 2C,
C >= K, against the fp64 oracle (causal conv with the truncated filter)."""
import numpy as np
import pytest

import synth
from oracle import oracle as orc
from parity import assert_parity, assert_parity_f32  # noqa: F401

torch = pytest.importorskip("torch")
REL_L2 = 2e-3
TDT = {"f16": torch.float16, "bf16": torch.bfloat16}


@pytest.mark.gpu
@pytest.mark.parametrize("N,L,K", [(16384, 4096, 2048), (16384, 4096, 700), (32768, 16384, 8192)])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("bf16", True)])
def test_partial_parity(N, L, K, dtype, gated):
    from paper_2311_05908_b200 import FFTConvPlan
    B, H = 2, 3
    plan = FFTConvPlan(N, fft_size=L, dtype=TDT[dtype], causal=True)
    assert plan.info.regime == 2
    q = lambda name: synth.quantize(synth.signal(11, name, B, H, N), dtype)
    u = q("u")
    w, v = (q("w"), q("v")) if gated else (None, None)
    k = synth.decay_filters(11, H, K).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=TDT[dtype], device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.gated_fwd(t(u), t(w), t(v), kf) if gated else plan.fwd(t(u), kf)
    got = y.float().cpu().numpy().astype(np.float64)
    ref = orc.conv_fwd(u, k.astype(np.float64), causal=True, w=w, v=v)
    assert_parity(got, ref)


@pytest.mark.gpu
def test_partial_cfg4_shape_sampled():
    """cfg 4: HyenaDNA partial conv B=1, H=256, N=2^20, K=8192 (fft 16384),
    fp16, DNA-like piecewise-constant input; sampled outputs vs direct sums."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H, N, K, L = 1, 256, 1 << 20, 8192, 16384
    plan = FFTConvPlan(N, fft_size=L, dtype=torch.float16, causal=True)
    u = synth.quantize(synth.dna_like(4, B, H, N), "f16")
    k = synth.decay_filters(4, H, K).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    y = plan.fwd(torch.tensor(u, dtype=torch.float16, device="cuda"), kf).float().cpu().numpy()
    rng = np.random.default_rng(4)
    got, ref = [], []
    for h in rng.choice(H, 12, replace=False):
        for i in list(rng.choice(N, 6, replace=False)) + [0, K - 1, K, N - 1]:
            ref.append(orc.direct_point(u[0, h], k[h].astype(np.float64), int(i)))
            got.append(y[0, h, i])
    got, ref = np.array(got), np.array(ref)
    assert_parity(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("N,L,K", [(16384, 4096, 2048), (16384, 4096, 700), (32768, 16384, 8192)])
@pytest.mark.parametrize("dtype,gated", [("f16", False), ("bf16", True)])
def test_partial_backward(N, L, K, dtype, gated):
    """Backward of the partial convolution (NEXT-3): dv from the windows'
    second halves, dg by overlap-add of the dc windows' correlations, dk from
    Sum_windows DC conj(G); against the oracle's causal-conv gradients with the
    truncated filter (A12, A15)."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H = 3, 2
    plan = FFTConvPlan(N, fft_size=L, dtype=TDT[dtype], causal=True)
    assert plan.info.regime == 2
    q = lambda name: synth.quantize(synth.signal(13, name, B, H, N), dtype)
    u, dy = q("u"), q("dy")
    w, v = (q("w"), q("v")) if gated else (None, None)
    k = synth.decay_filters(13, H, K).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=TDT[dtype], device="cuda") if a is not None else None
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    g = plan.bwd(t(dy), t(u), kf, K, w=t(w), v=t(v))
    torch.cuda.synchronize()
    ref = orc.conv_bwd(dy, u, k.astype(np.float64), w=w, v=v)
    for key in ("du", "dw", "dv", "dk"):
        if ref[key] is None:
            continue
        got = g[key].float().cpu().numpy().astype(np.float64)
        assert np.all(np.isfinite(got)), key
        assert_parity(got, ref[key], str(key))


@pytest.mark.gpu
def test_partial_cfg4_backward_full_size_sampled():
    """cfg 4 backward at full size (B=1, H=256, N=2^20, K=8192, fp16), bench's
    launch configuration: du rows and dk of sampled heads against the oracle
    run on those heads."""
    from paper_2311_05908_b200 import FFTConvPlan
    B, H, N, K, L = 1, 256, 1 << 20, 8192, 16384
    plan = FFTConvPlan(N, fft_size=L, dtype=torch.float16, causal=True)
    u = synth.quantize(synth.dna_like(4, B, H, N), "f16")
    dy = synth.quantize(synth.signal(4, "dy", B, H, N), "f16")
    k = synth.decay_filters(4, H, K).astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.float16, device="cuda")
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    g = plan.bwd(t(dy), t(u), kf, K)
    torch.cuda.synchronize()
    du = g["du"].float().cpu().numpy()
    dk = g["dk"].cpu().numpy()
    for h in np.random.default_rng(2).choice(H, 2, replace=False):
        sl = (slice(None), slice(h, h + 1), slice(None))
        ref = orc.conv_bwd(dy[sl], u[sl], k[h:h + 1].astype(np.float64))
        for key, got in (("du", du[sl]), ("dk", dk[h:h + 1])):
            assert_parity(got, ref[key], str((key, h)))
