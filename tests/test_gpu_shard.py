"""Head sharding: rows (b, h) are independent, so the
convolution of a head shard [h0, h1) of every batch row, with that shard's
k_f, must be BITWISE the corresponding slice of the unsharded call (two-row
packing pairs rows b, b+1 of one head, so sharding by heads keeps every
pair).  The shards run one after another on one GPU, exactly as the ranks
of bench.py --shard run them."""
import numpy as np
import pytest

import synth
from paper_2311_05908_b200.dist import head_shard

torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("N,fft,gated,bwd", [(1024, None, True, True), (8192, None, False, True),
                                              (65536, None, False, False), (1 << 16, 4096, False, True)])
@pytest.mark.parametrize("world", [2, 3])
def test_head_shards_bitwise(N, fft, gated, bwd, world):
    from paper_2311_05908_b200 import FFTConvPlan
    B, H = 3, 7
    plan = FFTConvPlan(N, fft_size=fft, dtype=torch.float16, causal=True)
    K = (fft // 2) if fft else N
    q = lambda name: torch.tensor(synth.quantize(synth.signal(41, name, B, H, N), "f16"), dtype=torch.float16,
                                  device="cuda")
    u, w, v, dy = q("u"), q("w"), q("v"), q("dy")
    k = torch.tensor(synth.decay_filters(41, H, K).astype(np.float32), device="cuda")

    def call(hs):
        kf = plan.precompute_kf(k[hs].contiguous())
        args = [t[:, hs].contiguous() for t in (u, w, v, dy)]
        y = plan.gated_fwd(args[0], args[1], args[2], kf) if gated else plan.fwd(args[0], kf)
        g = plan.bwd(args[3], args[0], kf, K, w=args[1] if gated else None, v=args[2] if gated else None) if bwd else {}
        return y, g

    y_full, g_full = call(slice(0, H))
    for r in range(world):
        h0, h1 = head_shard(H, r, world)
        y, g = call(slice(h0, h1))
        torch.cuda.synchronize()
        assert torch.equal(y, y_full[:, h0:h1]), r
        for key, t in g.items():
            if t is None:
                continue
            ref = g_full[key][h0:h1] if key == "dk" else g_full[key][:, h0:h1]
            assert torch.equal(t, ref), (r, key)
