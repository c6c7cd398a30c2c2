"""Quick parity check of the coupled order-3 kernel (N = 8192) vs the oracle."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import synth
from oracle import oracle as orc
from paper_2311_05908_b200 import FFTConvPlan
TDT = {"f16": torch.float16, "bf16": torch.bfloat16}
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
for dtype, gated, B, H in [("f16", False, 2, 1), ("f16", False, 37, 3), ("f16", True, 37, 3), ("bf16", True, 5, 2), ("bf16", False, 4, 2)]:
    plan = FFTConvPlan(N, dtype=TDT[dtype])
    print("order", plan.info.order, "regime", plan.info.regime, "factors", plan.info.factors, flush=True)
    u = synth.quantize(synth.signal(31, "u", B, H, N), dtype)
    k = synth.decay_filters(31, H, N).astype(np.float32)
    kf = plan.precompute_kf(torch.tensor(k, device="cuda"))
    tu = torch.tensor(u, dtype=TDT[dtype], device="cuda")
    if gated:
        w = synth.quantize(synth.signal(31, "w", B, H, N), dtype)
        v = synth.quantize(synth.signal(31, "v", B, H, N), dtype)
        y = plan.gated_fwd(tu, torch.tensor(w, dtype=TDT[dtype], device="cuda"), torch.tensor(v, dtype=TDT[dtype], device="cuda"), kf)
        ref = orc.conv_fwd(u, k.astype(np.float64), w=w, v=v)
    else:
        y = plan.fwd(tu, kf)
        ref = orc.conv_fwd(u, k.astype(np.float64))
    torch.cuda.synchronize()
    got = y.float().cpu().numpy().astype(np.float64)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    mx = np.abs(got - ref).max() / np.abs(ref).max()
    bad = np.argwhere(np.abs(got - ref) > 1e-2 * np.abs(ref).max())
    print(f"{dtype} gated={gated} B={B} H={H}: rel-L2 {rel:.2e} max {mx:.2e} bad {len(bad)} first {bad[:4].tolist()}", flush=True)
