"""Experiment: per-phase clock64 stamps of the fused forward kernel (CTA 0,
warpgroup 0, warps 0/4) from a -DFC_TRACE build (tools/trace_fwd.sh)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_05908_b200 import FFTConvPlan
from paper_2311_05908_b200 import _abi

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
B, H = 64, 768
dev = torch.device("cuda:0")
plan = FFTConvPlan(N, 2 * N, torch.float16, causal=True)
k = torch.randn(H, N, device=dev)
kf = plan.precompute_kf(k)
u = torch.randn(B, H, N, device=dev, dtype=torch.float16)
w = torch.randn_like(u); v = torch.randn_like(u)
for _ in range(3):
    y = plan.gated_fwd(u, w, v, kf)
torch.cuda.synchronize()
lib = _abi.lib()
buf = np.zeros((2, 64, 16), dtype=np.int64)
lib.fc_trace_dump(buf.ctypes.data_as(ctypes.c_void_p))
names = ["load", "syncA", "issA", "epi1", "syncB", "issB", "epi2", "syncBi", "issBi", "epi3", "syncAi", "issAi", "epi4", "endsync"]
for wsel in (0, 1):
    d = np.diff(buf[wsel, :, :15], axis=1)
    ok = buf[wsel, :, 0] > 0
    d = d[ok][2:]
    print(f"warp {4*wsel}: tiles {len(d)}  tile cycles median {np.median(buf[wsel,ok,14]-buf[wsel,ok,0]):.0f}")
    for i, nm in enumerate(names):
        print(f"  {nm:8s} {np.median(d[:, i]):8.0f} {np.mean(d[:, i]):8.0f}")
    e4w = (buf[wsel, ok, 15] - buf[wsel, ok, 12])[2:]
    print(f"  epi4 until MMA wait done {np.median(e4w):8.0f}")
    nxt = buf[wsel, ok, 0][1:] - buf[wsel, ok, 14][:-1]
    print("  gap to next tile", np.median(nxt))
