"""Experiment: per-phase clock64 stamps of the fused forward kernel (CTA 0,
warpgroup 0, warps 0/4) from a -DFC_TRACE build:
  FFTCONV_LIB=<trace build> python tools/trace_fwd.py N [circular]"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_05908_b200 import FFTConvPlan
from paper_2311_05908_b200 import _abi

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
circ = len(sys.argv) > 2 and sys.argv[2].startswith("circular")
gated = not (len(sys.argv) > 2 and sys.argv[2].endswith("plain"))
B, H = 64, 768
dev = torch.device("cuda:0")
plan = FFTConvPlan(N, N if circ else 2 * N, torch.float16, causal=not circ)
k = torch.randn(H, N, device=dev)
kf = plan.precompute_kf(k)
u = torch.randn(B, H, N, device=dev, dtype=torch.float16)
w = torch.randn_like(u); v = torch.randn_like(u)
for _ in range(3):
    y = plan.gated_fwd(u, w, v, kf) if gated else plan.fwd(u, kf)
torch.cuda.synchronize()
lib = _abi.lib()
buf = np.zeros((8, 64, 24), dtype=np.int64)
lib.fc_trace_dump(buf.ctypes.data_as(ctypes.c_void_p))
# stamp index -> phase ending there
seq = [(1, "load/build"), (2, "syncA"), (3, "issA"), (4, "epi1"), (5, "syncB"), (6, "issB"), (7, "epi2"),
       (8, "syncBi"), (9, "issBi"), (10, "epi3"), (11, "syncAi"), (12, "issAi"), (15, "epi4 wait"),
       (16, "epi4 tmem->smem"), (17, "epi4 stg wait"), (18, "epi4 sync"), (19, "epi4 out"), (13, "epi4 tail")]
print(f"N={N} {'circular' if circ else 'causal'} {'gated' if gated else 'plain'}")
# one column per warp: median cycles of each phase (phase = stamp[idx] - previous stamp)
ok = buf[0, :, 0] > 0
b = buf[:, ok][:, 2:]
t0 = b[0, :, 0][None, :]
print("tiles", b.shape[1], " tile cycles median", np.median(b[0, :, 14] - b[0, :, 0]))
print(f"  {'phase':16s}" + "".join(f"   w{w}" for w in range(8)) + "   (end, rel. to warp 0 tile start)")
prev = 0
for idx, nm in seq:
    if np.all(b[:, :, idx] == 0):
        continue
    d = np.median(b[:, :, idx] - b[:, :, prev], axis=1)
    e = np.median(b[:, :, idx] - t0, axis=1)
    print(f"  {nm:16s}" + "".join(f"{x:6.0f}" for x in d) + "  |" + "".join(f"{x:6.0f}" for x in e))
    prev = idx
nxt = buf[0, ok, 0][1:] - buf[0, ok, 14][:-1]
print("  gap to next tile", np.median(nxt))
