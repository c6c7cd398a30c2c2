"""Experiment: step time of precompute_kf + conv with no events between the
two calls (events between kernels serialise them), PDL on/off via
FFTCONV_PDL, plus kf-only and conv-only loops.
  python tools/pdl_probe.py [N] [gated]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_05908_b200 import FFTConvPlan

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
gated = len(sys.argv) > 2 and sys.argv[2] == "gated"
B, H = 64, 768
dev = torch.device("cuda:0")
plan = FFTConvPlan(N, 2 * N, torch.float16, causal=True)
k = torch.randn(H, N, device=dev)
kf = plan.precompute_kf(k)
u = torch.randn(B, H, N, device=dev, dtype=torch.float16)
w = torch.randn_like(u); v = torch.randn_like(u); y = torch.empty_like(u)
conv = (lambda: plan.gated_fwd(u, w, v, kf, out=y)) if gated else (lambda: plan.fwd(u, kf, out=y))
def loop(fn, n=300):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
both = lambda: (plan.precompute_kf(k, out=kf), conv())
print(f"N={N} gated={gated} PDL={os.environ.get('FFTCONV_PDL', '1')}: kf {loop(lambda: plan.precompute_kf(k, out=kf)):.2f} us, "
      f"conv {loop(conv):.2f} us, kf+conv {loop(both):.2f} us")
