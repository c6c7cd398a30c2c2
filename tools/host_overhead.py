"""Host-side cost of one API call (enqueue only) vs the GPU time of the same
call, for a few workloads (does the CPU keep the GPU fed?)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench, synth
from paper_2311_05908_b200 import FFTConvPlan
dev = torch.device("cuda:0")
for name in sys.argv[1:] or ["cfg2", "cfg5", "sweep8192"]:
    wl = bench.WORKLOADS[name]
    B, H, N, L = wl["B"], wl["H"], wl["N"], wl["fft"]
    plan = FFTConvPlan(N, fft_size=L, dtype=torch.float16, causal=wl["causal"], device=dev,
                       sparsity=bench.sparsity_spec(wl["sparse"], L))
    u = synth.signal_torch(0, "u", B, H, N, dev, torch.float16)
    k = synth.decay_filters_torch(0, H, wl["K"], dev)
    y = torch.empty_like(u)
    ws = plan.workspace(B, H, device=dev)
    kfb = plan.kf_buffer(H, dev)
    for _ in range(5):
        plan.fwd(u, plan.precompute_kf(k, out=kfb), out=y, workspace=ws)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        plan.precompute_kf(k, out=kfb)
    t1 = time.perf_counter()
    for _ in range(n):
        plan.fwd(u, kfb, out=y, workspace=ws)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        plan.fwd(u, kfb, out=y, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: host enqueue kf {1e6 * (t1 - t0) / n:.1f} us, fwd {1e6 * (t2 - t1) / n:.1f} us; "
          f"GPU fwd back-to-back {1e3 * e0.elapsed_time(e1) / n:.1f} us")
