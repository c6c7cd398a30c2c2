import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except Exception:
        print("BAD", l[:300]); continue
    c = d['config']; r = d['roofline']
    print(f"{c['workload'][:58]:58s} {d['value']:.3e} seq/s conv {r['kernel_ms']:.3f}ms frac {r['frac']:.3f} step {d['ms_per_step']:.3f}")
