"""Per-workload DRAM traffic of one conv call (sum over its kernels, k_f
precompute excluded) from ncu launch lists with dram__bytes_* metrics ->
profiles/ncu_traffic.json (read by bench.py for roofline.traffic)."""
import collections
import csv
import glob
import json
import os
import sys

KF = ("precompute_kf", "mp_kf_cols", "mp_kf_rows", "mp_cols_cplx")


def per_call(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ii, ki, mi, vi = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    launches = collections.OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    names = [d["name"] for d in launches.values()]
    steps = sum(1 for n in names if n.startswith("precompute_kf") or "mp_kf_cols" in n)
    if steps == 0:
        return None
    byts = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in launches.values():
        if any(k in d["name"] for k in KF):
            continue
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        byts[d["name"]] += b
        cnt[d["name"]] += 1
    total = sum(byts.values()) / steps
    return total, {n[:80]: cnt[n] / steps for n in cnt}


def main(d, out):
    res = json.load(open(out)) if os.path.exists(out) else {}
    for p in sorted(glob.glob(os.path.join(d, "launches_*.csv"))):
        w = os.path.basename(p)[len("launches_"):-4]
        r = per_call(p)
        if r is None:
            continue
        res[w] = {"dram_bytes_per_launch": r[0], "kernels_per_call": r[1],
                  "source": os.path.join("profiles", "r01_final", os.path.basename(p)),
                  "note": "sum of dram__bytes_read+write over the conv call's kernels (one step; k_f precompute excluded)"}
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
