"""Summarise ncu raw CSVs and launch lists into markdown (profiles/)."""
import collections
import csv
import glob
import os
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "lts__t_bytes.sum"]


def rows(path):
    return list(csv.reader(l for l in open(path) if not l.startswith("==")))


def raw_summary(path):
    r = rows(path)
    if len(r) < 3:
        return []
    hdr, units = r[0], r[1]
    out = []
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        out.append((d.get("Kernel Name", "?"), [(k, d[k], u.get(k, "")) for k in KEYS if k in d]))
    return out


UNIT = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9}


def launches(path):
    r = rows(path)
    hdr = r[0]
    ki, vi, mi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"),
                      hdr.index("Metric Unit"))
    agg = collections.OrderedDict()
    for row in r[1:]:
        if len(row) > vi and row[mi] == "gpu__time_duration.sum":
            agg.setdefault(row[ki], []).append(float(row[vi].replace(",", "")) * UNIT.get(row[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    return [(k, len(v), sum(v) / len(v), sum(v) / tot) for k, v in agg.items()]


def main(d, out):
    with open(out, "w") as f:
        f.write(f"# ncu summaries ({os.path.basename(d)}; --clock-control none)\n\n")
        f.write("## Launch lists (gpu__time_duration.sum, cold-cache serialised: compare shares)\n\n")
        for p in sorted(glob.glob(os.path.join(d, "launches_*.csv"))):
            f.write(f"### {os.path.basename(p)[9:-4]}\n\n| kernel | launches | mean us | share |\n|---|---|---|---|\n")
            for k, n, m, s in launches(p):
                f.write(f"| `{k[:90]}` | {n} | {m / 1e3:.1f} | {s:.1%} |\n")
            f.write("\n")
        f.write("## Full-set captures (--set full)\n\n")
        for p in sorted(glob.glob(os.path.join(d, "*_raw.csv"))):
            for name, kv in raw_summary(p):
                f.write(f"### {os.path.basename(p)[:-8]}: `{name[:100]}`\n\n")
                for k, v, u in kv:
                    f.write(f"- {k}: {v} {u}\n")
                f.write("\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
