"""Summarise an ncu report (raw page) for the kernels in it: time, DRAM bytes,
throughputs, occupancy, stall reasons.  Usage: python tools/ncu_summary.py rep [regex]"""
import csv, io, re, subprocess, sys

METRICS = [
    ("time_ms", "gpu__time_duration.sum", 1e-6),
    ("dram_read_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_write_MB", "dram__bytes_write.sum", 1e-6),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("l1_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("l2_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("l1_hit", "l1tex__t_sector_hit_rate.pct", 1),
    ("l2_hit", "lts__t_sector_hit_rate.pct", 1),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("fma_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("inst", "smsp__inst_executed.sum", 1),
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summary(rep, pat=None):
    h, units, data = load(rep)
    res = []
    for r in data:
        name = r[h.index("Kernel Name")]
        if pat and not re.search(pat, name):
            continue
        d = {"kernel": name.split("(")[0]}
        for key, m, sc in METRICS:
            if m in h:
                v = r[h.index(m)].replace(",", "")
                u = units[h.index(m)]
                try:
                    x = float(v)
                except ValueError:
                    continue
                if m == "gpu__time_duration.sum":
                    x *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ms": 1e6, "us": 1e3, "ns": 1}.get(u, 1)
                if m.startswith("dram__bytes"):
                    x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                d[key] = x * sc
        stalls = {k: float(r[i].replace(",", "") or 0) for i, k in enumerate(h)
                  if k.startswith("smsp__average_warp_latency_issue_stalled_") and
                  k.endswith("_per_issue_active.ratio") and r[i]}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
        d["top_stalls"] = {k.replace("smsp__average_warp_latency_issue_stalled_", "")
                           .replace("_per_issue_active.ratio", ""): round(v, 2) for k, v in top}
        res.append(d)
    return res


if __name__ == "__main__":
    import json
    for d in summary(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None):
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items()}))
