"""Summarise ncu outputs for profiles/: a launch list (--csv gpu__time_duration) and full captures (.ncu-rep).

    python tools/ncu_summary.py launches gpurun_out/launches.csv
    python tools/ncu_summary.py rep gpurun_out/sweep.ncu-rep [algorithmic_bytes]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    r"gpu__time_duration\.sum$", r"dram__bytes_read\.sum$", r"dram__bytes_write\.sum$",
    r"gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$", r"dram__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"launch__grid_size$", r"launch__block_size$", r"launch__registers_per_thread$",
    r"launch__shared_mem_per_block_dynamic$", r"sm__warps_active\.avg\.pct_of_peak_sustained_active$",
    r"lts__t_sectors_srcunit_tex_op_read\.sum$", r"lts__t_sectors_srcunit_tex_op_write\.sum$",
    r"sm__throughput\.avg\.pct_of_peak_sustained_elapsed$", r"lts__t_bytes\.sum$",
    r"smsp__inst_executed\.sum$", r"sm__cycles_elapsed\.avg\.per_second$",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    unit = None
    for r in rows[hi + 1:]:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
        unit = r[ui]
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':45s} {'launches':>8s} {'sum_' + unit:>14s} {'mean_' + unit:>12s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:45s} {len(v):8d} {sum(v):14.0f} {sum(v) / len(v):12.0f} {sum(v) / tot:6.1%}")


def rep(path, alg=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        print(f"--- {v[h.index('Kernel Name')][:80]}")
        vals = {}
        for i, n in enumerate(h):
            if any(re.search(k, n) for k in KEYS):
                print(f"  {n:70s} {u[i]:12s} {v[i]}")
                vals[n] = (u[i], v[i])
        stalls = [(n, v[i]) for i, n in enumerate(h)
                  if n.startswith("smsp__average_warp_latency_issue_stalled") or
                  (n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"))]
        tot = 0.0
        pcs = []
        for n, x in stalls:
            try:
                f = float(x.replace(",", ""))
            except ValueError:
                continue
            if n.startswith("smsp__pcsamp_warps_issue_stalled_"):
                pcs.append((f, n[len("smsp__pcsamp_warps_issue_stalled_"):]))
                tot += f
        if pcs and tot:
            print("  pc-sampling stall reasons (share of samples):")
            for f, n in sorted(pcs, reverse=True)[:8]:
                print(f"    {n:40s} {f / tot:6.1%}")
        if alg:
            def num(key, scale):
                un, x = vals[key]
                return float(x.replace(",", "")) * scale[un]
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
            try:
                tr = num("dram__bytes_read.sum", sc) + num("dram__bytes_write.sum", sc)
                print(f"  traffic {tr:.4g} B vs algorithmic {float(alg):.4g} B ({tr / float(alg):.3f}x)")
            except KeyError:
                pass


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        rep(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
