"""Stall reasons, key throughput metrics and the hottest source blocks of one ncu capture.

    python tools/ncu_stalls.py gpurun_out/psw_k0_r02.ncu-rep [algorithmic_bytes] [top]
"""
import csv
import io
import subprocess
import sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1.0, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}


def num(d, k):
    """Value in base units (bytes, seconds) when the unit is known."""
    try:
        return float(d[k][0].replace(",", "")) * SCALE.get(d[k][1], 1.0)
    except (KeyError, ValueError):
        return float("nan")


def main():
    path = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    d = raw(path)
    print("kernel:", d.get("Kernel Name", ("?",))[0][:90])
    dur = num(d, "gpu__time_duration.sum")
    rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
    print(f"duration {dur * 1e6:.1f} us; DRAM read {rd / 1e6:.1f} MB write {wr / 1e6:.1f} MB "
          f"({(rd + wr) / dur / 1e9:.0f} GB/s)" + (f"; algorithmic {alg / 1e6:.1f} MB -> {alg / dur / 1e9:.0f} GB/s, "
                                                   f"traffic/alg {(rd + wr) / alg:.2f}" if alg else ""))
    for k in ("sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"):
        if k in d:
            print(f"  {k:60s} {d[k][0]} {d[k][1]}")
    st = [(k, num(d, k)) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    print("stall samples:")
    for k, x in sorted(st, key=lambda kv: -kv[1])[:8]:
        print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {x / tot:6.1%}")
    # hottest CUDA source lines: SASS stall samples attributed to (file, line)
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, agg, hdr = "?", {}, None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].strip().isdigit():
            continue
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            w = float(r[wi] or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]))
        agg.setdefault(key, [0.0, r[1]])[0] += w
    tot = sum(v[0] for v in agg.values()) or 1
    print("hottest source lines (share of stall samples):")
    for (f, ln), (w, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {w / tot:6.1%}  {f}:{ln}: {src.strip()[:100]}")


if __name__ == "__main__":
    main()
