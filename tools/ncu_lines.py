"""Per-source-line stall samples (with the top stall reasons) of one ncu capture.

    python tools/ncu_lines.py gpurun_out/x.ncu-rep psweep.cu 300 560 [min_share]
"""
import csv
import io
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    path, want = sys.argv[1], sys.argv[2]
    lo, hi = int(sys.argv[3]), int(sys.argv[4])
    thr = float(sys.argv[5]) if len(sys.argv) > 5 else 0.001
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, agg = "?", None, {}
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].strip().isdigit():
            continue
        a = agg.setdefault((fname, int(r[0])), {"src": r[1], "n": 0.0, "inst": 0.0})
        a["n"] += f(r[hdr.index("Warp Stall Sampling (All Samples)")])
        a["inst"] += f(r[hdr.index("Instructions Executed")])
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                a[h] = a.get(h, 0.0) + f(r[i])
    tot = sum(a["n"] for a in agg.values()) or 1
    for (fn, ln), a in sorted(agg.items()):
        if fn == want and lo <= ln <= hi and a["n"] > thr * tot:
            rs = sorted(((k[6:], v) for k, v in a.items() if k.startswith("stall_") and v > 0), key=lambda kv: -kv[1])[:3]
            print(f"{ln:4d} {a['n'] / tot:6.2%} inst={a['inst']:10.0f} "
                  f"{' '.join(f'{k}:{v / a[chr(110)]:.0%}' for k, v in rs):42s} {a['src'].strip()[:70]}")


if __name__ == "__main__":
    main()
