"""Per-record timeline of the partitioned sweep (GPU): where does the time go?

    python tools/trace_psweep.py --nx 128 --k 0 --out gpurun_out/ptrace_k0.npz

Stamps per record (globaltimer ns, csrc/psweep.cu): 0 bulk copy issued,
1 bytes seen landed (gather stage), 2 inputs gather issued, 3 dependencies
ready (poll retired), 4 compute start, 5 compute end, 6 (cta << 32 | smid).
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def summarize(tr):
    cta = (tr[:, 6] >> 32).astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    t = (tr[:, :6] - t0) / 1e3   # us
    out = {"span_us": float(t[:, 5].max()), "records": int(tr.shape[0])}
    out["stage_us_median"] = {
        "issue->landed": float(np.median(t[:, 1] - t[:, 0])),
        "landed->gathered": float(np.median(t[:, 2] - t[:, 1])),
        "gathered->deps_ready": float(np.median(t[:, 3] - t[:, 2])),
        "deps_ready->compute_start": float(np.median(t[:, 4] - t[:, 3])),
        "compute": float(np.median(t[:, 5] - t[:, 4])),
    }
    # per-CTA: time between consecutive compute ends, and what the next record waited on
    gaps, busy, first, last = [], [], [], []
    for c in np.unique(cta):
        m = np.where(cta == c)[0]
        tc = t[m]
        first.append(tc[0, 4])
        last.append(tc[-1, 5])
        gaps.append(np.diff(tc[:, 5]))
        busy.append(tc[:, 5] - tc[:, 4])
    g = np.concatenate(gaps)
    out["cta_record_interval_us"] = {"median": float(np.median(g)), "mean": float(g.mean()),
                                     "p90": float(np.percentile(g, 90))}
    out["cta_first_start_us"] = {"min": float(min(first)), "median": float(np.median(first)), "max": float(max(first))}
    out["cta_last_end_us"] = {"min": float(min(last)), "median": float(np.median(last)), "max": float(max(last))}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--bs", type=int, default=3)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_1703_01325_b200 as b2
    n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, args.bs, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, args.k)
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
    out = torch.empty_like(rhs)
    for _ in range(3):
        b2.apply_preconditioner(f, rhs, out=out)
    torch.cuda.synchronize()
    tr = f.set_trace(True)
    for _ in range(2):
        b2.apply_preconditioner(f, rhs, out=out)
    torch.cuda.synchronize()
    f.status()
    h = tr.cpu().numpy().astype(np.int64)[: f.info["records"]]
    np.save((args.out or "/tmp/x.npz")[:-4] + "_dbg.npy", tr.cpu().numpy()[f.info["records"]:])
    s = summarize(h)
    print(s, flush=True)
    if args.out:
        np.savez_compressed(args.out, trace=h, info=np.array([f.info[k] for k in f.info]),
                            keys=np.array(list(f.info)))


if __name__ == "__main__":
    main()
