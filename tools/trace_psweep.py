"""Per-record timeline of the partitioned sweep (GPU): where does the time go?

    python tools/trace_psweep.py --nx 128 --k 0 --out gpurun_out/ptrace_k0.npz

Stamps per record (globaltimer ns, csrc/psweep.cu): 0 bulk copy issued,
1 landed (seen by the compute group), 2 staged, 3 dependencies ready,
4 compute start (before the hand-over barrier), 5 compute end,
6 (cta << 32 | smid), 7 flags.  The debug rows after the records hold, for the
first 16384 records, clock64 stamps of the compute group's stages (thread 0):
landed, prepared, dependencies waited, hand-over, products, published,
arrive + fence, released.
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
        "issue->poll_start": float(np.median(t[:, 1] - t[:, 0])),
        "poll": float(np.median(t[:, 3] - t[:, 1])),
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
    # is the hand-over chain waiting for the next group (start after the previous record's end)?
    late = np.concatenate([t[np.where(cta == c)[0]][1:, 4] - t[np.where(cta == c)[0]][:-1, 5] for c in np.unique(cta)])
    out["start_after_prev_end_us_median"] = float(np.median(late))
    out["cta_record_interval_us"] = {"median": float(np.median(g)), "mean": float(g.mean()),
                                     "p90": float(np.percentile(g, 90))}
    out["cta_first_start_us"] = {"min": float(min(first)), "median": float(np.median(first)), "max": float(max(first))}
    out["cta_last_end_us"] = {"min": float(min(last)), "median": float(np.median(last)), "max": float(max(last))}
    return out


def stages(dbg):
    """Median cycles of the compute group's stages (debug rows)."""
    d = dbg[dbg[:, 0] > 0].astype(np.int64)
    names = ["prep", "dep_wait", "handover", "products", "publish", "arrive_fence", "release"]
    dd = np.diff(d, axis=1)
    return {nm: float(np.median(dd[:, j][(dd[:, j] >= 0) & (dd[:, j] < 10**6)])) for j, nm in enumerate(names)}


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
    full = tr.cpu().numpy().astype(np.int64)
    h, dbg = full[: f.info["records"]], full[f.info["records"]:]
    s = summarize(h)
    s["compute_stage_cycles_median"] = stages(dbg)
    print(s, flush=True)
    if args.out:
        np.savez_compressed(args.out, trace=h, dbg=dbg, info=np.array([f.info[k] for k in f.info]),
                            keys=np.array(list(f.info)))


if __name__ == "__main__":
    main()
