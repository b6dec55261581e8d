"""Per-tile timeline of one persistent sweep (GPU): where does the time go?

    python tools/trace_sweep.py --nx 128 --k 0 --gap 2 --out gpurun_out/trace_k0.npz

Each tile record: t_ready (its data is in shared memory), t_released (the
progress gate let it poll), t_done (values published), SM id.
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def summarize(tr, levels, nl):
    t0 = tr[:, 0].min()
    ready, rel, done = tr[:, 0] - t0, tr[:, 1] - t0, tr[:, 2] - t0
    out = {"span_us": float(done.max() / 1e3), "tiles": int(tr.shape[0])}
    lv = levels
    nlev = int(lv.max())
    comp = np.zeros(nlev + 1)
    first_rel = np.zeros(nlev + 1)
    for l in range(1, nlev + 1):
        m = lv == l
        comp[l] = done[m].max()
        first_rel[l] = rel[m].min()
    step = np.diff(comp[1:])
    out["level_step_us"] = {"median": float(np.median(step) / 1e3), "mean": float(step.mean() / 1e3),
                            "p90": float(np.percentile(step, 90) / 1e3)}
    out["tile_gate_wait_us_median"] = float(np.median(rel - ready) / 1e3)
    out["tile_poll_compute_us_median"] = float(np.median(done - rel) / 1e3)
    # done spread within a level: max - min
    spread = [float((done[lv == l].max() - done[lv == l].min()) / 1e3) for l in range(1, nlev + 1, max(1, nlev // 50))]
    out["level_done_spread_us_median"] = float(np.median(spread))
    out["L_part_us"] = float(done[:nl].max() / 1e3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--bs", type=int, default=3)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--gap", type=int, nargs="+", default=[2])
    ap.add_argument("--coarse", type=int, default=64)
    ap.add_argument("--fine", type=int, default=0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_1703_01325_b200 as b2
    n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, args.bs, seed=0)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), args.k)
    info = f.info
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
    out = torch.empty_like(rhs)
    # tile levels (combined index) from the plan: recompute from the schedule sizes
    L = b2._native.lib()
    for gap in args.gap:
        f.tune(gap=gap, coarse_sleep_ns=args.coarse, fine_sleep_ns=args.fine)
        for _ in range(3):
            b2.apply_preconditioner(f, rhs, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            b2.apply_preconditioner(f, rhs, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        trace = f.set_trace(True)
        b2.apply_preconditioner(f, rhs, out=out)
        torch.cuda.synchronize()
        f.set_trace(False)
        tr = trace.cpu().numpy().astype(np.int64)
        lev = f.tile_levels()
        s = summarize(tr, lev, info["tiles_L"])
        s.update({"k": args.k, "gap": gap, "ms_untraced": ms, "warps": info["sweep_warps"] * info["sweep_ctas"]})
        print(json.dumps(s), flush=True)
        if args.out:
            base, ext = os.path.splitext(args.out)
            np.savez_compressed(f"{base}_gap{gap}{ext}", trace=tr, levels=lev, nl=info["tiles_L"])
        f.status()


if __name__ == "__main__":
    main()
