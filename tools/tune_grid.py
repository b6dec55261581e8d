"""Grid of sweep knobs at one problem size (GPU). Prints one JSON line per point.

    python tools/tune_grid.py --nx 128 --k 0 --grid 'warps=1,2,4,8,11 gap=0,2 poll_all=0,1'
"""

import argparse
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--bs", type=int, default=3)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--grid", default="warps=2,4,8 gap=0,2 poll_all=0,1")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--trace", default="", help="comma list of point indices to trace (saved to gpurun_out)")
    args = ap.parse_args()
    import torch
    import paper_1703_01325_b200 as b2
    from tools.trace_sweep import summarize
    n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, args.bs, seed=0)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), args.k)
    info = f.info
    print(json.dumps({"k": args.k, **{x: info[x] for x in ("sweep_warps", "stage_bytes", "levels_L", "tiles_L")}}))
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
    out = torch.empty_like(rhs)
    ref = b2.apply_preconditioner(f, rhs).clone()
    keys, vals_ = [], []
    for item in args.grid.split():
        k, v = item.split("=")
        keys.append(k)
        vals_.append([int(x) for x in v.split(",")])
    traced = {int(x) for x in args.trace.split(",") if x}
    lev = f.tile_levels()
    for idx, point in enumerate(itertools.product(*vals_)):
        knobs = dict(zip(keys, point))
        f.tune(**knobs)
        for _ in range(2):
            b2.apply_preconditioner(f, rhs, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            b2.apply_preconditioner(f, rhs, out=out)
        e1.record()
        torch.cuda.synchronize()
        f.status()
        ms = e0.elapsed_time(e1) / args.reps
        rec = {"i": idx, **knobs, "ms": round(ms, 4), "GBps": round(info["apply_bytes"] / ms / 1e6, 1),
               "same": bool(torch.equal(out, ref))}
        if idx in traced:
            tr = f.set_trace(True)
            b2.apply_preconditioner(f, rhs, out=out)
            torch.cuda.synchronize()
            f.set_trace(False)
            t = tr.cpu().numpy().astype(np.int64)
            rec.update(summarize(t, lev, info["tiles_L"]))
            os.makedirs("gpurun_out", exist_ok=True)
            np.savez_compressed(f"gpurun_out/grid_k{args.k}_{idx}.npz", trace=t, levels=lev, nl=info["tiles_L"])
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
