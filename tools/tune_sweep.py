"""Time the persistent sweep under different knobs (GPU; results never change).

    python tools/tune_sweep.py --nx 128 --k 0 2
"""

import argparse
import itertools
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--bs", type=int, default=3)
    ap.add_argument("--k", type=int, nargs="+", default=[0, 2])
    ap.add_argument("--gaps", type=int, nargs="+", default=[1, 2, 3, 5])
    ap.add_argument("--coarse", type=int, nargs="+", default=[0, 100])
    ap.add_argument("--fine", type=int, nargs="+", default=[0, 40])
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import paper_1703_01325_b200 as b2
    n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, args.bs, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
    out = torch.empty_like(rhs)
    for k in args.k:
        t0 = time.perf_counter()
        f = b2.build_preconditioner(a, k)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        info = f.info
        ref = b2.apply_preconditioner(f, rhs).clone()
        print(json.dumps({"k": k, "setup_s": setup, **{x: info[x] for x in
              ("nL", "levels_L", "levels_U", "tiles_L", "tiles_U", "sweep_ctas", "sweep_warps", "sweep_stages",
               "stage_bytes", "apply_bytes")}}), flush=True)
        for gap, cs, fs in itertools.product(args.gaps, args.coarse, args.fine):
            f.tune(gap=gap, coarse_sleep_ns=cs, fine_sleep_ns=fs)
            for _ in range(3):
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
            same = bool(torch.equal(out, ref))
            print(json.dumps({"k": k, "gap": gap, "coarse_ns": cs, "fine_ns": fs, "ms": round(ms, 4),
                              "GBps": round(info["apply_bytes"] / ms / 1e6, 1), "bitwise_same": same}), flush=True)
        del f


if __name__ == "__main__":
    main()
