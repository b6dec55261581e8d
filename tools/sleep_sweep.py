"""Apply time versus the dependency re-poll back-off (GPU).

    python tools/sleep_sweep.py --nx 128 --k 0 --sleep 0 100 200 400 800
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--sleep", type=int, nargs="+", default=[0, 100, 200, 400, 800])
    args = ap.parse_args()
    import torch
    import paper_1703_01325_b200 as b2
    n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, 3, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, args.k)
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
    out = torch.empty_like(rhs)
    for sl in args.sleep:
        f.tune(fine_sleep_ns=max(sl, 1))
        for _ in range(3):
            b2.apply_preconditioner(f, rhs, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            b2.apply_preconditioner(f, rhs, out=out)
        e1.record()
        torch.cuda.synchronize()
        f.status()
        print({"sleep_ns": sl, "us": e0.elapsed_time(e1) / 10 * 1e3}, flush=True)


if __name__ == "__main__":
    main()
