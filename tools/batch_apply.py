"""Batched apply: nsys independent 64^3 systems as one block-diagonal operator (GPU).

    python tools/batch_apply.py --nsys 8 --nx 64 --k 1
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nsys", type=int, default=8)
    ap.add_argument("--nx", type=int, default=64)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--engine", type=int, default=-1)
    args = ap.parse_args()
    if args.engine >= 0:
        os.environ["BILUK_ENGINE"] = str(args.engine)
    import torch
    import paper_1703_01325_b200 as b2
    mats = []
    for s in range(args.nsys):
        n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, 3, seed=s)
        mats.append(b2.BcsrMatrix(bs, n, n, rp, ci, vals))
    t0 = time.perf_counter()
    big = b2.block_diagonal(mats)
    f = b2.build_preconditioner(big, args.k)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    N = big.shape[0]
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(N)).cuda()
    out = torch.empty_like(rhs)
    for _ in range(3):
        b2.apply_preconditioner(f, rhs, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        b2.apply_preconditioner(f, rhs, out=out)
    e1.record()
    torch.cuda.synchronize()
    f.status()
    ms = e0.elapsed_time(e1) / 5
    inf = f.info
    print({"nsys": args.nsys, "engine": inf["engine"], "apply_ms": round(ms, 3), "GBps": round(inf["apply_bytes"] / ms / 1e6, 1),
           "system_applies_per_s": round(args.nsys / ms * 1e3, 1), "setup_s": round(setup, 2), "levels": inf["levels_L"]},
          flush=True)


if __name__ == "__main__":
    main()
