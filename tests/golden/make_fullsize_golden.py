"""Oracle iteration counts at BASELINE sizes -> tests/golden/fullsize_iters.json (TEST INFRASTRUCTURE).

The C restatement of the reference (oracle/coracle.c: factors, apply, BSR SpMV)
drives the oracle's own Krylov loops (oracle/iluk_oracle.py: ``bicgstab`` -- the
BiCGSTAB contract -- and ``gmres``, the restatement of reference gmres.py:76-186)
on the synthetic reservoir matrices of BASELINE configs[2] and configs[3].  These
runs take minutes on a CPU, so the counts are computed once here and the
``-m gpu`` tests compare the CUDA path's counts (within +-1) with them.

    python tests/golden/make_fullsize_golden.py [--threads 8]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fullsize_iters.json")

CASES = [
    # name, grid, bs, k, solver
    ("cfg2_128c_b3_k0_bicgstab", 128, 3, 0, "bicgstab"),
    ("cfg3_100c_b4_k1_gmres30", 100, 4, 1, "gmres"),
    ("cfg3_100c_b8_k1_gmres30", 100, 8, 1, "gmres"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    import paper_1703_01325_b200.synthetic as syn
    from oracle import coracle
    from oracle import iluk_oracle as orc
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name, nx, bs, k, solver in CASES:
        if args.only and args.only != name:
            continue
        t0 = time.time()
        n, bs, rp, ci, vals = syn.reservoir_block_grid(nx, nx, nx, bs, seed=0)
        b = syn.ones_rhs(n, bs, rp, ci, vals)
        cf = coracle.CFactors(n, bs, rp, ci, vals, k)
        t1 = time.time()
        mv = lambda v: coracle.bsr_spmv(n, bs, rp, ci, vals, v, threads=args.threads)  # noqa: E731
        pc = lambda v: cf.apply(v, threads=args.threads)  # noqa: E731
        if solver == "bicgstab":
            _, its, conv, rel, _ = orc.bicgstab(mv, b, pc, rel_tol=1e-6)
        else:
            _, its, conv, rel, _ = orc.gmres(mv, b, pc, restart=30, rel_tol=1e-6)
        res[name] = {"grid": nx, "bs": bs, "k": k, "solver": solver, "iterations": int(its), "converged": bool(conv),
                     "relres": float(rel), "setup_s": round(t1 - t0, 1), "solve_s": round(time.time() - t1, 1)}
        print(name, res[name], flush=True)
        json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)
        del cf


if __name__ == "__main__":
    main()
