"""One small factor + apply (+ a Krylov solve) for compute-sanitizer runs.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py --nx 10 --k 2 --engine 1 --nprod 1
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=10)
    ap.add_argument("--bs", type=int, default=3)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--engine", type=int, default=1)
    ap.add_argument("--nprod", type=int, default=2)
    ap.add_argument("--groups", type=int, default=3)
    ap.add_argument("--solve", type=int, default=1)
    args = ap.parse_args()
    os.environ["BILUK_ENGINE"] = str(args.engine)
    os.environ["BILUK_NPROD"] = str(args.nprod)
    os.environ["BILUK_GROUPS"] = str(args.groups)
    import paper_1703_01325_b200 as b2
    from oracle import iluk_oracle as orc
    n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, args.bs, seed=3)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, args.k)
    of = orc.build_preconditioner(n, bs, rp, ci, vals, args.k)
    rhs = np.random.default_rng(1).standard_normal(n * bs)
    for _ in range(2):
        z = b2.apply_preconditioner(f, rhs)
    err = np.abs(z - of.apply(rhs)).max() / np.abs(z).max()
    assert err <= 1e-12, err
    if args.solve:
        b = b2.spmv(a, np.ones(n * bs))
        _, st = b2.bicgstab(a, b, M=f)
        _, st2 = b2.gmres(a, b, M=f)
        assert st.converged and st2.converged
    print("ok", f.info["engine"], f.info["sweep_warps"], err, flush=True)


if __name__ == "__main__":
    main()
