"""Small driver for ncu captures of the hot kernels (one GPU).

    ncu --set full --import-source on -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/sweep \
        python tools/profile_sweep.py --nx 128 --k 0
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=128)
    ap.add_argument("--bs", type=int, default=3)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--applies", type=int, default=5)
    ap.add_argument("--spmv", type=int, default=2)
    args = ap.parse_args()
    import torch
    import paper_1703_01325_b200 as b2
    n, bs, rp, ci, vals = b2.reservoir_block_grid(args.nx, args.nx, args.nx, args.bs, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, args.k)
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
    out = torch.empty_like(rhs)
    for _ in range(args.applies):
        b2.apply_preconditioner(f, rhs, out=out)
    op = b2.DeviceOperator(a)
    for _ in range(args.spmv):
        op.matvec(rhs, out=out)
    torch.cuda.synchronize()
    f.status()
    print("ok", f.info["apply_bytes"], op.spmv_bytes)


if __name__ == "__main__":
    main()
