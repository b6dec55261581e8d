"""Diagnostics: one batched BiCGSTAB over S independent 64^3 b3 ILU(1) systems.

    python tools/batch_solve_profile.py [S] [MAX_ITERS]

Run under `ncu --metrics gpu__time_duration.sum` to get the per-kernel split of
a solver step (apply, SpMV, fused BLAS-1).
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_01325_b200 as b2  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 16
its = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mats = []
for s in range(S):
    n, bs, rp, ci, v = b2.reservoir_block_grid(64, 64, 64, 3, seed=s)
    mats.append(b2.BcsrMatrix(bs, n, n, rp, ci, v))
big = b2.block_diagonal(mats)
f = b2.build_preconditioner(big, 1)
b = b2.spmv(big, torch.ones(big.shape[0], dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
t0 = time.perf_counter()
x, st = b2.bicgstab_batched(big, b, M=f, cfg=b2.SolverConfig(rel_tol=1e-6, max_iters=its))
torch.cuda.synchronize()
print("systems", S, "iters", its, "s", time.perf_counter() - t0, [s.iterations for s in st][:4], flush=True)
