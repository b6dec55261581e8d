"""Diagnostics: build one synthetic system and apply the preconditioner `reps` times.

    python tools/one_apply.py NX K [REPS]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_01325_b200 as b2  # noqa: E402

nx, k = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, 3, seed=0)
a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
f = b2.build_preconditioner(a, k)
print(f.info["parts"], f.info["records"], flush=True)
rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
out = torch.empty_like(rhs)
for r in range(reps):
    b2.apply_preconditioner(f, rhs, out=out)
    torch.cuda.synchronize()
    f.status()
    print("ok", r, float(out.abs().max()), flush=True)
