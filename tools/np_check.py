"""Apply time for a list of (nx, bs, k) under the current BILUK_* environment (GPU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_01325_b200 as b2  # noqa: E402

for spec in sys.argv[1:]:
    nx, bs, k = (int(v) for v in spec.split("_"))
    n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, bs, seed=0)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), k)
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
    out = torch.empty_like(rhs)
    for _ in range(3):
        b2.apply_preconditioner(f, rhs, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        b2.apply_preconditioner(f, rhs, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"{spec} nprod-env={os.environ.get('BILUK_NPROD', '-')}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)
