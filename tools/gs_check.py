"""Grid sweep (engine 2) vs the partitioned sweep (engine 1): results and apply time.

    python tools/gs_check.py [nx,ny,nz,bs ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_01325_b200 as b2  # noqa: E402


def build(engine, n, bs, rp, ci, vals):
    os.environ["BILUK_ENGINE"] = str(engine)
    try:
        return b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 0)
    finally:
        del os.environ["BILUK_ENGINE"]


def timed(f, rhs, out, reps=20):
    for _ in range(3):
        b2.apply_preconditioner(f, rhs, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b2.apply_preconditioner(f, rhs, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


cases = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [
    (5, 4, 3, 3), (8, 8, 8, 3), (16, 16, 16, 3), (17, 9, 13, 2), (32, 32, 32, 1), (24, 20, 16, 4), (64, 64, 64, 3),
    (128, 128, 128, 3)]
for nx, ny, nz, bs in cases:
    n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, ny, nz, bs, seed=0)
    f1 = build(1, n, bs, rp, ci, vals)
    f2 = build(2, n, bs, rp, ci, vals)
    rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
    o1, o2 = torch.empty_like(rhs), torch.empty_like(rhs)
    t0 = time.time()
    b2.apply_preconditioner(f1, rhs, out=o1)
    b2.apply_preconditioner(f2, rhs, out=o2)
    torch.cuda.synchronize()
    f2.status()
    err = float((o1 - o2).abs().max() / o1.abs().max())
    line = f"{nx}x{ny}x{nz} b{bs}: engine {f2.info['engine']} parts {f2.info['parts']} rel diff {err:.2e}"
    if n * bs >= 3 * 64 ** 3:
        line += f"; apply us: e1 {timed(f1, rhs, o1):.1f} e2 {timed(f2, rhs, o2):.1f}"
        b2.apply_preconditioner(f2, rhs, out=o2)
        torch.cuda.synchronize()
        f2.status()
        line += f" (repeat diff {float((o1 - o2).abs().max() / o1.abs().max()):.2e})"
    print(line, flush=True)
