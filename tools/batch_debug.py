"""Diagnostics: batched BiCGSTAB vs single solves per system, for each engine (GPU).

    python tools/batch_debug.py

Prints, per engine and k, each system's (batched iterations, single
iterations, relative x difference, relative apply difference, engines).
"""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1703_01325_b200 as b2
def rel(a,b): return float(np.abs(a-b).max()/max(np.abs(b).max(),1e-300))
for eng in (None, "0", "1"):
    if eng is None: os.environ.pop("BILUK_ENGINE", None)
    else: os.environ["BILUK_ENGINE"] = eng
    for k in (0, 1):
        shapes = [(7, 6, 5), (9, 4, 6), (5, 5, 5), (8, 7, 3)]
        mats, rhs = [], []
        for s, (nx, ny, nz) in enumerate(shapes):
            n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, ny, nz, 3, seed=40 + s)
            mats.append(b2.BcsrMatrix(bs, n, n, rp, ci, vals))
            r = np.random.default_rng(s).standard_normal(n * bs)
            rhs.append(np.zeros_like(r) if s == 2 else r)
        big = b2.block_diagonal(mats)
        seg = big.batch_segments
        cfg = b2.SolverConfig(rel_tol=1e-9)
        fb = b2.build_preconditioner(big, k)
        for rep in range(2):
            xb, stats = b2.bicgstab_batched(big, np.concatenate(rhs), M=fb, cfg=cfg)
            out = []
            for i, (m, r) in enumerate(zip(mats, rhs)):
                fs = b2.build_preconditioner(m, k)
                xs, st = b2.bicgstab(m, r, M=fs, cfg=cfg)
                part = xb[seg[i] * 3:seg[i + 1] * 3]
                zb = b2.apply_preconditioner(fb, np.concatenate(rhs))[seg[i]*3:seg[i+1]*3]
                zs = b2.apply_preconditioner(fs, r)
                out.append((stats[i].iterations, st.iterations, f"{rel(part, xs) if i!=2 else 0:.1e}", f"apply {rel(zb,zs) if i!=2 else 0:.1e}", fb.info["engine"], fs.info["engine"]))
            print("eng", eng, "k", k, "rep", rep, out, flush=True)
