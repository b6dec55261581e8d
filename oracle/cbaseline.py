"""CPU baseline: the reference's apply algorithm, timed on this host's cores.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py cpu_baseline and --impl reference).

Setup (symbolic, factorization, split, point expansion, level schedules) uses
the C restatement (coracle.c) so 128^3 systems are ready in seconds; it is NOT
timed.  The timed part is the reference's apply algorithm restated in numpy
exactly as trisolve.py:121-182 runs it with workers=1 (its fastest mode,
SURVEY 3.2): per level one gather, one segmented reduction
(np.add.reduceat) and one scatter over packed level entries (trisolve.py:83-95),
then the batched D^-1 matmul (:148-166).  kind = "port".
"""

from __future__ import annotations

import importlib.util
import os
import time

import numpy as np

from . import coracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _synthetic():
    spec = importlib.util.spec_from_file_location(
        "_synth_for_baseline", os.path.join(os.path.dirname(HERE), "paper_1703_01325_b200", "synthetic.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _pack(rp, ci, v, lev):
    """Level-major packed (rows, cols, vals, segptr) per level (trisolve.py:83-95)."""
    nlev = int(lev.max()) if lev.size else 0
    by = np.argsort(lev, kind="stable")
    counts = np.bincount(lev, minlength=nlev + 1)[1:]
    groups = np.split(by, np.cumsum(counts)[:-1]) if nlev else []
    packed = []
    for rows in groups:
        lens = rp[rows + 1] - rp[rows]
        total = int(lens.sum())
        if total == 0:
            packed.append((rows, None, None, None))
            continue
        starts = rp[rows]
        heads = np.zeros(rows.size, np.int64)
        np.cumsum(lens[:-1], out=heads[1:])
        gather = np.repeat(starts - heads, lens) + np.arange(total, dtype=np.int64)
        seg = np.zeros(rows.size, np.int64)
        np.cumsum(lens[:-1], out=seg[1:])
        packed.append((rows, ci[gather], v[gather], seg))
    return packed


def _solve(packed, b):
    x = b.copy()
    for rows, cols, vals, seg in packed:
        if cols is None:
            continue
        x[rows] = b[rows] - np.add.reduceat(vals * x[cols], seg)
    return x


class PortApply:
    """numpy port of apply_preconditioner on C-oracle factors."""

    def __init__(self, cf: coracle.CFactors):
        L = coracle.lib()
        m = cf.m
        plrp = np.zeros(m + 1, np.int64)
        plci = np.zeros(cf.plnnz, np.int64)
        plv = np.zeros(cf.plnnz)
        purp = np.zeros(m + 1, np.int64)
        puci = np.zeros(cf.punnz, np.int64)
        puv = np.zeros(cf.punnz)
        L.co_get_points.argtypes = [coracle.P] * 7
        L.co_get_points(cf._h, plrp.ctypes.data, plci.ctypes.data, plv.ctypes.data, purp.ctypes.data,
                        puci.ctypes.data, puv.ctypes.data)
        self.lo = _pack(plrp, plci, plv, cf.lo_level_of_row)
        self.up = _pack(purp, puci, puv, cf.up_level_of_row)
        self.dinv = cf.dinv
        self.n, self.bs = cf.n, cf.bs

    def __call__(self, b):
        y = _solve(self.lo, b)
        z = np.matmul(self.dinv, y.reshape(self.n, self.bs, 1)).reshape(-1)
        return _solve(self.up, z)


def apply_bytes(n, bs, nl, nu):
    return 8 * bs * bs * (nl + nu + n) + 4 * (nl + nu) + 8 * (n + 1) + 32 * bs * n


def measure(nx, bs, k, steps=3, warmup=1, seed=0):
    """Time the port on an nx^3 system; returns GB/s of algorithmic apply bytes."""
    synth = _synthetic()
    n, bs, rp, ci, vals = synth.reservoir_block_grid(nx, nx, nx, bs, seed=seed)
    t0 = time.perf_counter()
    cf = coracle.CFactors(n, bs, rp, ci, vals, k)
    port = PortApply(cf)
    t_setup = time.perf_counter() - t0
    b = np.random.default_rng(1).standard_normal(n * bs)
    for _ in range(warmup):
        port(b)
    t0 = time.perf_counter()
    for _ in range(steps):
        port(b)
    t_port = (time.perf_counter() - t0) / steps
    t0 = time.perf_counter()
    for _ in range(max(1, steps)):
        cf.apply(b)
    t_c = (time.perf_counter() - t0) / max(1, steps)
    B = apply_bytes(n, bs, cf.nl, cf.nu)
    return {
        "GBps": B / t_port / 1e9, "ms_per_apply": t_port * 1e3, "cores": 1, "kind": "port",
        "sample": (f"numpy port of reference apply (trisolve.py:121-182, workers=1) on {nx}^3 b{bs} ILU({k}), "
                   f"{steps} applies after {warmup} warm-up: {t_port * 1e3:.1f} ms/apply; "
                   f"C restatement 1 thread: {t_c * 1e3:.1f} ms/apply ({B / t_c / 1e9:.2f} GB/s); "
                   f"untimed C-oracle setup {t_setup:.1f} s"),
        "c_port_GBps": B / t_c / 1e9, "bytes": B,
    }
