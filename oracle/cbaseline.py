"""CPU baseline: the reference's algorithms, timed on this host's cores.

TEST / BASELINE INFRASTRUCTURE ONLY (bench.py cpu_baseline and --impl reference).

Setup (symbolic, factorization, split, point expansion, level schedules) uses
the C restatement (coracle.c) so 128^3 systems are ready in seconds; it is NOT
timed.  The timed parts are the reference's algorithms restated in numpy
exactly as the reference runs them:

* apply (trisolve.py:121-182): per level one gather, one segmented reduction
  (np.add.reduceat) and one scatter over packed level entries
  (trisolve.py:83-95), then the batched D^-1 matmul (:148-166).  ``workers``
  splits each level's rows into contiguous chunks on a shared thread pool,
  fork-join per level (parallel.py:32-53) -- numpy releases the GIL there.
* spmv (sparse.py:278-301): the same gather / reduceat over the point CSR
  expansion of A.
* Krylov: the oracle's BiCGSTAB contract and its GMRES restatement
  (gmres.py:76-186) over those two operators.

kind = "port" (the reference is Python; it cannot run where /root/reference is
absent, so its algorithm is restated here and pinned to its goldens by tests/).
"""

from __future__ import annotations

import importlib.util
import os
import subprocess
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import coracle
from . import iluk_oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))
_POOLS = {}


def _synthetic():
    spec = importlib.util.spec_from_file_location(
        "_synth_for_baseline", os.path.join(os.path.dirname(HERE), "paper_1703_01325_b200", "synthetic.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def host_cores():
    """(logical CPUs usable by this process, lscpu summary line)."""
    n = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    desc = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        desc = (f"{kv.get('Model name', '?')}; {kv.get('Socket(s)', '?')} socket(s) x "
                f"{kv.get('Core(s) per socket', '?')} cores x {kv.get('Thread(s) per core', '?')} threads; "
                f"CPU(s) {kv.get('CPU(s)', '?')}")
    except (OSError, subprocess.SubprocessError):
        pass
    return n, desc


def _pool(workers):
    if workers not in _POOLS:
        _POOLS[workers] = ThreadPoolExecutor(max_workers=workers)
    return _POOLS[workers]


def _run_chunks(body, n, workers):
    """parallel.py:32-53: contiguous chunks, fork-join, inline for one worker."""
    if n <= 0:
        return
    if workers <= 1 or n == 1:
        body(0, n)
        return
    chunks = min(workers, n)
    bounds = [n * i // chunks for i in range(chunks + 1)]
    futs = [_pool(workers).submit(body, bounds[i], bounds[i + 1]) for i in range(chunks) if bounds[i + 1] > bounds[i]]
    for f in futs:
        f.result()


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
        heads = np.zeros(rows.size + 1, np.int64)
        np.cumsum(lens, out=heads[1:])
        gather = np.repeat(starts - heads[:-1], lens) + np.arange(total, dtype=np.int64)
        packed.append((rows, ci[gather], v[gather], heads))
    return packed


def _solve(packed, b, workers):
    x = b.copy()
    for rows, cols, vals, seg in packed:
        if cols is None:
            continue

        def body(lo, hi, rows=rows, cols=cols, vals=vals, seg=seg):
            e0, e1 = int(seg[lo]), int(seg[hi])
            prod = vals[e0:e1] * x[cols[e0:e1]]
            x[rows[lo:hi]] = b[rows[lo:hi]] - np.add.reduceat(prod, seg[lo:hi] - e0)

        _run_chunks(body, rows.size, workers)
    return x


class PortApply:
    """numpy port of apply_preconditioner on C-oracle factors."""

    def __init__(self, cf: coracle.CFactors, workers=1):
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
        self.workers = workers

    def __call__(self, b):
        y = _solve(self.lo, b, self.workers)
        z = np.empty_like(y)
        yb, zb = y.reshape(self.n, self.bs, 1), z.reshape(self.n, self.bs, 1)

        def body(lo, hi):
            np.matmul(self.dinv[lo:hi], yb[lo:hi], out=zb[lo:hi])

        _run_chunks(body, self.n, self.workers)
        return _solve(self.up, z, self.workers)


class PortSpmv:
    """numpy port of spmv (sparse.py:278-301) on the point expansion of A."""

    def __init__(self, n, bs, rp, ci, vals, workers=1):
        self.rp, self.ci, self.v = orc.csr_expand(n, bs, rp, ci, vals)
        self.m = n * bs
        self.workers = workers

    def __call__(self, x):
        y = np.zeros(self.m)
        rp, ci, v = self.rp, self.ci, self.v

        def body(lo, hi):
            e0, e1 = int(rp[lo]), int(rp[hi])
            if e1 > e0:
                starts = rp[lo:hi] - e0
                nz = np.diff(rp[lo:hi + 1]) > 0
                s = np.add.reduceat(v[e0:e1] * x[ci[e0:e1]], starts[nz])
                y[lo:hi][nz] = s

        _run_chunks(body, self.m, self.workers)
        return y


def apply_bytes(n, bs, nl, nu):
    return 8 * bs * bs * (nl + nu + n) + 4 * (nl + nu) + 8 * (n + 1) + 32 * bs * n


_LAST = {}


def _system(nx, bs, k, seed=0):
    """(synthetic module, matrix arrays, C-oracle factors); the last one is kept
    (the apply baseline and the solve of the same config share it)."""
    key = (nx, bs, k, seed)
    if key not in _LAST:
        _LAST.clear()
        synth = _synthetic()
        n, bs, rp, ci, vals = synth.reservoir_block_grid(nx, nx, nx, bs, seed=seed)
        cf = coracle.CFactors(n, bs, rp, ci, vals, k)
        _LAST[key] = (synth, (n, bs, rp, ci, vals), cf)
    return _LAST[key]


def measure(nx, bs, k, steps=3, warmup=1, seed=0, workers=None):
    """Time the apply port on an nx^3 system with workers = 1 and = all cores;
    GB/s of algorithmic apply bytes.  ``value`` is the faster mode."""
    cores, desc = host_cores()
    t0 = time.perf_counter()
    _, (n, bs, rp, ci, vals), cf = _system(nx, bs, k, seed)
    t_setup = time.perf_counter() - t0
    B = apply_bytes(n, bs, cf.nl, cf.nu)
    b = np.random.default_rng(1).standard_normal(n * bs)
    rows = {}
    for w in (workers if workers else sorted({1, cores})):
        port = PortApply(cf, workers=w)
        for _ in range(warmup):
            port(b)
        t0 = time.perf_counter()
        for _ in range(steps):
            port(b)
        dt = (time.perf_counter() - t0) / steps
        rows[w] = {"workers": w, "ms_per_apply": dt * 1e3, "GBps": B / dt / 1e9}
    best = min(rows.values(), key=lambda r: r["ms_per_apply"])
    return {
        "GBps": best["GBps"], "ms_per_apply": best["ms_per_apply"], "cores": best["workers"], "kind": "port",
        "host": desc, "host_cpus": cores, "rows": list(rows.values()), "bytes": B,
        "sample": (f"numpy port of the reference apply (trisolve.py:121-182) on {nx}^3 b{bs} ILU({k}), "
                   f"{steps} applies after {warmup} warm-up per mode; workers=" +
                   ", ".join(f"{r['workers']}: {r['ms_per_apply']:.1f} ms" for r in rows.values()) +
                   f"; value = the faster mode; untimed C-oracle setup {t_setup:.1f} s; host: {desc}"),
    }


def time_to_solution(nx, bs, k, solver, its_full=None, max_measured=None, workers=1, seed=0):
    """The reference solve (b = A 1, x0 = 0, rel tol 1e-6) with the port operators.

    Runs to convergence when ``max_measured`` is None; otherwise times
    ``max_measured`` iterations and projects to ``its_full`` iterations (the
    count the GPU solve reported).  Setup (C oracle) is not timed.
    """
    synth, (n, bs, rp, ci, vals), cf = _system(nx, bs, k, seed)
    port = PortApply(cf, workers=workers)
    mv = PortSpmv(n, bs, rp, ci, vals, workers=workers)
    b = synth.ones_rhs(n, bs, rp, ci, vals)
    kw = {"rel_tol": 1e-6}
    if max_measured:
        kw["max_iters"] = int(max_measured)
    t0 = time.perf_counter()
    if solver == "bicgstab":
        _, its, conv, rel, _ = orc.bicgstab(mv, b, port, **kw)
    else:
        _, its, conv, rel, _ = orc.gmres(mv, b, port, restart=30, **kw)
    dt = time.perf_counter() - t0
    out = {"workers": workers, "iterations_run": int(its), "converged": bool(conv), "seconds_run": dt}
    if max_measured and not conv:
        per = dt / max(1, its)
        out["seconds"] = per * (its_full or its)
        out["projected_from"] = f"{its} timed iterations x {its_full} iterations"
    else:
        out["seconds"] = dt
    return out
