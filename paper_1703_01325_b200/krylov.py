"""Krylov solvers on the device: restarted GMRES (reference gmres.py) and BiCGSTAB (new).

Both loops run in libbiluk (``biluk_gmres`` / ``biluk_bicgstab``): BSR SpMV,
preconditioner apply and fused deterministic BLAS-1 reductions are CUDA
kernels; the host only reads the scalars its stopping tests need.

The preconditioner ``M`` is, as in the reference (gmres.py:85-87), optional:
* ``None``                    -- unpreconditioned;
* a ``BlockIlukFactors``      -- the device path (no host round trip);
* any callable ``v -> M^-1 v`` -- the reference's opaque callable, called with
  numpy vectors through a C callback (correct, but it crosses PCIe twice per
  application; pass the factors themselves for speed).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from time import perf_counter

import numpy as np

from . import _native as nat
from .device import alloc_bytes, enter, operator_for, to_device_f64, torch

__all__ = ["SolverConfig", "SolveStats", "gmres", "bicgstab", "bicgstab_batched"]

_RHS_MODES = ("ones-solution", "given")


# field -> (accepts, requirement): the reference's rules (gmres.py:36-46)
_CONFIG_RULES = {
    "restart": (lambda v: v >= 1, "an integer >= 1"),
    "max_iters": (lambda v: v >= 1, "an integer >= 1"),
    "rel_tol": (lambda v: v > 0.0, "a positive number"),   # (NaN fails too)
    "abs_tol": (lambda v: v > 0.0, "a positive number"),
    "rhs_mode": (lambda v: v in _RHS_MODES, f"one of {_RHS_MODES}"),
}


@dataclass
class SolverConfig:
    """Solver settings with the reference's fields and defaults (gmres.py:23-35);
    every field is checked against `_CONFIG_RULES` (ValueError naming it)."""

    restart: int = 20
    max_iters: int = 10000
    rel_tol: float = 1e-6
    abs_tol: float = 1e-30
    rhs_mode: str = "ones-solution"

    def __post_init__(self):
        for name, (accepts, requirement) in _CONFIG_RULES.items():
            value = getattr(self, name)
            if not accepts(value):
                raise ValueError(f"SolverConfig.{name} = {value!r}: must be {requirement}")


@dataclass
class SolveStats:
    """Iteration and residual accounting for one solve (reference gmres.py:49-65)."""

    iterations: int = 0
    converged: bool = False
    final_relative_residual: float = math.inf
    residual_history: list = field(default_factory=list)
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0


def _precond_args(M, length):
    """(plan handle, C callback, keep-alive) for the three kinds of M."""
    from .factor import BlockIlukFactors
    if M is None:
        return None, nat.PRECOND_FN(0), None
    if isinstance(M, BlockIlukFactors):
        if M.n * M.bs != length:
            raise ValueError("preconditioner dimension does not match the matrix")
        return M.handle, nat.PRECOND_FN(0), None
    if not callable(M):
        raise TypeError("M must be None, BlockIlukFactors or a callable")
    t = torch()
    caught = []   # an exception raised by M, re-raised once the C call has returned

    def _cb(user, din, dout, stream):
        try:
            src = _DevView(din, length)
            v = t.as_tensor(src, device="cuda").cpu().numpy()
            res = np.asarray(M(v), dtype=np.float64)
            if res.shape != (length,):
                caught.append(ValueError(f"preconditioner returned shape {res.shape}, expected ({length},)"))
                return nat.EARG
            t.as_tensor(_DevView(dout, length), device="cuda").copy_(t.from_numpy(res))
            return nat.OK
        except Exception as exc:   # the C side stops the solve; the exception is re-raised in Python
            caught.append(exc)
            return nat.ECUDA
    fn = nat.PRECOND_FN(_cb)
    return None, fn, (fn, caught)


class _DevView:
    """__cuda_array_interface__ over a raw device pointer (no copy)."""

    def __init__(self, p, length):
        self.__cuda_array_interface__ = {"shape": (length,), "typestr": "<f8", "data": (int(p), False),
                                         "version": 3, "strides": None}


def _solve(kind, a, b, M, cfg, restart):
    cfg = SolverConfig() if cfg is None else cfg
    t0 = perf_counter()
    t = torch()
    op = operator_for(a)
    if op.n != op.ncols:
        raise ValueError(f"{kind} requires a square matrix")
    length = op.n * op.bs
    on_device = isinstance(b, t.Tensor) and b.is_cuda
    if not on_device:
        b = np.asarray(b, dtype=np.float64)
        if b.shape != (length,):
            raise ValueError(f"right-hand side length {b.shape} does not match n={length}")
    elif b.numel() != length:
        raise ValueError(f"right-hand side length {tuple(b.shape)} does not match n={length}")
    plan, cb, keep = _precond_args(M, length)
    stream = enter()
    bd = to_device_f64(b)
    x = t.empty(length, dtype=t.float64, device="cuda")
    L = nat.lib()
    work, workp = alloc_bytes(L.biluk_krylov_workspace_bytes(length, restart if kind == "gmres" else 0))
    stats = (ctypes.c_double * 4)()
    cap = cfg.max_iters + 2 * (cfg.max_iters // max(1, restart) + 2) + 16
    hist = np.zeros(cap)
    hist_p = hist.ctypes.data_as(nat.P_dbl)
    if kind == "gmres":
        rc = L.biluk_gmres(op.handle, plan, cb, None, bd.data_ptr(), x.data_ptr(), workp, int(cfg.restart),
                           int(cfg.max_iters), float(cfg.rel_tol), float(cfg.abs_tol), stats, hist_p, cap, stream)
    else:
        rc = L.biluk_bicgstab(op.handle, plan, cb, None, bd.data_ptr(), x.data_ptr(), workp, int(cfg.max_iters),
                              float(cfg.rel_tol), stats, hist_p, cap, stream)
    if keep is not None and keep[1]:
        raise keep[1][0]
    del keep
    nat.check(rc, stage=kind)
    st = SolveStats()
    st.iterations = int(stats[0])
    st.converged = bool(stats[1])
    st.final_relative_residual = float(stats[2])
    st.residual_history = hist[:min(int(stats[3]), cap)].tolist()
    out = x if on_device else x.cpu().numpy()
    st.solve_seconds = perf_counter() - t0
    return out, st


def gmres(a, b, M=None, cfg=None, workers=1):
    """Restarted GMRES(m), left preconditioned (drop-in for reference gmres.py:76-186).

    Same stopping logic: monitored ``||M^-1 r|| / ||M^-1 b||`` with true
    residual verification and target tightening; ``iterations`` counts Arnoldi
    steps.  Returns ``(x, SolveStats)``; ``x`` is numpy unless ``b`` is a CUDA
    tensor.  ``workers`` is accepted and ignored.
    """
    cfg = SolverConfig() if cfg is None else cfg
    return _solve("gmres", a, b, M, cfg, int(cfg.restart))


def bicgstab(a, b, M=None, cfg=None, workers=1):
    """Right-preconditioned BiCGSTAB, x0 = 0 (contract: oracle/iluk_oracle.py:bicgstab).

    Stops when ||r|| / ||b|| <= rel_tol, tested at the half step s and at the
    full step (a half-step exit counts as a full iteration); reports the true
    residual.  ``cfg.restart`` is ignored.
    """
    cfg = SolverConfig() if cfg is None else cfg
    return _solve("bicgstab", a, b, M, cfg, 0)


def bicgstab_batched(a, b, segments=None, M=None, cfg=None):
    """BiCGSTAB over independent systems packed as one block-diagonal matrix.

    ``a`` is the batch operator (e.g. ``sparse.block_diagonal(mats)``), ``M``
    its preconditioner (``build_preconditioner(a, k)`` -- ILU(k) decouples over
    the diagonal blocks), ``segments`` the block-row offsets of the systems
    (``[0, n_0, n_0 + n_1, ..., n]``; default ``a.batch_segments``, which
    ``block_diagonal`` sets; explicit segments are checked not to couple).
    Each system iterates as :func:`bicgstab` would on it alone (its own
    scalars and stopping tests; the result is the single solve's up to the
    preconditioner's rounding) while every SpMV and preconditioner apply covers
    the whole batch in one launch.  Returns ``(x, [SolveStats per
    system])``; ``x`` is numpy unless ``b`` is a CUDA tensor.  Residual
    histories are not kept.
    """
    cfg = SolverConfig() if cfg is None else cfg
    t0 = perf_counter()
    t = torch()
    trusted = segments is None   # block_diagonal output: no coupling by construction
    if trusted:
        segments = getattr(a, "batch_segments", None)
        if segments is None:
            raise ValueError("segments required (the matrix does not come from block_diagonal)")
    seg = np.ascontiguousarray(np.asarray(segments, dtype=np.int64))
    if seg.ndim != 1 or seg.size < 2:
        raise ValueError("segments must hold at least two offsets")
    op = operator_for(a)
    if op.n != op.ncols:
        raise ValueError("bicgstab requires a square matrix")
    if seg[0] != 0 or seg[-1] != op.n or np.any(np.diff(seg) < 0):
        raise ValueError("segments must be non-decreasing offsets from 0 to n")
    rp = getattr(a, "row_ptr", None) if not trusted else None
    if rp is not None:   # the systems must not couple: every entry stays inside its row's segment
        rp = np.asarray(rp, dtype=np.int64)
        ci = np.asarray(a.col_idx, dtype=np.int64)
        rows = np.repeat(np.arange(rp.size - 1, dtype=np.int64), np.diff(rp))
        if np.any(np.searchsorted(seg, rows, side="right") != np.searchsorted(seg, ci, side="right")):
            raise ValueError("matrix couples two batch systems (not block diagonal over segments)")
    length = op.n * op.bs
    on_device = isinstance(b, t.Tensor) and b.is_cuda
    if not on_device:
        b = np.asarray(b, dtype=np.float64)
        if b.shape != (length,):
            raise ValueError(f"right-hand side length {b.shape} does not match n={length}")
    elif b.numel() != length:
        raise ValueError(f"right-hand side length {tuple(b.shape)} does not match n={length}")
    plan, cb, keep = _precond_args(M, length)
    stream = enter()
    bd = to_device_f64(b)
    x = t.empty(length, dtype=t.float64, device="cuda")
    L = nat.lib()
    nsys = seg.size - 1
    work, workp = alloc_bytes(L.biluk_krylov_batched_workspace_bytes(length, nsys))
    stats = (ctypes.c_double * (4 * nsys))()
    rc = L.biluk_bicgstab_batched(op.handle, plan, cb, None, nsys, seg.ctypes.data_as(nat.P_i64), bd.data_ptr(),
                                  x.data_ptr(), workp, int(cfg.max_iters), float(cfg.rel_tol), stats, stream)
    if keep is not None and keep[1]:
        raise keep[1][0]
    del keep
    nat.check(rc, stage="bicgstab_batched")
    out = x if on_device else x.cpu().numpy()
    dt = perf_counter() - t0
    res = []
    for i in range(nsys):
        st = SolveStats()
        st.iterations = int(stats[4 * i])
        st.converged = bool(stats[4 * i + 1])
        st.final_relative_residual = float(stats[4 * i + 2])
        st.solve_seconds = dt
        res.append(st)
    return out, res
