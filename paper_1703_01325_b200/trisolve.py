"""apply_preconditioner and the level-schedule views (reference trisolve.py).

``apply_preconditioner(f, b)`` runs Alg. 7 (L y = b, z = D^-1 y, U' x = z) as
ONE persistent sync-free CUDA kernel (``biluk_plan_apply``): block rows are
streamed in level order, each warp owns 32 block rows of a level, and a row
waits only for the rows it reads (no barrier per level, no launch per level).
The reference runs the same three stages point-wise on zero-dropped
expansions with one fork-join per level (trisolve.py:121-182); results agree
to rounding (<= 1e-12 relative), see tests/test_gpu_parity.py.

``TriangularOperand`` / ``LevelSchedule`` / ``build_level_schedule`` reproduce
the reference's point-wise schedule objects exactly (integer parity); the
level computation is libbiluk's host C++ (``biluk_level_schedule``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .device import enter, to_device_f64, torch
from .errors import StructuralError
from .sparse import CsrMatrix

__all__ = ["TriangularOperand", "LevelSchedule", "strict_triangle", "build_level_schedule", "apply_preconditioner",
           "apply_preconditioner_many", "solve_unit_triangular", "apply_block_diagonal"]


class TriangularOperand:
    """Strictly lower or strictly upper CSR matrix with an implied unit diagonal (trisolve.py:28-48)."""

    def __init__(self, matrix, orientation):
        if orientation not in ("lower", "upper"):
            raise ValueError("orientation must be 'lower' or 'upper'")
        if matrix.num_rows != matrix.num_cols:
            raise StructuralError("triangular operand must be square")
        erow = np.repeat(np.arange(matrix.num_rows, dtype=np.int64), np.diff(matrix.row_ptr))
        ok = matrix.col_idx < erow if orientation == "lower" else matrix.col_idx > erow
        if not np.all(ok):
            raise StructuralError(f"entry on or across the diagonal in a {orientation} operand")
        self.matrix = matrix
        self.orientation = orientation

    @property
    def n(self):
        return self.matrix.num_rows


def strict_triangle(a, orientation):
    """TriangularOperand of the strictly lower / upper part of a CSR matrix (trisolve.py:51-58)."""
    erow = np.repeat(np.arange(a.num_rows, dtype=np.int64), np.diff(a.row_ptr))
    keep = a.col_idx < erow if orientation == "lower" else a.col_idx > erow
    rp = np.zeros(a.num_rows + 1, np.int64)
    np.cumsum(np.bincount(erow[keep], minlength=a.num_rows), out=rp[1:])
    return TriangularOperand(CsrMatrix(a.num_rows, a.num_cols, rp, a.col_idx[keep], a.values[keep]), orientation)


class LevelSchedule:
    """Rows grouped by Eq. (4) dependency level (trisolve.py:61-80).

    ``levels[l]`` lists the rows of level l+1 in ascending order,
    ``level_of_row`` is 1-based, ``num_levels`` the depth.
    """

    def __init__(self, level_of_row, levels, num_levels, orientation, source):
        self.level_of_row = level_of_row
        self.levels = levels
        self.num_levels = num_levels
        self.orientation = orientation
        self._source = source

    def __repr__(self):
        return f"LevelSchedule({self.orientation}, n={self.level_of_row.size}, levels={self.num_levels})"


def build_level_schedule(t):
    """Eq. (4) levels of a triangular operand; exact parity with trisolve.py:98-118."""
    m = t.matrix
    n = int(m.num_rows)
    rp = np.ascontiguousarray(m.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(m.col_idx, dtype=np.int64)
    lev = np.zeros(n, np.int64)
    num = ctypes.c_int64(0)
    nat.check(nat.lib().biluk_level_schedule(n, nat.ptr(rp), nat.ptr(ci), 1 if t.orientation == "upper" else 0,
                                             nat.ptr(lev), ctypes.byref(num)))
    nlev = int(num.value)
    by = np.argsort(lev, kind="stable")
    counts = np.bincount(lev, minlength=nlev + 1)[1:]
    groups = np.split(by, np.cumsum(counts)[:-1]) if nlev else []
    return LevelSchedule(lev, groups, nlev, t.orientation, t)


def _unit_triangular_plan(t):
    """A GPU plan whose factored matrix is I + T: D = I and T as L (lower) or
    U' (upper), so its apply is (I + T)^-1 -- the sweep kernels run the solve."""
    from .factor import BlockIlukFactors, _new_plan
    m = t.matrix
    n = int(m.num_rows)
    rp = np.asarray(m.row_ptr, np.int64)
    ci = np.asarray(m.col_idx, np.int64)
    vals = np.asarray(m.values, np.float64)
    cnt = np.diff(rp)
    nrp = np.zeros(n + 1, np.int64)
    np.cumsum(cnt + 1, out=nrp[1:])
    # the diagonal goes after the row's entries (lower) or before them (upper)
    dpos = nrp[1:] - 1 if t.orientation == "lower" else nrp[:-1]
    nci = np.empty(int(nrp[-1]), np.int64)
    nv = np.empty(int(nrp[-1]))
    off = np.ones(int(nrp[-1]), bool)
    off[dpos] = False
    nci[dpos] = np.arange(n)
    nv[dpos] = 1.0
    nci[off] = ci
    nv[off] = vals
    rc, erow, plan = _new_plan(1, n, nrp, nci, 0)
    nat.check(rc, stage="solve_unit_triangular", row=erow)
    h, ws, wsp = plan
    dv = to_device_f64(nv)
    err = ctypes.c_int64(-1)
    try:
        nat.check(nat.lib().biluk_plan_load_factored(h, dv.data_ptr(), enter(), ctypes.byref(err)),
                  stage="solve_unit_triangular")
    except BaseException:
        nat.lib().biluk_plan_destroy(h)
        raise
    return BlockIlukFactors(h, ws, wsp, dv, 1, n, 0)


def solve_unit_triangular(t, schedule, b, workers=1):
    """Solve (I + T) x = b, T strictly triangular (reference trisolve.py:121-145).

    The unit diagonal means no divisions.  The schedule must have been built
    from ``t`` (StructuralError otherwise); ``workers`` never changes a bit of
    the result; ``b`` is left untouched.  Runs as the GPU sweep of a plan of
    I + T, built on first use and kept with the schedule (like the
    reference's packed levels, a snapshot of T's values).  numpy in -> numpy
    out; a CUDA tensor in -> a CUDA tensor out.
    """
    if getattr(schedule, "_source", None) is not t:
        raise StructuralError("schedule was not built from this operand")
    tt = torch()
    on_device = isinstance(b, tt.Tensor) and b.is_cuda
    if on_device:
        if b.numel() != t.n or b.dim() != 1:
            raise ValueError(f"right-hand side length {tuple(b.shape)} does not match n={t.n}")
    else:
        b = np.asarray(b, dtype=np.float64)
        if b.shape != (t.n,):
            raise ValueError(f"right-hand side length {b.shape} does not match n={t.n}")
    if t.n == 0:
        return b.clone() if on_device else b.copy()
    plan = getattr(schedule, "_b200_plan", None)
    if plan is None:
        plan = _unit_triangular_plan(t)
        schedule._b200_plan = plan
    return apply_preconditioner(plan, b)


def apply_block_diagonal(dinv, y, workers=1):
    """z with z_I = dinv[I] @ y_I for each block row I (reference trisolve.py:148-166).

    ``dinv`` is an (n, bs, bs) row-major stack; one small dense multiply per
    block row on the GPU (``biluk_block_diag_apply``).  numpy in -> numpy out.
    """
    t = torch()
    on_device = isinstance(y, t.Tensor) and y.is_cuda
    d = dinv if isinstance(dinv, t.Tensor) else np.asarray(dinv, dtype=np.float64)
    if d.ndim != 3 or d.shape[1] != d.shape[2]:
        raise ValueError("dinv must be an (n, bs, bs) stack")
    n, bs = int(d.shape[0]), int(d.shape[1])
    yv = y if on_device else np.asarray(y, dtype=np.float64)
    if tuple(yv.shape) != (n * bs,):
        raise ValueError(f"operand length {tuple(yv.shape)} does not match {n * bs}")
    stream = enter()
    dd = to_device_f64(d.reshape(-1) if isinstance(d, t.Tensor) else np.ascontiguousarray(d).reshape(-1))
    yd = to_device_f64(yv)
    z = t.empty(n * bs, dtype=t.float64, device="cuda")
    nat.check(nat.lib().biluk_block_diag_apply(bs, n, dd.data_ptr(), yd.data_ptr(), z.data_ptr(), stream),
              stage="apply_block_diagonal")
    return z if on_device else z.cpu().numpy()


def _check_out(out, length, bd):
    """``out`` must be a contiguous float64 CUDA vector of the right length on
    the current device, not overlapping the right-hand side."""
    t = torch()
    if not (isinstance(out, t.Tensor) and out.is_cuda):
        raise ValueError("out must be a CUDA tensor")
    if out.dtype != t.float64 or not out.is_contiguous() or out.numel() != length:
        raise ValueError(f"out must be a contiguous float64 vector of length {length}")
    if out.device.index != t.cuda.current_device():
        raise ValueError("out is on another device")
    lo, hi = out.data_ptr(), out.data_ptr() + 8 * length
    blo, bhi = bd.data_ptr(), bd.data_ptr() + 8 * length
    if lo < bhi and blo < hi:
        raise ValueError("output may not overlap the right-hand side")


def apply_preconditioner(f, b, workers=1, out=None):
    """x = U'^-1 D^-1 L^-1 b on the GPU (reference trisolve.py:169-182).

    ``b`` may be a numpy array (returns a new numpy array, like the reference)
    or a CUDA tensor (returns a CUDA tensor; asynchronous on the current
    stream).  ``workers`` is accepted for signature compatibility: the result
    never depends on it (nor on anything else -- the sweep is deterministic).
    """
    t = torch()
    length = f.n * f.bs
    on_device = isinstance(b, t.Tensor) and b.is_cuda
    if on_device:
        if b.numel() != length or b.dim() != 1:
            raise ValueError(f"right-hand side length {tuple(b.shape)} does not match {length}")
    else:
        b = np.asarray(b, dtype=np.float64)
        if b.shape != (length,):
            raise ValueError(f"right-hand side length {b.shape} does not match {length}")
    stream = enter()
    bd = to_device_f64(b)
    if out is not None:
        _check_out(out, length, bd)
    x = out if out is not None else t.empty(length, dtype=t.float64, device="cuda")
    nat.check(nat.lib().biluk_plan_apply(f.handle, bd.data_ptr(), x.data_ptr(), stream), stage="apply")
    if on_device:
        return x
    host = x.cpu().numpy()
    f.status()
    return host


def apply_preconditioner_many(f, rhs, out=None):
    """x_j = M^-1 b_j for k right-hand sides held in host memory, pipelined.

    ``rhs`` is a (k, n*bs) float64 array (pinned torch CPU tensor or numpy;
    numpy is staged once into pinned memory).  The copy in of b_{j+1} and the
    copy out of x_{j-1} run on their own streams while the sweep of b_j runs,
    so PCIe transfers in both directions overlap the device work; each x_j is
    exactly ``apply_preconditioner(f, b_j)``.  Returns a (k, n*bs) pinned CPU
    tensor (``out`` if given).
    """
    t = torch()
    length = f.n * f.bs
    if isinstance(rhs, t.Tensor):
        if rhs.is_cuda:
            raise ValueError("rhs must be in host memory (use apply_preconditioner for device tensors)")
        host = rhs if (rhs.is_pinned() and rhs.dtype == t.float64 and rhs.is_contiguous()) else \
            rhs.to(t.float64).contiguous().pin_memory()
    else:
        host = t.from_numpy(np.ascontiguousarray(rhs, dtype=np.float64)).pin_memory()
    if host.dim() != 2 or host.shape[1] != length:
        raise ValueError(f"right-hand sides {tuple(host.shape)} do not match (k, {length})")
    k = host.shape[0]
    res = out if out is not None else t.empty((k, length), dtype=t.float64).pin_memory()
    if tuple(res.shape) != (k, length) or res.is_cuda:
        raise ValueError("out must be a (k, n) host tensor")
    enter()
    comp = t.cuda.current_stream()
    s_in, s_out = t.cuda.Stream(), t.cuda.Stream()
    d_in = [t.empty(length, dtype=t.float64, device="cuda") for _ in range(2)]
    d_out = [t.empty(length, dtype=t.float64, device="cuda") for _ in range(2)]
    ev = {name: [t.cuda.Event() for _ in range(2)] for name in ("in_ready", "in_free", "out_ready", "out_free")}
    for j in range(k):
        u = j % 2
        with t.cuda.stream(s_in):
            if j >= 2:
                s_in.wait_event(ev["in_free"][u])
            d_in[u].copy_(host[j], non_blocking=True)
            ev["in_ready"][u].record(s_in)
        comp.wait_event(ev["in_ready"][u])
        if j >= 2:
            comp.wait_event(ev["out_free"][u])
        nat.check(nat.lib().biluk_plan_apply(f.handle, d_in[u].data_ptr(), d_out[u].data_ptr(), comp.cuda_stream),
                  stage="apply")
        ev["in_free"][u].record(comp)
        ev["out_ready"][u].record(comp)
        with t.cuda.stream(s_out):
            s_out.wait_event(ev["out_ready"][u])
            res[j].copy_(d_out[u], non_blocking=True)
            ev["out_free"][u].record(s_out)
    s_out.synchronize()   # after it every copy and sweep above has completed
    f.status()
    return res
