"""build_preconditioner and the factor container (reference factor.py:208-323).

Pipeline (the reference stages, factor.py:302-323, with the same stage
names in error messages):

* extract-pattern + symbolic-phase + schedules: host C++ in libbiluk
  (``biluk_plan_create``) -- exact integer work;
* materialize + factorize + split: device kernels (``biluk_plan_factor``):
  level-scheduled block ILU(0) with the U = D U' split fused behind it, and
  the factors packed straight into the level-ordered tile records that the
  persistent triangular sweeps stream.

``BlockIlukFactors`` keeps the factors on the device.  The reference's
parity accessors (``L``, ``dinv``, ``uprime``, ``lower_op``, ``upper_op``,
``lower_schedule``, ``upper_schedule``) are materialized lazily on the host
from the device factors, in the reference layouts.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _native as nat
from .device import alloc_bytes, enter, to_device_f64
from .errors import FactorizationError, SingularBlockError, StructuralError
from .sparse import BcsrMatrix, CsrMatrix, PatternMatrix, as_bsr, csr_expand

__all__ = ["BlockIlukFactors", "block_ilu0_factorize", "block_invert", "build_preconditioner", "materialize",
           "point_ilu0_factorize", "split_ldu", "symbolic_phase"]

_INFO_KEYS = ("n", "bs", "k", "nnzb_a", "nnzb_p", "nL", "nU", "levels_L", "levels_U", "tiles_L", "tiles_U",
              "rows_per_tile", "workspace_bytes", "apply_bytes", "spmv_bytes", "sweep_ctas", "sweep_warps",
              "sweep_stages", "stage_bytes", "max_slots", "engine", "parts", "records", "est_ns", "record_bytes",
              "fetched_entries", "partition", "split_y", "split_z")


def symbolic_phase(pattern, k):
    """ILU(k) level-of-fill pattern (reference symbolic.py:27-72), computed by libbiluk.

    Bit-exact with the reference.  ``pattern`` is a PatternMatrix (ours or the
    reference's); returns a PatternMatrix.
    """
    k = int(k)
    if k < 0:
        raise ValueError("fill level k must be nonnegative")
    n = int(pattern.n)
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in pattern.rows])
    ci = np.fromiter((j for r in pattern.rows for j in r), dtype=np.int64, count=int(rp[-1]))
    L = nat.lib()
    h = ctypes.c_void_p()
    err = ctypes.c_int64(-1)
    nat.check(L.biluk_symbolic(n, nat.ptr(rp), nat.ptr(ci), k, ctypes.byref(h), ctypes.byref(err)))
    try:
        nnz = L.biluk_pattern_nnz(h)
        orp = np.zeros(n + 1, np.int64)
        oci = np.zeros(nnz, np.int64)
        nat.check(L.biluk_pattern_copy(h, nat.ptr(orp), nat.ptr(oci)))
    finally:
        L.biluk_pattern_free(h)
    return PatternMatrix.from_csr_arrays(n, orp, oci)


class BlockIlukFactors:
    """Factor triple (L, D^-1, U') on the device, ready for repeated application.

    Mirrors reference factor.py:208-227: ``L`` and ``uprime`` (BcsrMatrix,
    column-major blocks), ``dinv`` ((n, bs, bs) row-major), ``bs``, ``n``,
    ``lower_op``/``upper_op`` (point-wise zero-dropped triangles) and their
    ``lower_schedule``/``upper_schedule`` -- all host views built on first
    access from the device factors.
    """

    def __init__(self, handle, ws, wsp, a_dev, bs, n, k):
        self._h = handle
        self._ws = ws
        self._wsp = wsp
        self._a_dev = a_dev
        self.bs = bs
        self.n = n
        self.k = k
        self._cache = {}
        self._finalizer = weakref.finalize(self, nat.lib().biluk_plan_destroy, handle)

    # ---- device side -------------------------------------------------------
    @property
    def handle(self):
        return self._h

    @property
    def info(self):
        buf = (ctypes.c_int64 * len(_INFO_KEYS))()
        nat.check(nat.lib().biluk_plan_info(self._h, buf, len(_INFO_KEYS)))
        return dict(zip(_INFO_KEYS, list(buf)))

    def apply(self, b, out=None):
        from .trisolve import apply_preconditioner
        return apply_preconditioner(self, b, out=out)

    def tune(self, **knobs):
        """Sweep-kernel knobs (gap, coarse_sleep_ns, fine_sleep_ns); results never depend on them."""
        for key, val in knobs.items():
            nat.check(nat.lib().biluk_plan_tune(self._h, key.encode(), int(val)))
        return self

    def tile_levels(self):
        """Combined dependency level of every sweep tile (L tiles, then U' tiles)."""
        inf = self.info
        out = np.zeros(inf["tiles_L"] + inf["tiles_U"], np.int32)
        nat.check(nat.lib().biluk_plan_tile_levels(self._h, nat.ptr(out)))
        return out

    def set_sweep_timing(self, enable=True):
        """Diagnostics: CUDA events around the sweep launch of every later apply."""
        nat.check(nat.lib().biluk_plan_set_timing(self._h, 1 if enable else 0))

    def sweep_ms(self):
        """Duration of the last apply's sweep kernel (waits for it); needs set_sweep_timing."""
        ms = ctypes.c_float()
        nat.check(nat.lib().biluk_plan_sweep_ms(self._h, ctypes.byref(ms)))
        return float(ms.value)

    def set_trace(self, enable=True):
        """Diagnostics: record per-tile globaltimer stamps on later applies; returns the (T, 4) buffer."""
        if not enable:
            nat.check(nat.lib().biluk_plan_set_trace(self._h, None))
            self._trace = None
            return None
        from .device import torch
        t = torch()
        inf = self.info
        if inf["engine"] >= 1:   # partitioned / grid sweep: 8 stamps per record (csrc/psweep.cu, gsweep.cu)
            self._trace = t.zeros((inf["records"] + 16384, 8), dtype=t.int64, device="cuda")
        else:
            self._trace = t.zeros((inf["tiles_L"] + inf["tiles_U"], 4), dtype=t.int64, device="cuda")
        nat.check(nat.lib().biluk_plan_set_trace(self._h, self._trace.data_ptr()))
        return self._trace

    def status(self):
        """Synchronise and raise if a device dependency wait timed out."""
        nat.check(nat.lib().biluk_plan_status(self._h, enter()), stage="apply")

    # ---- reference parity views (host, lazy) -----------------------------------
    def _factors(self):
        if "f" not in self._cache:
            inf = self.info
            n, bs, nL, nU = inf["n"], inf["bs"], inf["nL"], inf["nU"]
            lrp = np.zeros(n + 1, np.int64)
            lci = np.zeros(nL, np.int64)
            lv = np.zeros(nL * bs * bs)
            dinv = np.zeros((n, bs, bs))
            urp = np.zeros(n + 1, np.int64)
            uci = np.zeros(nU, np.int64)
            uv = np.zeros(nU * bs * bs)
            stream = enter()
            nat.check(nat.lib().biluk_plan_copy_factors(self._h, nat.ptr(lrp), nat.ptr(lci), nat.ptr(lv),
                                                        nat.ptr(dinv), nat.ptr(urp), nat.ptr(uci), nat.ptr(uv),
                                                        stream))
            self._cache["f"] = (BcsrMatrix(bs, n, n, lrp, lci, lv), dinv, BcsrMatrix(bs, n, n, urp, uci, uv))
        return self._cache["f"]

    @property
    def L(self):
        return self._factors()[0]

    @property
    def dinv(self):
        return self._factors()[1]

    @property
    def uprime(self):
        return self._factors()[2]

    def _operand(self, which):
        from .trisolve import TriangularOperand, build_level_schedule
        key = "op_" + which
        if key not in self._cache:
            mat = self.L if which == "lower" else self.uprime
            op = TriangularOperand(csr_expand(mat), which)
            self._cache[key] = (op, build_level_schedule(op))
        return self._cache[key]

    @property
    def lower_op(self):
        return self._operand("lower")[0]

    @property
    def lower_schedule(self):
        return self._operand("lower")[1]

    @property
    def upper_op(self):
        return self._operand("upper")[0]

    @property
    def upper_schedule(self):
        return self._operand("upper")[1]

    def __repr__(self):
        return f"BlockIlukFactors(n={self.n}, bs={self.bs}, k={self.k})"


def _new_plan(bs, n, rp, ci, k, flags=0):
    """(handle, workspace tensor, aligned pointer) of a bound plan; raises with the
    C status mapped (the caller adds the stage text)."""
    L = nat.lib()
    h = ctypes.c_void_p()
    err = ctypes.c_int64(-1)
    rc = L.biluk_plan_create_ex(bs, n, nat.ptr(rp), nat.ptr(ci), int(k), int(flags), ctypes.byref(h),
                                ctypes.byref(err))
    if rc != nat.OK:
        return rc, int(err.value), None
    try:
        stream = enter()
        nbytes = L.biluk_plan_workspace_bytes(h)
        ws, wsp = alloc_bytes(nbytes)
        nat.check(L.biluk_plan_bind(h, wsp, nbytes, stream), stage="materialize")
    except BaseException:
        L.biluk_plan_destroy(h)
        raise
    return nat.OK, -1, (h, ws, wsp)


def _diag_slots(n, rp, ci):
    """Slot of each row's diagonal entry, or the first row without one (-1, i)."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    hit = np.flatnonzero(ci == rows)
    has = np.zeros(n, bool)
    has[rows[hit]] = True
    if not has.all():
        return None, int(np.flatnonzero(~has)[0])
    slot = np.empty(n, np.int64)
    slot[rows[hit]] = hit
    return slot, -1


def block_invert(b):
    """Inverse of a small dense block by LU with partial pivoting (reference factor.py:38-70).

    Runs on the GPU (``biluk_block_invert``); also accepts a stack ``(m, bs, bs)``
    and then inverts every block.  Raises ``SingularBlockError`` when a pivot
    falls below 1e-13 times the block's largest magnitude or the block is all
    zero.  Block sizes 1..8.
    """
    from .device import torch
    arr = np.asarray(b, dtype=np.float64)
    if arr.ndim not in (2, 3) or arr.shape[-1] != arr.shape[-2]:
        raise StructuralError("block_invert needs a square block")
    bs = arr.shape[-1]
    stack = arr.reshape(-1, bs, bs)
    if stack.shape[0] == 0:
        return arr.copy()
    t = torch()
    stream = enter()
    din = t.from_numpy(np.ascontiguousarray(stack)).cuda()
    dout = t.empty_like(din)
    bad = ctypes.c_int64(-1)
    rc = nat.lib().biluk_block_invert(bs, stack.shape[0], din.data_ptr(), dout.data_ptr(), ctypes.byref(bad), stream)
    if rc == nat.ESINGULAR:
        where = "" if arr.ndim == 2 else f" (block {bad.value})"
        raise SingularBlockError(f"singular block: pivot below 1e-13 of the largest magnitude{where}")
    nat.check(rc, stage="block_invert")
    return dout.cpu().numpy().reshape(arr.shape)


def materialize(a, pprime):
    """Copy of ``a`` with pattern exactly ``pprime``, zeros at the added
    positions (reference factor.py:83-121).

    ``a`` is a BcsrMatrix (zero blocks backfilled) or a CsrMatrix; every
    stored position of ``a`` must appear in ``pprime`` (StructuralError
    otherwise).  The slot map is integer host work; the values are scattered on
    the GPU (``biluk_scatter_blocks``).
    """
    from .device import torch
    bs, n, m, rp, ci, vals = as_bsr(a)
    if m != n:
        raise StructuralError("materialize requires a square matrix")
    if int(pprime.n) != n:
        raise StructuralError(f"pattern dimension {pprime.n} does not match matrix dimension {n}")
    prp, pci = pprime.to_csr_arrays() if hasattr(pprime, "to_csr_arrays") else \
        PatternMatrix(pprime.n, pprime.rows).to_csr_arrays()
    # slot of every stored (i, j) of a inside pprime: keys i*n + j are sorted in both
    arow = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    pkey = np.repeat(np.arange(n, dtype=np.int64), np.diff(prp)) * max(n, 1) + pci
    akey = arow * max(n, 1) + ci
    pos = np.searchsorted(pkey, akey)
    bad = (pos >= pkey.size) | (pkey[np.minimum(pos, max(pkey.size - 1, 0))] != akey) if akey.size else \
        np.zeros(0, bool)
    if bad.any():
        t0 = int(np.flatnonzero(bad)[0])
        raise StructuralError(f"pattern is missing stored position ({int(arow[t0])}, {int(ci[t0])})")
    bs2 = bs * bs
    out = np.zeros(int(prp[-1]) * bs2)
    if akey.size:
        t = torch()
        stream = enter()
        dsrc = to_device_f64(vals)
        dmap = t.from_numpy(np.ascontiguousarray(pos, np.int64)).cuda()
        ddst = t.zeros(out.size, dtype=t.float64, device="cuda")
        nat.check(nat.lib().biluk_scatter_blocks(bs2, akey.size, dmap.data_ptr(), dsrc.data_ptr(), ddst.data_ptr(),
                                                 stream), stage="materialize")
        out = ddst.cpu().numpy()
    if hasattr(a, "block_size"):
        return BcsrMatrix(bs, n, n, prp, pci, out)
    return CsrMatrix(n, n, prp, pci, out)


def _ilu0_in_place(aprime, point):
    """Stages materialize + factorize of an ILU(0) on aprime's own pattern, on the GPU."""
    bs, n, m, rp, ci, vals = as_bsr(aprime)
    if n != m:
        raise StructuralError("factorization requires a square matrix")
    slot, missing = _diag_slots(n, rp, ci)
    if slot is None:
        raise StructuralError(f"row {missing} has no diagonal entry" if point else
                              f"block row {missing} has no diagonal block")
    rc, erow, plan = _new_plan(bs, n, rp, ci, 0, flags=1)   # BILUK_PLAN_FACTOR_ONLY
    nat.check(rc, stage="factorize", row=erow)
    h, ws, wsp = plan
    L = nat.lib()
    try:
        from .device import torch
        t = torch()
        stream = enter()
        dvals = to_device_f64(vals)
        dout = t.empty_like(dvals)
        err = ctypes.c_int64(-1)
        rc = L.biluk_plan_factor_lu(h, dvals.data_ptr(), dout.data_ptr(), stream, ctypes.byref(err))
        if rc == nat.EZEROPIVOT:
            raise FactorizationError(f"zero pivot at row {err.value}", row=int(err.value))
        if rc == nat.ESINGULAR:
            raise SingularBlockError(f"singular diagonal block at row {err.value}", row=int(err.value))
        nat.check(rc, stage="factorize")
        aprime.values[...] = dout.cpu().numpy().reshape(aprime.values.shape)
    finally:
        L.biluk_plan_destroy(h)
    return aprime


def point_ilu0_factorize(aprime):
    """ILU(0) on the stored pattern of a CsrMatrix, overwriting its values in
    place (reference factor.py:151-162): unit-lower multipliers strictly below
    the diagonal, the upper factor with its diagonal on and above it.  Runs the
    level-scheduled factorization kernel on the GPU; a pivot below 1e-300
    raises ``FactorizationError`` with ``.row``."""
    if aprime.num_rows != aprime.num_cols:
        raise StructuralError("factorization requires a square matrix")
    return _ilu0_in_place(aprime, point=True)


def block_ilu0_factorize(aprime):
    """Block ILU(0) on the stored block pattern of a BcsrMatrix, in place
    (reference factor.py:165-205), on the GPU.  A_ip <- A_ip D_p^-1, then
    A_ij -= A_ip A_pj over the stored slots; U stays unscaled.  Block size one
    is the point kernel.  A singular diagonal block raises
    ``SingularBlockError`` with ``.row``."""
    if aprime.num_block_rows != aprime.num_block_cols:
        raise StructuralError("factorization requires a square matrix")
    return _ilu0_in_place(aprime, point=aprime.block_size == 1)


def split_ldu(f):
    """Split an in-place factored block matrix into BlockIlukFactors (reference
    factor.py:230-289): L = the strictly lower blocks, D_i^-1 =
    block_invert(U_ii), U'_ij = D_i^-1 U_ij.  The factors live on the GPU and
    are ready for ``apply_preconditioner``."""
    bs, n, m, rp, ci, vals = as_bsr(f)
    if n != m:
        raise StructuralError("split requires a square matrix")
    slot, missing = _diag_slots(n, rp, ci)
    if slot is None:
        raise StructuralError(f"block row {missing} has no diagonal block")
    rc, erow, plan = _new_plan(bs, n, rp, ci, 0)
    nat.check(rc, stage="split", row=erow)
    h, ws, wsp = plan
    L = nat.lib()
    try:
        stream = enter()
        dvals = to_device_f64(vals)
        err = ctypes.c_int64(-1)
        rc = L.biluk_plan_load_factored(h, dvals.data_ptr(), stream, ctypes.byref(err))
        if rc == nat.ESINGULAR:
            raise SingularBlockError(f"singular diagonal block at row {err.value}", row=int(err.value))
        nat.check(rc, stage="split")
    except BaseException:
        L.biluk_plan_destroy(h)
        raise
    return BlockIlukFactors(h, ws, wsp, dvals, bs, n, 0)


def build_preconditioner(a, k):
    """Two-phase block ILU(k) on the GPU; drop-in for reference factor.py:302-323.

    ``a`` is a BcsrMatrix or CsrMatrix (ours or the reference's; a point CSR
    matrix is block size one).  The input is never modified.  Errors carry the
    reference stage names: ``StructuralError("symbolic-phase: ...")``,
    ``SingularBlockError("factorize: ...", row=i)`` (bs > 1) and
    ``FactorizationError("factorize: ...", row=i)`` (bs == 1 zero pivot).
    """
    bs, n, m, rp, ci, vals = as_bsr(a)
    if n != m:
        raise StructuralError("extract-pattern: pattern extraction requires a square matrix")
    if int(k) < 0:
        raise ValueError("fill level k must be nonnegative")
    L = nat.lib()
    h = ctypes.c_void_p()
    err = ctypes.c_int64(-1)
    rc = L.biluk_plan_create(bs, n, nat.ptr(rp), nat.ptr(ci), int(k), ctypes.byref(h), ctypes.byref(err))
    nat.check(rc, stage="symbolic-phase")
    try:
        stream = enter()
        nbytes = L.biluk_plan_workspace_bytes(h)
        ws, wsp = alloc_bytes(nbytes)
        nat.check(L.biluk_plan_bind(h, wsp, nbytes, stream), stage="materialize")
        a_dev = to_device_f64(vals)
        rc = L.biluk_plan_factor(h, a_dev.data_ptr(), stream, ctypes.byref(err))
        nat.check(rc, stage="factorize", row=int(err.value))
    except BaseException:
        L.biluk_plan_destroy(h)
        raise
    return BlockIlukFactors(h, ws, wsp, a_dev, bs, n, int(k))


__all__ += ["FactorizationError"]
