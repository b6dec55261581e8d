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
from .errors import FactorizationError, StructuralError
from .sparse import BcsrMatrix, PatternMatrix, as_bsr, csr_expand

__all__ = ["BlockIlukFactors", "build_preconditioner", "symbolic_phase"]

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
        if inf["engine"] == 1:   # partitioned sweep: 8 stamps per record (see csrc/psweep.cu)
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
