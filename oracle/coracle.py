"""ctypes wrapper of the C oracle (oracle/coracle.c) -- TEST / BASELINE INFRASTRUCTURE ONLY.

Built by ``make -C oracle`` (also run by ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libcoracle.so")
_lib = None

P = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "coracle.c")):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = ctypes.CDLL(SO)
        L.co_build.argtypes = [ctypes.c_int64, ctypes.c_int, P, P, P, ctypes.c_int, ctypes.POINTER(P),
                               ctypes.POINTER(ctypes.c_int64)]
        L.co_build.restype = ctypes.c_int
        L.co_free.argtypes = [P]
        L.co_sizes.argtypes = [P, P]
        L.co_get.argtypes = [P] * 10
        L.co_apply.argtypes = [P, P, P, P, ctypes.c_int]
        L.co_bsr_spmv.argtypes = [ctypes.c_int64, ctypes.c_int, P, P, P, P, P, ctypes.c_int]
        L.co_symbolic.argtypes = [ctypes.c_int64, P, P, ctypes.c_int, ctypes.POINTER(P), ctypes.POINTER(P),
                                  ctypes.POINTER(ctypes.c_int64)]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data


class COracleError(RuntimeError):
    def __init__(self, code, row):
        super().__init__(f"oracle build failed with code {code} at row {row}")
        self.code, self.row = code, row


class CFactors:
    """Factors + point schedules computed by the C restatement."""

    def __init__(self, n, bs, rp, ci, vals, k):
        L = lib()
        self._rp = np.ascontiguousarray(rp, np.int64)
        self._ci = np.ascontiguousarray(ci, np.int64)
        self._vals = np.ascontiguousarray(vals, np.float64)
        h = P()
        err = ctypes.c_int64(-1)
        rc = L.co_build(n, bs, _p(self._rp), _p(self._ci), _p(self._vals), int(k), ctypes.byref(h), ctypes.byref(err))
        if rc:
            raise COracleError(rc, err.value)
        self._h = h
        s = np.zeros(9, np.int64)
        L.co_sizes(h, _p(s))
        self.n, self.bs, self.nl, self.nu, self.m, self.plnnz, self.punnz, self.nll, self.nul = (int(v) for v in s)
        bs2 = self.bs * self.bs
        self.L_rp = np.zeros(self.n + 1, np.int64)
        self.L_ci = np.zeros(self.nl, np.int64)
        self.L_vals = np.zeros(self.nl * bs2)
        self.dinv = np.zeros((self.n, self.bs, self.bs))
        self.U_rp = np.zeros(self.n + 1, np.int64)
        self.U_ci = np.zeros(self.nu, np.int64)
        self.U_vals = np.zeros(self.nu * bs2)
        self.lo_level_of_row = np.zeros(self.m, np.int64)
        self.up_level_of_row = np.zeros(self.m, np.int64)
        L.co_get(h, _p(self.L_rp), _p(self.L_ci), _p(self.L_vals), _p(self.dinv), _p(self.U_rp), _p(self.U_ci),
                 _p(self.U_vals), _p(self.lo_level_of_row), _p(self.up_level_of_row))
        self._work = np.zeros(self.m)

    def apply(self, b, threads=1):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.m)
        lib().co_apply(self._h, _p(b), _p(x), _p(self._work), int(threads))
        return x

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.co_free(self._h)
            self._h = None


def bsr_spmv(n, bs, rp, ci, vals, x, threads=1):
    rp = np.ascontiguousarray(rp, np.int64)
    ci = np.ascontiguousarray(ci, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(n * bs)
    lib().co_bsr_spmv(n, bs, _p(rp), _p(ci), _p(vals), _p(x), _p(y), int(threads))
    return y
