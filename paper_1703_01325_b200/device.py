"""Device plumbing: torch tensors as raw buffers, streams, operator caching.

PyTorch is used only for device memory (its caching allocator), the current
stream and host<->device copies; every computation is a libbiluk kernel.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _native as nat


def torch():
    import torch as _t
    if not _t.cuda.is_available():
        raise RuntimeError("paper_1703_01325_b200 needs a CUDA device (B200); none is visible")
    return _t


def device_index() -> int:
    t = torch()
    return t.cuda.current_device()


def enter() -> int:
    """Make torch's current device current for libbiluk too; returns the stream handle."""
    dev = device_index()
    nat.set_device(dev)
    return nat.current_stream_handle()


def alloc_bytes(nbytes: int):
    """A 256-byte aligned device byte buffer (torch uint8 tensor)."""
    t = torch()
    buf = t.empty(max(int(nbytes), 256) + 256, dtype=t.uint8, device="cuda")
    off = (-buf.data_ptr()) % 256
    return buf, buf.data_ptr() + off


def to_device_f64(arr):
    """numpy/torch vector -> contiguous float64 CUDA tensor (no copy if already there)."""
    t = torch()
    if isinstance(arr, t.Tensor):
        if arr.is_cuda and arr.dtype == t.float64 and arr.is_contiguous():
            return arr
        return arr.to(device="cuda", dtype=t.float64).contiguous()
    a = np.ascontiguousarray(arr, dtype=np.float64)
    return t.from_numpy(a).to(device="cuda", non_blocking=False)


class DeviceOperator:
    """y = A x on the device for a block (or point, bs = 1) matrix (sparse.py:278-301)."""

    def __init__(self, a):
        from .sparse import as_bsr
        bs, n, m, rp, ci, vals = as_bsr(a)
        self.bs, self.n, self.ncols = bs, n, m
        self.batch_segments = getattr(a, "batch_segments", None)   # block_diagonal batches stay batches
        L = nat.lib()
        h = ctypes.c_void_p()
        nat.check(L.biluk_op_create(bs, n, m, nat.ptr(rp), nat.ptr(ci), ctypes.byref(h)))
        self._h = h
        self._finalizer = weakref.finalize(self, L.biluk_op_destroy, h)
        stream = enter()
        self._ws, wsp = alloc_bytes(L.biluk_op_workspace_bytes(h))
        nat.check(L.biluk_op_bind(h, wsp, L.biluk_op_workspace_bytes(h), stream))
        self._vals = None
        self.set_values(vals)
        self.spmv_bytes = 8 * bs * bs * int(rp[-1]) + 4 * int(rp[-1]) + 4 * (n + 1) + 16 * bs * n

    @property
    def handle(self):
        return self._h

    def set_values(self, vals):
        """(Re)load the block values (same pattern) -- host or device float64, column-major blocks."""
        t = torch()
        stream = enter()
        if self._vals is None:   # an own copy (never alias the caller's tensor)
            self._vals = to_device_f64(vals)
            if isinstance(vals, t.Tensor) and self._vals.data_ptr() == vals.data_ptr():
                self._vals = self._vals.clone()
        else:
            src = vals if isinstance(vals, t.Tensor) else t.from_numpy(np.ascontiguousarray(vals, np.float64))
            if src.numel() != self._vals.numel():
                raise ValueError("set_values: value count does not match the operator's pattern")
            self._vals.copy_(src.reshape(-1))
        nat.check(nat.lib().biluk_op_set_values(self._h, self._vals.data_ptr(), stream))

    def matvec(self, x, out=None):
        t = torch()
        stream = enter()
        xd = to_device_f64(x)
        if xd.numel() != self.ncols * self.bs:
            raise ValueError(f"spmv: operand length {xd.numel()} does not match {self.ncols * self.bs} columns")
        y = out if out is not None else t.empty(self.n * self.bs, dtype=t.float64, device="cuda")
        nat.check(nat.lib().biluk_op_spmv(self._h, xd.data_ptr(), y.data_ptr(), stream))
        return y


_op_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def operator_for(a) -> DeviceOperator:
    """Device operator of a matrix object for one call (spmv / gmres / bicgstab).

    The pattern analysis and workspace are cached per matrix object; the VALUES
    are re-read on every call, because the reference containers let callers
    edit them in place (``.blocks`` is a writable view, reference
    test_sparse.py:123) -- e.g. a Newton loop refreshing its Jacobian.  Pass a
    ``DeviceOperator`` to keep the values resident across calls.
    """
    if isinstance(a, DeviceOperator):
        return a
    try:
        op = _op_cache.get(a)
    except TypeError:
        op = None
    if op is None:
        op = DeviceOperator(a)
        try:
            _op_cache[a] = op
        except TypeError:
            pass
    else:
        from .sparse import as_bsr
        op.set_values(as_bsr(a)[5])
    return op
