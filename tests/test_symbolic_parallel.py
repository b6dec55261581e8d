"""The row-parallel symbolic phase (plan.cpp, path characterisation of the
level of fill) against the reference's row-merge order (BILUK_SYMBOLIC=sequential)
on grids and random patterns, k = 1..3, including the first row without a
diagonal.  Host-only (no GPU)."""

import ctypes
import os

import numpy as np
import pytest

import paper_1703_01325_b200 as b2
from paper_1703_01325_b200 import _native as nat


def _symbolic(n, rp, ci, k, sequential):
    L = nat.lib()
    rp = np.ascontiguousarray(rp, np.int64)
    ci = np.ascontiguousarray(ci, np.int64)
    h = ctypes.c_void_p()
    err = ctypes.c_int64(-1)
    old = os.environ.get("BILUK_SYMBOLIC")
    if sequential:
        os.environ["BILUK_SYMBOLIC"] = "sequential"
    else:
        os.environ.pop("BILUK_SYMBOLIC", None)
    try:
        rc = L.biluk_symbolic(n, nat.ptr(rp), nat.ptr(ci), k, ctypes.byref(h), ctypes.byref(err))
    finally:
        if old is None:
            os.environ.pop("BILUK_SYMBOLIC", None)
        else:
            os.environ["BILUK_SYMBOLIC"] = old
    if rc != nat.OK:
        return rc, int(err.value), None, None
    nnz = L.biluk_pattern_nnz(h)
    orp = np.zeros(n + 1, np.int64)
    oci = np.zeros(nnz, np.int64)
    L.biluk_pattern_copy(h, nat.ptr(orp), nat.ptr(oci))
    L.biluk_pattern_free(h)
    return rc, -1, orp, oci


def _random_pattern(n, per_row, seed, drop_diag=None):
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        # mostly near-diagonal couplings, some far ones
        near = i + rng.integers(-40, 41, per_row)
        far = rng.integers(0, n, 1)
        cols = set(int(c) for c in np.concatenate([near, far]) if 0 <= c < n)
        if i != drop_diag:
            cols.add(i)
        else:
            cols.discard(i)
        rows.append(sorted(cols))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    return rp, np.array([c for r in rows for c in r], np.int64)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_grid_patterns_match_row_merge(k):
    for shape in [(24, 20, 16), (40, 7, 19)]:
        n, bs, rp, ci, _ = b2.reservoir_block_grid(*shape, 1, seed=0)
        a = _symbolic(n, rp, ci, k, sequential=False)
        s = _symbolic(n, rp, ci, k, sequential=True)
        assert a[0] == s[0] == nat.OK
        assert np.array_equal(a[2], s[2]) and np.array_equal(a[3], s[3])


@pytest.mark.parametrize("k", [1, 2, 3])
def test_random_patterns_match_row_merge(k):
    for seed in range(3):
        rp, ci = _random_pattern(6000, 4, seed)
        a = _symbolic(6000, rp, ci, k, sequential=False)
        s = _symbolic(6000, rp, ci, k, sequential=True)
        assert a[0] == s[0] == nat.OK
        assert np.array_equal(a[2], s[2]) and np.array_equal(a[3], s[3])


def test_first_row_without_diagonal_is_reported():
    rp, ci = _random_pattern(6000, 3, 7, drop_diag=4321)
    a = _symbolic(6000, rp, ci, 2, sequential=False)
    s = _symbolic(6000, rp, ci, 2, sequential=True)
    assert a[0] == s[0] != nat.OK
    assert a[1] == s[1] == 4321
