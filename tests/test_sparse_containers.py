"""Host containers: the structural rules of the reference (sparse.py:35-52)
on hand-made and random index pairs; layout round trips."""

import numpy as np
import pytest

from paper_1703_01325_b200 import BcsrMatrix, CsrMatrix, StructuralError


def _rules_hold(nrows, ncols, rp, ci):
    """Independent statement of the rules, row by row."""
    if nrows < 0 or ncols < 0 or len(rp) != nrows + 1 or rp[0] != 0:
        return False
    if any(rp[i + 1] < rp[i] for i in range(nrows)) or len(ci) != rp[-1]:
        return False
    for i in range(nrows):
        row = list(ci[rp[i]:rp[i + 1]])
        if any(c < 0 or c >= ncols for c in row) or any(a >= b for a, b in zip(row, row[1:])):
            return False
    return True


def test_random_index_pairs_follow_the_rules():
    rng = np.random.default_rng(0)
    for _ in range(400):
        nrows, ncols = int(rng.integers(0, 6)), int(rng.integers(1, 6))
        lens = rng.integers(0, 4, nrows)
        rp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
        ci = np.concatenate([np.sort(rng.choice(ncols + 1, size=min(int(k), ncols + 1), replace=False)) - 0
                             for k in lens]).astype(np.int64) if nrows else np.zeros(0, np.int64)
        # perturb sometimes: a swapped pair, a duplicate, a bad pointer
        mode = rng.integers(0, 5)
        if mode == 1 and len(ci) > 1:
            j = int(rng.integers(0, len(ci) - 1))
            ci[j], ci[j + 1] = ci[j + 1], ci[j]
        elif mode == 2 and len(ci) > 1:
            ci[-1] = ci[0]
        elif mode == 3 and nrows > 1:
            rp[1] = rp[-1] + 1
        ok = _rules_hold(nrows, ncols, rp, ci)
        vals = np.ones(len(ci))
        if ok:
            m = CsrMatrix(nrows, ncols, rp, ci, vals)
            assert m.nnz == len(ci)
        else:
            with pytest.raises(StructuralError):
                CsrMatrix(nrows, ncols, rp, ci, vals)


def test_messages_name_the_fault():
    with pytest.raises(StructuralError, match="row 1"):
        CsrMatrix(2, 3, [0, 1, 3], [0, 2, 1], [1.0, 2.0, 3.0])
    with pytest.raises(StructuralError, match="outside"):
        CsrMatrix(1, 2, [0, 1], [2], [1.0])
    with pytest.raises(StructuralError, match="values"):
        BcsrMatrix(2, 1, 1, [0, 1], [0], np.ones(3))
    with pytest.raises(StructuralError, match="block size"):
        BcsrMatrix(0, 1, 1, [0, 1], [0], np.ones(0))


def test_block_layout_is_column_major():
    vals = np.arange(8.0)   # two 2x2 blocks, column-major
    m = BcsrMatrix(2, 1, 2, [0, 2], [0, 1], vals)
    d = m.to_dense()
    assert d[0, 0] == 0.0 and d[1, 0] == 1.0 and d[0, 1] == 2.0 and d[1, 1] == 3.0
    assert d[0, 2] == 4.0 and d[1, 3] == 7.0
    assert m.blocks[1, 0, 1] == 6.0 and m.nnzb == 2 and m.shape == (2, 4)
    c = CsrMatrix(2, 2, [0, 1, 2], [1, 0], [5.0, 6.0])
    assert np.array_equal(c.to_dense(), [[0, 5], [6, 0]])
    cols, vals_r = c.row(1)
    assert list(cols) == [0] and list(vals_r) == [6.0]
