"""Host-side sparse containers of the drop-in API (reference sparse.py).

The constructors take the reference's arguments and expose its fields and
layouts (`CsrMatrix` sparse.py:55-89, `BcsrMatrix` :92-151 with column-major
blocks, `PatternMatrix` :154-221) and enforce its structural rules, so objects
can be passed back and forth; the index checks live in one place
(`_compressed_violation`) and name the offending row or index.  These
are index/value holders only: every numeric operation on the path runs on the
GPU through libbiluk.  Reference objects are accepted anywhere through
duck typing (``as_bsr``).
"""

from __future__ import annotations

import numpy as np

from .errors import StructuralError

__all__ = ["CsrMatrix", "BcsrMatrix", "PatternMatrix", "bcsr_from_csr", "csr_expand",
           "extract_point_pattern", "csr_from_triplets", "assemble_csr", "as_bsr", "block_diagonal"]


def _index_vector(a, label):
    v = np.asarray(a, dtype=np.int64)
    if v.ndim != 1:
        raise StructuralError(f"{label}: expected a one-dimensional index array, got shape {v.shape}")
    return np.ascontiguousarray(v)


def _compressed_violation(nrows, ncols, rp, ci):
    """The first structural rule a compressed-row index pair breaks, or None.

    Rules (the reference's, sparse.py:35-52): non-negative dimensions; a row
    pointer of nrows + 1 entries from 0, never decreasing; one column index
    per stored entry, inside [0, ncols), strictly increasing within a row.
    """
    if nrows < 0 or ncols < 0:
        return f"dimensions ({nrows}, {ncols}) must be non-negative"
    if len(rp) != nrows + 1:
        return f"row pointer has {len(rp)} entries, {nrows + 1} expected"
    if rp[0] != 0:
        return f"row pointer starts at {int(rp[0])}, not 0"
    steps = np.diff(rp)
    if (steps < 0).any():
        return f"row pointer decreases after row {int(np.argmax(steps < 0))}"
    nnz = int(rp[-1])
    if len(ci) != nnz:
        return f"{len(ci)} column indices for {nnz} stored entries"
    if nnz == 0:
        return None
    lo, hi = int(ci.min()), int(ci.max())
    if lo < 0 or hi >= ncols:
        return f"column index {lo if lo < 0 else hi} outside [0, {ncols})"
    # consecutive entries (t, t + 1) of one row must increase; a row start breaks the pair
    same_row = np.ones(nnz - 1, dtype=bool)
    starts = rp[1:-1]
    same_row[starts[(starts > 0) & (starts < nnz)] - 1] = False
    bad = np.flatnonzero(same_row & (np.diff(ci) <= 0))
    if bad.size:
        row = int(np.searchsorted(rp, bad[0], side="right") - 1)
        return f"column indices of row {row} are not strictly increasing"
    return None


class _RowCompressed:
    """Index half shared by the point and block containers: the row pointer,
    the column indices and the checks on them."""

    def _set_index(self, kind, nrows, ncols, row_ptr, col_idx):
        rp = _index_vector(row_ptr, f"{kind} row_ptr")
        ci = _index_vector(col_idx, f"{kind} col_idx")
        why = _compressed_violation(nrows, ncols, rp, ci)
        if why is not None:
            raise StructuralError(f"{kind}: {why}")
        self.row_ptr, self.col_idx = rp, ci

    def _stored(self):
        return int(self.row_ptr[-1])

    def _span(self, i):
        return int(self.row_ptr[i]), int(self.row_ptr[i + 1])

    def _row_of_entry(self, nrows):
        return np.repeat(np.arange(nrows), np.diff(self.row_ptr))


class CsrMatrix(_RowCompressed):
    """Point-wise CSR matrix: num_rows, num_cols, row_ptr, col_idx, values
    (the fields of reference sparse.py:55-89)."""

    def __init__(self, num_rows, num_cols, row_ptr, col_idx, values):
        self.num_rows, self.num_cols = int(num_rows), int(num_cols)
        self._set_index("CsrMatrix", self.num_rows, self.num_cols, row_ptr, col_idx)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        if self.values.shape != (self._stored(),):
            raise StructuralError(f"CsrMatrix: {self.values.size} values for {self._stored()} stored entries")

    shape = property(lambda self: (self.num_rows, self.num_cols))
    nnz = property(lambda self: self._stored())

    def row(self, i):
        s, e = self._span(i)
        return self.col_idx[s:e], self.values[s:e]

    def to_dense(self):
        dense = np.zeros(self.shape)
        dense[self._row_of_entry(self.num_rows), self.col_idx] = self.values
        return dense

    def __repr__(self):
        return f"CsrMatrix({self.num_rows}x{self.num_cols}, nnz={self.nnz})"


class BcsrMatrix(_RowCompressed):
    """Block CSR: bs x bs blocks stored flat and column-major, block t at
    values[t*bs*bs:(t+1)*bs*bs] (the fields and layout of reference sparse.py:92-151)."""

    def __init__(self, block_size, num_block_rows, num_block_cols, row_ptr, col_idx, values):
        self.block_size = int(block_size)
        self.num_block_rows, self.num_block_cols = int(num_block_rows), int(num_block_cols)
        if self.block_size < 1:
            raise StructuralError(f"BcsrMatrix: block size {self.block_size} is not positive")
        self._set_index("BcsrMatrix", self.num_block_rows, self.num_block_cols, row_ptr, col_idx)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        want = self._stored() * self.block_size ** 2
        if self.values.shape != (want,):
            raise StructuralError(f"BcsrMatrix: {self.values.size} values, {want} expected "
                                  f"({self._stored()} blocks of {self.block_size}x{self.block_size})")

    nnzb = property(lambda self: self._stored())
    shape = property(lambda self: (self.num_block_rows * self.block_size, self.num_block_cols * self.block_size))

    @property
    def blocks(self):
        """(nnzb, bs, bs) view; element [t, r, c] is row r, column c of block t."""
        bs = self.block_size
        return self.values.reshape(self.nnzb, bs, bs).swapaxes(1, 2)

    def block_row(self, i):
        s, e = self._span(i)
        return self.col_idx[s:e], s

    def to_dense(self):
        bs = self.block_size
        off = np.arange(bs)
        rows = self._row_of_entry(self.num_block_rows)[:, None, None] * bs + off[None, :, None]
        cols = self.col_idx[:, None, None] * bs + off[None, None, :]
        dense = np.zeros(self.shape)
        dense[rows, cols] = self.blocks
        return dense

    def __repr__(self):
        return (f"BcsrMatrix(bs={self.block_size}, {self.num_block_rows}x{self.num_block_cols} blocks, "
                f"nnzb={self.nnzb})")


class PatternMatrix:
    """Value-free square pattern with sorted rows (reference sparse.py:154-221)."""

    def __init__(self, n, rows=None):
        self.n = int(n)
        if self.n < 0:
            raise StructuralError("PatternMatrix: negative dimension")
        if rows is None:
            self.rows = [[] for _ in range(self.n)]
            return
        rows = [[int(j) for j in r] for r in rows]
        if len(rows) != self.n:
            raise StructuralError("PatternMatrix: need one row list per row")
        for i, r in enumerate(rows):
            if any(r[t] >= r[t + 1] for t in range(len(r) - 1)):
                raise StructuralError(f"PatternMatrix: row {i} is not strictly increasing")
            if r and (r[0] < 0 or r[-1] >= self.n):
                raise StructuralError(f"PatternMatrix: row {i} has an index out of range")
        self.rows = rows

    @classmethod
    def from_csr_arrays(cls, n, rp, ci):
        out = cls(n)
        rp = np.asarray(rp)
        ci = np.asarray(ci)
        out.rows = [ci[rp[i]:rp[i + 1]].tolist() for i in range(n)]
        return out

    def to_csr_arrays(self):
        rp = np.zeros(self.n + 1, dtype=np.int64)
        rp[1:] = np.cumsum([len(r) for r in self.rows])
        ci = np.fromiter((j for r in self.rows for j in r), dtype=np.int64, count=int(rp[-1]))
        return rp, ci

    @property
    def row_lengths(self):
        return [len(r) for r in self.rows]

    @property
    def nnz(self):
        return sum(len(r) for r in self.rows)

    def as_set(self):
        return {(i, j) for i, r in enumerate(self.rows) for j in r}

    def __eq__(self, other):
        if not hasattr(other, "rows") or not hasattr(other, "n"):
            return NotImplemented
        return self.n == other.n and self.rows == other.rows

    def __repr__(self):
        return f"PatternMatrix(n={self.n}, nnz={self.nnz})"


def assemble_csr(num_rows, num_cols, rows, cols, vals):
    """CSR from parallel (row, col, value) arrays, duplicates summed (reference sparse.py:224-245)."""
    r = np.asarray(rows, dtype=np.int64).ravel()
    c = np.asarray(cols, dtype=np.int64).ravel()
    v = np.asarray(vals, dtype=np.float64).ravel()
    if not (r.size == c.size == v.size):
        raise StructuralError("triplet arrays must have equal length")
    if r.size == 0:
        return CsrMatrix(num_rows, num_cols, np.zeros(num_rows + 1, np.int64), [], [])
    if r.min() < 0 or r.max() >= num_rows or c.min() < 0 or c.max() >= num_cols:
        raise StructuralError("triplet index outside the matrix")
    key = r * num_cols + c
    order = np.argsort(key, kind="stable")
    key, v = key[order], v[order]
    uniq, first = np.unique(key, return_index=True)
    summed = np.add.reduceat(v, first)
    rp = np.zeros(num_rows + 1, np.int64)
    np.cumsum(np.bincount(uniq // num_cols, minlength=num_rows), out=rp[1:])
    return CsrMatrix(num_rows, num_cols, rp, uniq % num_cols, summed)


def csr_from_triplets(num_rows, num_cols, entries):
    """CSR from (row, col, value) triplets, duplicates summed (reference sparse.py:248-258)."""
    entries = list(entries)
    if not entries:
        return CsrMatrix(num_rows, num_cols, np.zeros(num_rows + 1, np.int64), [], [])
    r, c, v = (np.asarray(x) for x in zip(*entries))
    r = r.astype(np.int64)
    c = c.astype(np.int64)
    v = v.astype(np.float64)
    if r.min() < 0 or r.max() >= num_rows or c.min() < 0 or c.max() >= num_cols:
        raise StructuralError("triplet index outside the matrix")
    key = r * num_cols + c
    order = np.argsort(key, kind="stable")
    key, v = key[order], v[order]
    uniq, first = np.unique(key, return_index=True)
    vals = np.add.reduceat(v, first)
    rows = uniq // num_cols
    rp = np.zeros(num_rows + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=num_rows), out=rp[1:])
    return CsrMatrix(num_rows, num_cols, rp, uniq % num_cols, vals)


def bcsr_from_csr(a, bs):
    """Reblock a point CSR matrix into bs x bs blocks (reference sparse.py:304-334)."""
    bs = int(bs)
    if bs < 1:
        raise StructuralError("block size must be at least 1")
    if a.num_rows % bs or a.num_cols % bs:
        raise StructuralError(f"block size {bs} does not divide matrix shape {a.num_rows}x{a.num_cols}")
    nbr, nbc = a.num_rows // bs, a.num_cols // bs
    if a.row_ptr[-1] == 0:
        return BcsrMatrix(bs, nbr, nbc, np.zeros(nbr + 1, np.int64), [], [])
    erow = np.repeat(np.arange(a.num_rows, dtype=np.int64), np.diff(a.row_ptr))
    col = np.asarray(a.col_idx, dtype=np.int64)
    key = (erow // bs) * nbc + col // bs
    uniq = np.unique(key)
    rp = np.zeros(nbr + 1, np.int64)
    np.cumsum(np.bincount(uniq // nbc, minlength=nbr), out=rp[1:])
    vals = np.zeros(uniq.size * bs * bs)
    slot = np.searchsorted(uniq, key)
    vals[slot * bs * bs + (col % bs) * bs + (erow % bs)] = a.values
    return BcsrMatrix(bs, nbr, nbc, rp, uniq % nbc, vals)


def csr_expand(a):
    """Point CSR of a block matrix with exact zeros dropped (reference sparse.py:337-374).

    Within point row (I, r) the entries follow block order, then the in-block
    column, as in the reference.
    """
    bs = int(a.block_size)
    n, m = int(a.num_block_rows), int(a.num_block_cols)
    rp = np.asarray(a.row_ptr, dtype=np.int64)
    ci = np.asarray(a.col_idx, dtype=np.int64)
    nnzb = int(rp[-1])
    blk = np.asarray(a.values, dtype=np.float64).reshape(nnzb, bs, bs)   # [slot][c][r]
    brow = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    # order (block row, r, slot, c): slots of a block row are contiguous
    vals = blk.transpose(0, 2, 1)                                       # [slot][r][c]
    # per block row: (r, slot, c) ordering = transpose of (slot, r, c) inside the row
    order = np.lexsort((np.tile(np.arange(bs), nnzb * bs),
                        np.repeat(np.arange(nnzb), bs * bs),
                        np.tile(np.repeat(np.arange(bs), bs), nnzb),
                        np.repeat(brow, bs * bs)))
    v = vals.reshape(-1)[order]
    cols = (np.repeat(ci, bs * bs) * bs + np.tile(np.arange(bs), nnzb * bs))[order]
    prow = (np.repeat(brow, bs * bs) * bs + np.tile(np.repeat(np.arange(bs), bs), nnzb))[order]
    keep = v != 0.0
    v, cols, prow = v[keep], cols[keep], prow[keep]
    prp = np.zeros(n * bs + 1, np.int64)
    np.cumsum(np.bincount(prow, minlength=n * bs), out=prp[1:])
    return CsrMatrix(n * bs, m * bs, prp, cols, v)


def extract_point_pattern(a):
    """Pattern of the stored (block) structure; values never read (reference sparse.py:261-275)."""
    if hasattr(a, "block_size"):
        n, m = a.num_block_rows, a.num_block_cols
    else:
        n, m = a.num_rows, a.num_cols
    if n != m:
        raise StructuralError("pattern extraction requires a square matrix")
    return PatternMatrix.from_csr_arrays(n, a.row_ptr, a.col_idx)


def as_bsr(a):
    """(bs, n_rows, n_cols, row_ptr int64, col_idx int64, values f64) of any BSR/CSR-like object.

    A point CSR matrix is block size one (reference factor.py:312-313).
    """
    if hasattr(a, "block_size"):
        return (int(a.block_size), int(a.num_block_rows), int(a.num_block_cols),
                np.ascontiguousarray(a.row_ptr, dtype=np.int64), np.ascontiguousarray(a.col_idx, dtype=np.int64),
                np.ascontiguousarray(a.values, dtype=np.float64))
    if hasattr(a, "num_rows"):
        return (1, int(a.num_rows), int(a.num_cols), np.ascontiguousarray(a.row_ptr, dtype=np.int64),
                np.ascontiguousarray(a.col_idx, dtype=np.int64), np.ascontiguousarray(a.values, dtype=np.float64))
    raise TypeError("expected a BcsrMatrix or CsrMatrix")


def block_diagonal(mats):
    """One BcsrMatrix holding independent systems on its diagonal (batch config).

    ILU(k) of a block-diagonal matrix is the ILU(k) of each block: the symbolic
    phase, the factors and the level sets decouple (a row only ever meets rows
    of its own system), so factoring and applying the batch as one operator
    equals factoring and applying every system alone -- while one persistent
    sweep interleaves their level chains.  Vectors of the batch are the
    systems' vectors concatenated in order; ``batch_segments`` holds the
    systems' block-row offsets (what ``bicgstab_batched`` takes).
    """
    parts = [as_bsr(m) for m in mats]   # (bs, n_rows, n_cols, row_ptr, col_idx, values)
    if not parts:
        raise ValueError("empty batch")
    bs = parts[0][0]
    if any(q[0] != bs for q in parts):
        raise StructuralError("batch systems must share the block size")
    if any(q[1] != q[2] for q in parts):
        raise StructuralError("batch systems must be square")
    n_tot = sum(q[1] for q in parts)
    nnz_tot = sum(int(q[3][-1]) for q in parts)
    rp = np.zeros(n_tot + 1, np.int64)
    ci = np.empty(nnz_tot, np.int64)
    vals = np.empty(nnz_tot * bs * bs, np.float64)
    r = z = 0
    for _, nb, _, qrp, qci, qv in parts:
        nz = int(qrp[-1])
        rp[r + 1:r + nb + 1] = qrp[1:] + z
        ci[z:z + nz] = qci + r
        vals[z * bs * bs:(z + nz) * bs * bs] = qv.reshape(-1)
        r += nb
        z += nz
    out = BcsrMatrix(bs, n_tot, n_tot, rp, ci, vals)
    # block-row offsets of the systems; block diagonal by construction
    out.batch_segments = np.concatenate([[0], np.cumsum([q[1] for q in parts])]).astype(np.int64)
    return out
