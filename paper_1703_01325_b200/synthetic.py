"""Synthetic reservoir-style block 7-point matrices.

Host-side numpy input generation shared by the bench, the tests and the
golden-vector script, so every side is fed the *same arrays*.

Block pattern: the 7-point stencil of ``gen_poisson_3d`` (reference
poisson.py:11-52; x fastest, then y, then z; columns strictly increasing per
row).  Values, with one ``np.random.default_rng(seed)`` drawn in this order:

1. xi ~ N(0, 1)^n; cell permeability kappa = exp(sigma * xi), sigma = 1;
2. R ~ U(-1, 1)^(m, b, b) for the m off-diagonal slots in stored CSR order;
   coupling C_ij = I + 0.2 R (R indexed [row, col]);
3. u ~ U(0, 1)^n.

Transmissibility T_ij = 2 / (1/kappa_i + 1/kappa_j); off-diagonal block
A_ij = -T_ij C_ij; diagonal A_ii = sum_j T_ij C_ij (accumulated in slot order)
+ 1e-2 (1 + u_i) I.  Blocks are stored column-major (reference sparse.py:96-99).
"""

from __future__ import annotations

import numpy as np


def poisson7_pattern(nx: int, ny: int, nz: int):
    """(row_ptr, col_idx) of the 7-point stencil, x-fastest numbering (int64)."""
    nx, ny, nz = int(nx), int(ny), int(nz)
    if min(nx, ny, nz) < 1:
        raise ValueError("grid dimensions must be at least 1")
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    ix = idx % nx
    iy = (idx // nx) % ny
    iz = idx // (nx * ny)
    offs = [(iz > 0, -nx * ny), (iy > 0, -nx), (ix > 0, -1), (np.ones(n, bool), 0),
            (ix < nx - 1, 1), (iy < ny - 1, nx), (iz < nz - 1, nx * ny)]
    counts = np.zeros(n, dtype=np.int64)
    for mask, _ in offs:
        counts += mask
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = np.empty(int(rp[-1]), dtype=np.int64)
    cur = rp[:-1].copy()
    for mask, off in offs:
        nodes = idx[mask]
        ci[cur[nodes]] = nodes + off
        cur[nodes] += 1
    return rp, ci


def gen_poisson_3d(nx: int, ny: int, nz: int):
    """The reference's 7-point operator as a CsrMatrix (reference poisson.py:11-52).

    6 on the diagonal, -1 for each existing axis neighbour (Dirichlet
    truncation), x-fastest numbering, columns increasing within a row.
    """
    from .errors import StructuralError
    from .sparse import CsrMatrix
    if min(int(nx), int(ny), int(nz)) < 1:
        raise StructuralError("grid dimensions must be at least 1")
    rp, ci = poisson7_pattern(nx, ny, nz)
    rows = np.repeat(np.arange(rp.size - 1, dtype=np.int64), np.diff(rp))
    return CsrMatrix(rp.size - 1, rp.size - 1, rp, ci, np.where(ci == rows, 6.0, -1.0))


def reservoir_block_grid(nx: int, ny: int, nz: int, bs: int, seed: int = 0,
                         sigma: float = 1.0, eps: float = 0.2, acc: float = 1e-2):
    """Return (n, bs, row_ptr, col_idx, values) of the synthetic block matrix."""
    bs = int(bs)
    rp, ci = poisson7_pattern(nx, ny, nz)
    n = rp.size - 1
    nnzb = int(rp[-1])
    rng = np.random.default_rng(seed)
    kappa = np.exp(sigma * rng.standard_normal(n))
    erow = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    off = erow != ci
    m = int(off.sum())
    T = 2.0 / (1.0 / kappa[erow[off]] + 1.0 / kappa[ci[off]])
    C = np.eye(bs)[None] + eps * rng.uniform(-1.0, 1.0, (m, bs, bs))
    TC = T[:, None, None] * C
    blocks = np.empty((nnzb, bs, bs))
    blocks[off] = -TC
    # diagonal: sum of the row's coupling blocks in slot order (<= 6 terms:
    # reduceat is sequential at that length), then the accumulation term
    orow = erow[off]
    starts = np.flatnonzero(np.r_[True, orow[1:] != orow[:-1]]) if m else np.zeros(0, np.int64)
    dsum = np.zeros((n, bs, bs))
    if m:
        dsum[orow[starts]] = np.add.reduceat(TC, starts, axis=0)
    dsum += acc * np.eye(bs)[None] * (1.0 + rng.uniform(0.0, 1.0, (n, 1, 1)))
    blocks[~off] = dsum
    vals = np.ascontiguousarray(blocks.transpose(0, 2, 1)).reshape(-1)
    return n, bs, rp, ci, vals


def ones_rhs(n, bs, rp, ci, vals):
    """b = A @ 1 (reference bench.py:83-85), computed block-wise on the host."""
    blk = vals.reshape(-1, bs, bs)            # [slot][col][row] (column-major)
    rowsum = blk.sum(axis=1)                  # sum over columns -> (nnzb, bs) per row
    out = np.zeros((n, bs))
    nz = np.diff(rp) > 0
    out[nz] = np.add.reduceat(rowsum, rp[:-1][nz], axis=0)
    return out.reshape(-1)
