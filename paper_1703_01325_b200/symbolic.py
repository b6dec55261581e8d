"""The symbolic phase and the coupled ILU(k) oracle (reference symbolic.py).

``symbolic_phase`` is computed by libbiluk (host C++, bit-exact with the
reference).  ``coupled_iluk_oracle`` is the reference's own dense checker of
the two-phase pipeline (symbolic.py:75-122): a single pass interleaving the
level-of-fill updates with the elimination, on a dense copy -- small matrices
only, host numpy by design (it is a test oracle in the reference's public API,
not a step of the preconditioner).
"""

from __future__ import annotations

import numpy as np

from .errors import FactorizationError, StructuralError
from .factor import symbolic_phase
from .sparse import CsrMatrix, PatternMatrix

__all__ = ["coupled_iluk_oracle", "symbolic_phase"]

_ZERO_PIVOT = 1e-300


def coupled_iluk_oracle(a, k):
    """Single-pass dense ILU(k) of a CsrMatrix -> (factored CsrMatrix, PatternMatrix).

    Row i is eliminated against every earlier row p whose current level
    lev(i, p) <= k (pivot order ascending); each elimination lowers the levels
    of row i's later columns to lev(i, p) + lev(p, j) + 1.  Positions ending
    above level k are dropped.  The factored values hold the unit-lower
    multipliers below the diagonal and U on and above it.
    """
    k = int(k)
    if k < 0:
        raise ValueError("fill level k must be nonnegative")
    if a.num_rows != a.num_cols:
        raise StructuralError("oracle requires a square matrix")
    n = int(a.num_rows)
    rp = np.asarray(a.row_ptr, np.int64)
    ci = np.asarray(a.col_idx, np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    w = np.zeros((n, n))
    w[rows, ci] = np.asarray(a.values, np.float64)
    far = np.int64(1) << 40                  # "not in the pattern"
    lev = np.full((n, n), far, dtype=np.int64)
    lev[rows, ci] = 0
    for i in range(1, n):
        wi, li = w[i], lev[i]
        for p in range(i):                   # levels of row i drop while it is eliminated: in order
            if li[p] > k:
                continue
            piv = w[p, p]
            if abs(piv) < _ZERO_PIVOT:
                raise FactorizationError(f"zero pivot in row {p}", row=p)
            wi[p] /= piv
            if p + 1 < n:
                wi[p + 1:] -= wi[p] * w[p, p + 1:]
                np.minimum(li[p + 1:], li[p] + lev[p, p + 1:] + 1, out=li[p + 1:])
        wi[li > k] = 0.0
    keep = lev <= k
    kr, kc = np.nonzero(keep)                # row-major: rows ascending, columns sorted
    out_rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(kr, minlength=n), out=out_rp[1:])
    fac = CsrMatrix(n, n, out_rp, kc.astype(np.int64), w[kr, kc])
    return fac, PatternMatrix.from_csr_arrays(n, out_rp, kc)
