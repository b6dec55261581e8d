"""CPU restatement of the reference block ILU(k) hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity *oracle*.  It is imported only by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference`` legs
of ``bench.py``; the product (``paper_1703_01325_b200``) never imports it and
has no CPU fallback.

It restates, in plain numpy / Python, the algorithms of the reference package
``blockiluk`` (``/root/reference/pkg/src/blockiluk``) for the path named in
``BASELINE.json``'s north star.  Every function cites the reference lines it
follows.  It is written independently (different data structures, no shared
code) and is *pinned* against golden vectors produced by running the
reference itself (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``,
checked by ``tests/test_oracle_golden.py``).

BiCGSTAB has no reference counterpart; ``bicgstab``
below *defines* the contract, built only from the restated ``spmv`` and
``apply_preconditioner``.  Its golden vectors are produced by running this
same definition on top of the reference's own ``spmv``/``apply_preconditioner``.

Array conventions (same as the reference):
  * BSR: ``rp`` (n+1), ``ci`` (nnzb), ``vals`` (nnzb*bs*bs) with every block
    flattened column-major (sparse.py:92-99, :126-130).
  * ``dinv``: (n, bs, bs) ordinary row-major ndarray (factor.py:247).
"""

from __future__ import annotations

import heapq
import math

import numpy as np

PIVOT_RTOL = 1e-13      # factor.py:32-33
ZERO_PIVOT = 1e-300     # factor.py:34-35 (point kernel), symbolic.py:24


class OracleStructuralError(ValueError):
    pass


class OracleSingularBlock(RuntimeError):
    def __init__(self, msg, row=None):
        super().__init__(msg)
        self.row = row


class OracleZeroPivot(RuntimeError):
    def __init__(self, msg, row=None):
        super().__init__(msg)
        self.row = row


# ----------------------------------------------------------------------------
# block helpers
# ----------------------------------------------------------------------------

def blocks_of(vals, bs):
    """(nnzb, bs, bs) matrices from column-major flattened storage (sparse.py:126-130)."""
    return np.asarray(vals, dtype=np.float64).reshape(-1, bs, bs).transpose(0, 2, 1)


def flatten_blocks(blocks):
    """Inverse of :func:`blocks_of`: column-major flattening."""
    return np.ascontiguousarray(np.asarray(blocks).transpose(0, 2, 1)).reshape(-1)


def block_invert(m):
    """Inverse by LU with partial pivoting; rules of factor.py:38-70.

    * an all-zero block is singular (factor.py:48-50)
    * 1x1: 1/b (factor.py:51-52)
    * singular when |pivot| < 1e-13 * max|B| (factor.py:57-58)
    """
    m = np.array(m, dtype=np.float64)
    bs = m.shape[0]
    amax = float(np.max(np.abs(m))) if bs else 0.0
    if amax == 0.0:
        raise OracleSingularBlock("all-zero block")
    if bs == 1:
        return np.array([[1.0 / m[0, 0]]])
    perm = list(range(bs))
    lu = m
    for c in range(bs):
        piv = c + int(np.argmax(np.abs(lu[c:, c])))
        if abs(lu[piv, c]) < PIVOT_RTOL * amax:
            raise OracleSingularBlock(f"pivot {lu[piv, c]:.3e} at step {c}")
        if piv != c:
            lu[[c, piv]] = lu[[piv, c]]
            perm[c], perm[piv] = perm[piv], perm[c]
        for r in range(c + 1, bs):
            lu[r, c] /= lu[c, c]
            lu[r, c + 1:] -= lu[r, c] * lu[c, c + 1:]
    # solve L U X = P  column by column (forward then backward substitution)
    inv = np.zeros((bs, bs))
    for col in range(bs):
        e = np.array([1.0 if perm[r] == col else 0.0 for r in range(bs)])
        for r in range(1, bs):
            e[r] -= lu[r, :r] @ e[:r]
        for r in range(bs - 1, -1, -1):
            e[r] = (e[r] - lu[r, r + 1:] @ e[r + 1:]) / lu[r, r]
        inv[:, col] = e
    return inv


# ----------------------------------------------------------------------------
# symbolic phase (symbolic.py:27-72)
# ----------------------------------------------------------------------------

def symbolic_phase(n, rows, k):
    """Level-of-fill ILU(k) pattern; ``rows`` is a list of sorted column lists.

    Row-by-row elimination with a min-heap of pivots < i; the candidate level
    of (i, j) through pivot p is lev(i,p) + lev(p,j) + 1, the minimum wins and
    levels above k are never stored (symbolic.py:46-71).  Returns the grown
    row lists.  Missing diagonal -> OracleStructuralError (symbolic.py:49-50).
    """
    k = int(k)
    if k < 0:
        raise ValueError("fill level k must be nonnegative")
    ups = [None] * n          # finalized (cols, levels) strictly right of diagonal
    out = []
    for i in range(n):
        level = {int(j): 0 for j in rows[i]}
        if i not in level:
            raise OracleStructuralError(f"row {i} has no diagonal entry")
        heap = [j for j in level if j < i]
        heapq.heapify(heap)
        while heap:
            p = heapq.heappop(heap)
            base = level[p]
            ucols, ulevs = ups[p]
            for j, lpj in zip(ucols, ulevs):
                lv = base + lpj + 1
                if lv > k:
                    continue
                cur = level.get(j)
                if cur is None:
                    level[j] = lv
                    if j < i:
                        heapq.heappush(heap, j)
                elif lv < cur:
                    level[j] = lv
        cols = sorted(level)
        out.append(cols)
        right = [j for j in cols if j > i]
        ups[i] = (right, [level[j] for j in right])
    return out


# ----------------------------------------------------------------------------
# materialize (factor.py:83-121)
# ----------------------------------------------------------------------------

def materialize(n, bs, rp, ci, vals, prows):
    """Values of A on pattern ``prows`` (zero-filled fill slots)."""
    prp = np.zeros(n + 1, dtype=np.int64)
    prp[1:] = np.cumsum([len(r) for r in prows])
    pci = np.fromiter((j for r in prows for j in r), dtype=np.int64, count=int(prp[-1]))
    per = bs * bs
    pv = np.zeros((int(prp[-1]), per))
    old = np.asarray(vals, dtype=np.float64).reshape(-1, per)
    for i in range(n):
        s, e = int(rp[i]), int(rp[i + 1])
        if s == e:
            continue
        seg = pci[prp[i]:prp[i + 1]]
        pos = np.searchsorted(seg, ci[s:e])
        if np.any(pos >= seg.size) or np.any(seg[np.minimum(pos, seg.size - 1)] != ci[s:e]):
            raise OracleStructuralError(f"pattern is missing stored position in row {i}")
        pv[prp[i] + pos] = old[s:e]
    return prp, pci, pv.reshape(-1)


# ----------------------------------------------------------------------------
# numeric factorization (factor.py:124-205) and split (factor.py:230-289)
# ----------------------------------------------------------------------------

def _diag_slot(pci, s, e, i):
    d = s + int(np.searchsorted(pci[s:e], i))
    if d == e or pci[d] != i:
        raise OracleStructuralError(f"block row {i} has no diagonal block")
    return d


def block_ilu0(n, bs, prp, pci, pvals):
    """In-place block IKJ ILU(0) on the materialized pattern.

    bs > 1 (factor.py:165-205): for each lower slot p (ascending)
    A_ip <- A_ip Dinv_p, then A_ij -= A_ip A_pj on stored (i, j), j > p; the
    diagonal block of row i is inverted once the row is eliminated.  U stays
    unscaled.  bs == 1 delegates to the point kernel (factor.py:124-148):
    division by the pivot, zero pivot < 1e-300 -> OracleZeroPivot.
    Returns (factored values (copy), dinv (n,bs,bs) or None for bs==1).
    """
    per = bs * bs
    blk = blocks_of(np.array(pvals, dtype=np.float64), bs).copy()   # (nnz, bs, bs)
    if bs == 1:
        diag = np.zeros(n)
        for i in range(n):
            s, e = int(prp[i]), int(prp[i + 1])
            d = _diag_slot(pci, s, e, i)
            colpos = {int(pci[t]): t for t in range(s, e)}
            for t in range(s, d):
                p = int(pci[t])
                blk[t, 0, 0] = blk[t, 0, 0] / diag[p]
                ps, pe = int(prp[p]), int(prp[p + 1])
                pd = _diag_slot(pci, ps, pe, p)
                for u in range(pd + 1, pe):
                    q = colpos.get(int(pci[u]))
                    if q is not None:
                        blk[q, 0, 0] -= blk[t, 0, 0] * blk[u, 0, 0]
            dv = blk[d, 0, 0]
            if abs(dv) < ZERO_PIVOT:
                raise OracleZeroPivot(f"zero pivot at row {i}", row=i)
            diag[i] = dv
        return flatten_blocks(blk), None
    dinv = np.zeros((n, bs, bs))
    for i in range(n):
        s, e = int(prp[i]), int(prp[i + 1])
        d = _diag_slot(pci, s, e, i)
        colpos = {int(pci[t]): t for t in range(s, e)}
        for t in range(s, d):
            p = int(pci[t])
            lip = blk[t] @ dinv[p]
            blk[t] = lip
            ps, pe = int(prp[p]), int(prp[p + 1])
            pd = _diag_slot(pci, ps, pe, p)
            for u in range(pd + 1, pe):
                q = colpos.get(int(pci[u]))
                if q is not None:
                    blk[q] -= lip @ blk[u]
        try:
            dinv[i] = block_invert(blk[d])
        except OracleSingularBlock as err:
            raise OracleSingularBlock(f"singular diagonal block at row {i}", row=i) from err
    return flatten_blocks(blk), dinv


def split_ldu(n, bs, prp, pci, fvals):
    """(L, dinv, U') from factored values, factor.py:230-289.

    L = strict-lower slots verbatim; dinv[i] = inv(U_ii); U'_ij = dinv[i] U_ij.
    Returns dict with L_rp, L_ci, L_vals, dinv, U_rp, U_ci, U_vals (col-major).
    """
    blk = blocks_of(fvals, bs)
    lrp = np.zeros(n + 1, dtype=np.int64)
    urp = np.zeros(n + 1, dtype=np.int64)
    lsel, usel = [], []
    dinv = np.zeros((n, bs, bs))
    uscaled = []
    for i in range(n):
        s, e = int(prp[i]), int(prp[i + 1])
        d = _diag_slot(pci, s, e, i)
        try:
            dinv[i] = block_invert(blk[d])
        except OracleSingularBlock as err:
            raise OracleSingularBlock(f"singular diagonal block at row {i}", row=i) from err
        lrp[i + 1] = lrp[i] + (d - s)
        urp[i + 1] = urp[i] + (e - d - 1)
        lsel.extend(range(s, d))
        usel.extend(range(d + 1, e))
        if e > d + 1:
            uscaled.append(np.einsum("ab,nbc->nac", dinv[i], blk[d + 1:e]))
    lsel = np.asarray(lsel, dtype=np.int64)
    usel = np.asarray(usel, dtype=np.int64)
    ub = np.concatenate(uscaled) if uscaled else np.zeros((0, bs, bs))
    return {
        "L_rp": lrp, "L_ci": pci[lsel].astype(np.int64), "L_vals": flatten_blocks(blk[lsel]),
        "dinv": dinv,
        "U_rp": urp, "U_ci": pci[usel].astype(np.int64), "U_vals": flatten_blocks(ub),
    }


# ----------------------------------------------------------------------------
# point expansion (sparse.py:337-374) and level schedules (trisolve.py:98-118)
# ----------------------------------------------------------------------------

def csr_expand(n, bs, rp, ci, vals):
    """Point CSR of a BSR matrix, exact zeros dropped (sparse.py:340-343, :366).

    Within point row (i, r) entries follow block order then in-block column.
    """
    rp = np.asarray(rp, dtype=np.int64)
    ci = np.asarray(ci, dtype=np.int64)
    nnzb = int(rp[-1])
    blk = blocks_of(vals, bs)                             # (nnzb, r, c)
    brow = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    # entry arrays ordered (block row, r, slot, c)
    r_idx = np.arange(bs)
    # build per (slot, r, c) arrays then sort by (brow, r, slot, c)
    slot = np.arange(nnzb, dtype=np.int64)
    S, R, C = np.meshgrid(slot, r_idx, r_idx, indexing="ij")   # (nnzb, bs, bs)
    prow = brow[S] * bs + R
    pcol = ci[S] * bs + C
    v = blk[S, R, C]
    key_order = np.lexsort((C.ravel(), S.ravel(), R.ravel(), brow[S].ravel()))
    prow = prow.ravel()[key_order]
    pcol = pcol.ravel()[key_order]
    v = v.ravel()[key_order]
    keep = v != 0.0
    prow, pcol, v = prow[keep], pcol[keep], v[keep]
    prp = np.zeros(n * bs + 1, dtype=np.int64)
    np.cumsum(np.bincount(prow, minlength=n * bs), out=prp[1:])
    return prp, pcol, v


def level_schedule(m, rp, ci, orientation):
    """Eq. (4) levels, 1-based; forward for lower, reverse for upper (trisolve.py:98-118).

    Returns (level_of_row, levels) where levels[l] lists the rows of level l+1
    in ascending order (stable argsort, trisolve.py:114).
    """
    lev = np.zeros(m, dtype=np.int64)
    order = range(m) if orientation == "lower" else range(m - 1, -1, -1)
    rp_l = rp.tolist()
    ci_l = ci.tolist()
    lev_l = [0] * m
    for i in order:
        s, e = rp_l[i], rp_l[i + 1]
        best = 0
        for t in range(s, e):
            lj = lev_l[ci_l[t]]
            if lj > best:
                best = lj
        lev_l[i] = best + 1
    lev[:] = lev_l
    num = int(lev.max()) if m else 0
    by = np.argsort(lev, kind="stable")
    counts = np.bincount(lev, minlength=num + 1)[1:]
    levels = np.split(by, np.cumsum(counts)[:-1]) if num else []
    return lev, levels


def solve_unit_triangular(m, rp, ci, vals, levels, b):
    """(I + T) x = b, rows level by level, stored-order reduction (trisolve.py:121-145)."""
    x = np.array(b, dtype=np.float64)
    for rows in levels:
        lens = rp[rows + 1] - rp[rows]
        if int(lens.sum()) == 0:
            continue
        idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
        prod = vals[idx] * x[ci[idx]]
        seg = np.zeros(rows.size + 1, dtype=np.int64)
        np.cumsum(lens, out=seg[1:])
        nz = lens > 0
        sums = np.zeros(rows.size)
        sums[nz] = np.add.reduceat(prod, seg[:-1][nz])
        x[rows] = x[rows] - sums
    return x


def apply_block_diagonal(dinv, y):
    """z_I = dinv[I] @ y_I (trisolve.py:148-166)."""
    n, bs = dinv.shape[0], dinv.shape[1]
    return np.matmul(dinv, np.asarray(y, dtype=np.float64).reshape(n, bs, 1)).reshape(-1)


# ----------------------------------------------------------------------------
# the whole preconditioner (factor.py:302-323, trisolve.py:169-182)
# ----------------------------------------------------------------------------

class OracleFactors:
    """Everything ``build_preconditioner`` produces, as plain arrays."""

    def __init__(self, n, bs, split, pattern_rows):
        self.n, self.bs = n, bs
        self.pattern_rows = pattern_rows
        self.__dict__.update(split)
        m = n * bs
        self.lo = csr_expand(n, bs, split["L_rp"], split["L_ci"], split["L_vals"])
        self.up = csr_expand(n, bs, split["U_rp"], split["U_ci"], split["U_vals"])
        self.lo_level_of_row, self.lo_levels = level_schedule(m, self.lo[0], self.lo[1], "lower")
        self.up_level_of_row, self.up_levels = level_schedule(m, self.up[0], self.up[1], "upper")

    def apply(self, b):
        """x = U'^{-1} D^{-1} L^{-1} b (Alg. 7; trisolve.py:169-182)."""
        b = np.asarray(b, dtype=np.float64)
        if b.shape != (self.n * self.bs,):
            raise ValueError("right-hand side length mismatch")
        y = solve_unit_triangular(self.n * self.bs, *self.lo, self.lo_levels, b)
        z = apply_block_diagonal(self.dinv, y)
        return solve_unit_triangular(self.n * self.bs, *self.up, self.up_levels, z)


def build_preconditioner(n, bs, rp, ci, vals, k):
    """extract-pattern -> symbolic -> materialize -> factorize -> split (factor.py:302-323)."""
    rp = np.asarray(rp, dtype=np.int64)
    ci = np.asarray(ci, dtype=np.int64)
    rows = [ci[rp[i]:rp[i + 1]].tolist() for i in range(n)]
    prows = symbolic_phase(n, rows, k)
    prp, pci, pv = materialize(n, bs, rp, ci, vals, prows)
    fv, _ = block_ilu0(n, bs, prp, pci, pv)
    split = split_ldu(n, bs, prp, pci, fv)
    return OracleFactors(n, bs, split, prows)


# ----------------------------------------------------------------------------
# SpMV (sparse.py:278-301) on BSR, and Krylov drivers
# ----------------------------------------------------------------------------

def bsr_spmv(n, bs, rp, ci, vals, x):
    """y = A x for BSR A (point-wise result identical up to summation order)."""
    blk = blocks_of(vals, bs)
    xb = np.asarray(x, dtype=np.float64).reshape(-1, bs)
    prod = np.einsum("nrc,nc->nr", blk, xb[np.asarray(ci, dtype=np.int64)])
    rp = np.asarray(rp, dtype=np.int64)
    y = np.zeros((n, bs))
    nz = np.diff(rp) > 0
    if prod.shape[0]:
        y[nz] = np.add.reduceat(prod, rp[:-1][nz], axis=0)
    return y.reshape(-1)


def gmres(matvec, b, precond=None, restart=20, max_iters=10000, rel_tol=1e-6, abs_tol=1e-30):
    """Left-preconditioned restarted GMRES(m) with MGS + Givens (gmres.py:76-186).

    Returns (x, iterations, converged, final_rel_residual, history).
    """
    M = precond if precond is not None else (lambda v: v)
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    if n == 0 or bnorm == 0.0:
        return x, 0, True, 0.0, []
    mbnorm = float(np.linalg.norm(M(b)))
    if mbnorm == 0.0:
        mbnorm = bnorm
    target = rel_tol
    its = 0
    hist = []
    breakdown = False
    while its < max_iters and not breakdown:
        z = M(b - matvec(x))
        beta = float(np.linalg.norm(z))
        hist.append(beta / mbnorm)
        if beta / mbnorm <= target or beta <= abs_tol:
            if float(np.linalg.norm(b - matvec(x))) / bnorm <= rel_tol:
                break
            target *= 0.25
            if target < 1e-16:
                break
            continue
        V = np.zeros((restart + 1, n))
        V[0] = z / beta
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        used = 0
        while used < restart and its < max_iters:
            j = used
            w = M(matvec(V[j]))
            its += 1
            for i in range(j + 1):
                H[i, j] = float(V[i] @ w)
                w = w - H[i, j] * V[i]
            hn = float(np.linalg.norm(w))
            H[j + 1, j] = hn
            for i in range(j):
                a_, b_ = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a_ + sn[i] * b_
                H[i + 1, j] = -sn[i] * a_ + cs[i] * b_
            den = math.hypot(H[j, j], H[j + 1, j])
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            used = j + 1
            est = abs(g[j + 1]) / mbnorm
            hist.append(est)
            if hn <= abs_tol:
                breakdown = True
                break
            V[j + 1] = w / hn
            if est <= target:
                break
        if used:
            y = np.zeros(used)
            for i in range(used - 1, -1, -1):
                acc = g[i] - H[i, i + 1:used] @ y[i + 1:used]
                y[i] = acc / H[i, i] if H[i, i] != 0.0 else 0.0
            x = x + V[:used].T @ y
    rel = float(np.linalg.norm(b - matvec(x))) / bnorm
    return x, its, rel <= rel_tol, rel, hist


def bicgstab(matvec, b, precond=None, max_iters=10000, rel_tol=1e-6):
    """Right-preconditioned BiCGSTAB -- the contract this repo DEFINES.

    x0 = 0, r0 = b, shadow residual r^ = r0.  Per iteration i = 1, 2, ...::

        rho_i  = <r^, r>;       beta = (rho_i / rho_{i-1}) (alpha / omega)
        p      = r + beta (p - omega v)
        p^     = M p;  v = A p^;  alpha = rho_i / <r^, v>
        s      = r - alpha v
        if ||s|| / ||b|| <= tol:  x += alpha p^  -> stop (half step counts as a full iteration i)
        s^     = M s;  t = A s^;  omega = <t, s> / <t, t>
        x     += alpha p^ + omega s^;  r = s - omega t
        if ||r|| / ||b|| <= tol:  stop

    Breakdown (rho_i == 0, <r^, v> == 0 or <t, t> == 0) stops early.  The
    reported residual is the TRUE relative residual ||b - A x|| / ||b|| and
    ``converged`` is that <= tol.  Returns (x, iterations, converged, rel, history)
    where history holds the recurrence residuals ||r|| / ||b|| (or ||s||/||b||
    at a half-step exit) per iteration.
    """
    M = precond if precond is not None else (lambda v: v)
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    x = np.zeros(n)
    bnorm = float(np.linalg.norm(b))
    if n == 0 or bnorm == 0.0:
        return x, 0, True, 0.0, []
    r = b.copy()
    rh = r.copy()
    rho_prev = alpha = omega = 1.0
    v = np.zeros(n)
    p = np.zeros(n)
    hist = []
    its = 0
    for it in range(1, max_iters + 1):
        rho = float(rh @ r)
        if rho == 0.0:
            break
        beta = (rho / rho_prev) * (alpha / omega)
        rho_prev = rho
        p = r + beta * (p - omega * v)
        ph = M(p)
        v = matvec(ph)
        rv = float(rh @ v)
        if rv == 0.0:
            break
        alpha = rho / rv
        s = r - alpha * v
        its = it
        sn = float(np.linalg.norm(s)) / bnorm
        if sn <= rel_tol:
            x = x + alpha * ph
            hist.append(sn)
            break
        sh = M(s)
        t = matvec(sh)
        tt = float(t @ t)
        if tt == 0.0:
            x = x + alpha * ph
            hist.append(sn)
            break
        omega = float(t @ s) / tt
        x = x + alpha * ph + omega * sh
        r = s - omega * t
        rn = float(np.linalg.norm(r)) / bnorm
        hist.append(rn)
        if rn <= rel_tol:
            break
        if omega == 0.0:
            break
    rel = float(np.linalg.norm(b - matvec(x))) / bnorm
    return x, its, rel <= rel_tol, rel, hist
