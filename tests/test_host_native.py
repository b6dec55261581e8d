"""CPU tests of libbiluk's host side (no GPU needed): the library loads and
exports every symbol of include/biluk.h, and the integer work -- symbolic
phase, level schedules, plan analysis -- is exactly the reference's.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_files, load_golden
from oracle import iluk_oracle as orc
import paper_1703_01325_b200 as b2
from paper_1703_01325_b200 import _native as nat

CASES = golden_files()
IDS = [os.path.basename(p)[:-4] for p in CASES]


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "biluk.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]*?\b(biluk_\w+)\s*\(", header, re.M))
    declared = {d for d in declared if not d.endswith("_fn")}
    lib = nat.lib()
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared <= set(nat.declared_symbols()) | {"biluk_precond_fn"}
    assert len(declared) >= 25


@pytest.mark.parametrize("path", CASES, ids=IDS)
def test_symbolic_phase_matches_reference(path):
    g = load_golden(path)
    n, k = int(g["n"]), int(g["k"])
    pat = b2.PatternMatrix.from_csr_arrays(n, g["rp"], g["ci"])
    got = b2.symbolic_phase(pat, k)
    rp, ci = got.to_csr_arrays()
    assert np.array_equal(rp, g["P_rp"]) and np.array_equal(ci, g["P_ci"])


@pytest.mark.parametrize("path", CASES, ids=IDS)
def test_point_level_schedules_match_reference(path):
    g = load_golden(path)
    n, bs = int(g["n"]), int(g["bs"])
    Lm = b2.BcsrMatrix(bs, n, n, g["L_rp"], g["L_ci"], g["L_vals"])
    Um = b2.BcsrMatrix(bs, n, n, g["U_rp"], g["U_ci"], g["U_vals"])
    lo = b2.TriangularOperand(b2.csr_expand(Lm), "lower")
    up = b2.TriangularOperand(b2.csr_expand(Um), "upper")
    assert lo.matrix.nnz == int(g["lo_nnz"]) and up.matrix.nnz == int(g["up_nnz"])
    sl = b2.build_level_schedule(lo)
    su = b2.build_level_schedule(up)
    assert np.array_equal(sl.level_of_row, g["lo_level_of_row"]) and sl.num_levels == int(g["lo_num_levels"])
    assert np.array_equal(su.level_of_row, g["up_level_of_row"]) and su.num_levels == int(g["up_num_levels"])
    # csr_expand agrees with the oracle's restatement entry for entry
    prp, pci, pv = orc.csr_expand(n, bs, g["L_rp"], g["L_ci"], g["L_vals"])
    assert np.array_equal(prp, lo.matrix.row_ptr) and np.array_equal(pci, lo.matrix.col_idx)
    assert np.array_equal(pv, lo.matrix.values)


def _random_pattern(rng, n, offdiag=3):
    # same recipe as reference tests/helpers.py:31-39
    rows = []
    for i in range(n):
        m = min(int(rng.integers(0, offdiag + 1)), n - 1)
        picks = rng.permutation(n - 1)[:m]
        picks = picks + (picks >= i)
        rows.append(sorted({i, *(int(j) for j in picks)}))
    return rows


def _ge_fill(rows, n):
    filled = np.zeros((n, n), dtype=bool)
    for i, r in enumerate(rows):
        filled[i, r] = True
    for p in range(n):
        for i in range(p + 1, n):
            if filled[i, p]:
                filled[i, p + 1:] |= filled[p, p + 1:]
    return filled


def test_symbolic_random_patterns_vs_oracle_and_ge_fill():
    rng = np.random.default_rng(808)
    for _ in range(60):
        n = int(rng.integers(5, 90))
        rows = _random_pattern(rng, n)
        pat = b2.PatternMatrix(n, rows)
        prev = None
        for k in range(4):
            got = b2.symbolic_phase(pat, k).rows
            assert got == orc.symbolic_phase(n, rows, k)
            cur = {(i, j) for i, r in enumerate(got) for j in r}
            assert prev is None or prev <= cur     # monotone in k (acceptance 08)
            prev = cur
        full = b2.symbolic_phase(pat, n)
        dense = np.zeros((n, n), dtype=bool)
        for i, r in enumerate(full.rows):
            dense[i, r] = True
        assert np.array_equal(dense, _ge_fill(rows, n))


def test_symbolic_known_answers_and_errors():
    grid = b2.PatternMatrix(4, [[0, 1, 2], [0, 1, 3], [0, 2, 3], [1, 2, 3]])
    assert b2.symbolic_phase(grid, 0) == grid
    assert b2.symbolic_phase(grid, 1).as_set() - grid.as_set() == {(1, 2), (2, 1)}
    tri = b2.PatternMatrix(7, [sorted({max(i - 1, 0), i, min(i + 1, 6)}) for i in range(7)])
    for k in range(5):
        assert b2.symbolic_phase(tri, k) == tri
    arrow = b2.PatternMatrix(5, [list(range(5))] + [sorted({0, i}) for i in range(1, 5)])
    assert b2.symbolic_phase(arrow, 1).nnz == 25
    with pytest.raises(b2.StructuralError):
        b2.symbolic_phase(b2.PatternMatrix(2, [[0, 1], [0]]), 1)
    with pytest.raises(ValueError):
        b2.symbolic_phase(grid, -1)


def test_level_schedule_known_answers():
    chain = b2.csr_from_triplets(5, 5, [(i, i - 1, -1.0) for i in range(1, 5)])
    s = b2.build_level_schedule(b2.TriangularOperand(chain, "lower"))
    assert s.num_levels == 5 and s.level_of_row.tolist() == [1, 2, 3, 4, 5]
    assert [r.tolist() for r in s.levels] == [[0], [1], [2], [3], [4]]
    flat = b2.build_level_schedule(b2.TriangularOperand(b2.csr_from_triplets(4, 4, []), "lower"))
    assert flat.num_levels == 1 and flat.levels[0].tolist() == [0, 1, 2, 3]
    # 2-D grid wavefronts nx + ny - 1 (reference acceptance 05)
    from paper_1703_01325_b200.synthetic import poisson7_pattern
    for nx, ny in ((5, 5), (10, 10), (13, 7)):
        rp, ci = poisson7_pattern(nx, ny, 1)
        a = b2.CsrMatrix(nx * ny, nx * ny, rp, ci, np.ones(ci.size))
        assert b2.build_level_schedule(b2.strict_triangle(a, "lower")).num_levels == nx + ny - 1
    with pytest.raises(b2.StructuralError):
        b2.TriangularOperand(b2.csr_from_triplets(2, 2, [(0, 1, 1.0)]), "lower")


@pytest.mark.parametrize("path", CASES[:6], ids=IDS[:6])
def test_plan_analysis_counts(path):
    """biluk_plan_create (host only) sizes L / U' and their block level sets like the oracle."""
    g = load_golden(path)
    n, bs, k = int(g["n"]), int(g["bs"]), int(g["k"])
    L = nat.lib()
    h = ctypes.c_void_p()
    err = ctypes.c_int64(-1)
    rp = np.ascontiguousarray(g["rp"], np.int64)
    ci = np.ascontiguousarray(g["ci"], np.int64)
    nat.check(L.biluk_plan_create(bs, n, rp.ctypes.data, ci.ctypes.data, k, ctypes.byref(h), ctypes.byref(err)))
    try:
        info = (ctypes.c_int64 * 20)()
        nat.check(L.biluk_plan_info(h, info, 20))
        assert info[0] == n and info[1] == bs and info[4] == g["P_ci"].size
        assert info[5] == g["L_ci"].size and info[6] == g["U_ci"].size
        # block levels: the Eq. (4) recurrence on the block triangles
        lev_l, nl = orc.level_schedule(n, g["L_rp"], g["L_ci"], "lower")[0], None
        assert info[7] == int(lev_l.max()) if n else 0
        lev_u = orc.level_schedule(n, g["U_rp"], g["U_ci"], "upper")[0]
        assert info[8] == int(lev_u.max())
        b = bs
        nLU = g["L_ci"].size + g["U_ci"].size
        assert info[13] == 8 * b * b * (nLU + n) + 4 * nLU + 8 * (n + 1) + 32 * b * n
    finally:
        L.biluk_plan_destroy(h)


def test_plan_create_structural_errors():
    L = nat.lib()
    h = ctypes.c_void_p()
    err = ctypes.c_int64(-1)
    rp = np.array([0, 1, 2], np.int64)
    ci = np.array([1, 0], np.int64)      # no diagonal in row 0
    rc = L.biluk_plan_create(2, 2, rp.ctypes.data, ci.ctypes.data, 0, ctypes.byref(h), ctypes.byref(err))
    assert rc == nat.ESTRUCT and err.value == 0
    with pytest.raises(b2.StructuralError, match="symbolic-phase: row 0 has no diagonal entry"):
        nat.check(rc, stage="symbolic-phase")
    rc = L.biluk_plan_create(2, 2, rp.ctypes.data, ci.ctypes.data, -1, ctypes.byref(h), ctypes.byref(err))
    assert rc == nat.EARG


def test_partitioned_sweep_plan_geometry():
    """Structured grids get (y, z) column parts, other patterns contiguous ranges;
    every record's static ring place and issue point are consistent (host only)."""
    import ctypes
    L = nat.lib()
    for nx, expect_kind in ((24, 1), (0, 0)):
        if nx:
            n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, 3, seed=0)
        else:
            rng = np.random.default_rng(0)
            n, bs = 3000, 3
            rows = [sorted(set(rng.choice(n, 5, replace=False).tolist()) | {i}) for i in range(n)]
            rp = np.zeros(n + 1, np.int64)
            rp[1:] = np.cumsum([len(r) for r in rows])
            ci = np.array([c for r in rows for c in r], np.int64)
        h = ctypes.c_void_p()
        err = ctypes.c_int64(-1)
        rp = np.ascontiguousarray(rp, np.int64)
        ci = np.ascontiguousarray(ci, np.int64)
        nat.check(L.biluk_plan_create(bs, n, nat.ptr(rp), nat.ptr(ci), 0, ctypes.byref(h), ctypes.byref(err)))
        try:
            from paper_1703_01325_b200.factor import _INFO_KEYS
            buf = (ctypes.c_int64 * len(_INFO_KEYS))()
            L.biluk_plan_info(h, buf, len(_INFO_KEYS))
            info = dict(zip(_INFO_KEYS, list(buf)))
            assert info["engine"] == 1 and info["partition"] == expect_kind
            if expect_kind == 1:
                assert info["split_y"] * info["split_z"] == info["parts"] <= 148
            nrec = L.biluk_plan_records(h, None, 0)
            assert nrec == info["records"] > 0
        finally:
            L.biluk_plan_destroy(h)


def test_block_diagonal_batch_assembly():
    """Batch assembly: offsets, values and the decoupled ILU(k) pattern."""
    ms = [b2.reservoir_block_grid(3 + s, 3, 2, 2, seed=s) for s in range(3)]
    big = b2.block_diagonal([b2.BcsrMatrix(bs, n, n, rp, ci, v) for n, bs, rp, ci, v in ms])
    assert big.shape == (sum(n for n, *_ in ms) * 2,) * 2
    assert big.batch_segments.tolist() == [0, ms[0][0], ms[0][0] + ms[1][0], sum(n for n, *_ in ms)]
    r = z = 0
    for n, bs, rp, ci, v in ms:
        assert np.array_equal(big.row_ptr[r:r + n + 1] - big.row_ptr[r], rp)
        assert np.array_equal(big.col_idx[z:z + rp[-1]] - r, ci)
        assert np.array_equal(big.values[z * 4:(z + rp[-1]) * 4], v)
        r += n
        z += rp[-1]
    # the symbolic phase of the batch is the per-system patterns, shifted
    pb = b2.symbolic_phase(b2.PatternMatrix.from_csr_arrays(big.num_block_rows, big.row_ptr, big.col_idx), 1)
    rb, cb = pb.to_csr_arrays()
    r = z = 0
    for n, bs, rp, ci, v in ms:
        p1 = b2.symbolic_phase(b2.PatternMatrix.from_csr_arrays(n, rp, ci), 1)
        r1, c1 = p1.to_csr_arrays()
        assert np.array_equal(rb[r:r + n + 1] - rb[r], r1) and np.array_equal(cb[rb[r]:rb[r + n]] - r, c1)
        r += n
    with pytest.raises(b2.StructuralError):
        b2.block_diagonal([b2.BcsrMatrix(2, 1, 1, [0, 1], [0], np.ones(4)), b2.BcsrMatrix(3, 1, 1, [0, 1], [0], np.ones(9))])
