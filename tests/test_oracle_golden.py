"""Pin the CPU oracle (oracle/iluk_oracle.py) against the reference's own outputs.

The golden .npz files were produced by running the reference package itself
(tests/golden/make_golden.py).  Tolerances: integer structure exact; factors
and preconditioned vectors 1e-12 relative (the north-star bar); Krylov
iteration counts within +-1 (in practice identical).
"""

import os

import numpy as np
import pytest

from conftest import golden_files, load_golden, rel_err
from oracle import iluk_oracle as orc

CASES = golden_files()


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(p)[:-4] for p in CASES])
def test_oracle_matches_reference_golden(path):
    g = load_golden(path)
    n, bs, k = int(g["n"]), int(g["bs"]), int(g["k"])
    rows = [g["ci"][g["rp"][i]:g["rp"][i + 1]].tolist() for i in range(n)]
    prows = orc.symbolic_phase(n, rows, k)
    prp = np.zeros(n + 1, np.int64)
    prp[1:] = np.cumsum([len(r) for r in prows])
    assert np.array_equal(prp, g["P_rp"])
    assert np.array_equal(np.concatenate(prows), g["P_ci"])

    f = orc.build_preconditioner(n, bs, g["rp"], g["ci"], g["vals"], k)
    assert np.array_equal(f.L_rp, g["L_rp"]) and np.array_equal(f.L_ci, g["L_ci"])
    assert np.array_equal(f.U_rp, g["U_rp"]) and np.array_equal(f.U_ci, g["U_ci"])
    assert rel_err(f.L_vals, g["L_vals"]) <= 1e-12
    assert rel_err(f.U_vals, g["U_vals"]) <= 1e-12
    assert rel_err(f.dinv, g["dinv"]) <= 1e-12
    # point-wise schedules on the zero-dropped expansions: exact
    assert np.array_equal(f.lo_level_of_row, g["lo_level_of_row"])
    assert np.array_equal(f.up_level_of_row, g["up_level_of_row"])
    assert f.lo[0][-1] == int(g["lo_nnz"]) and f.up[0][-1] == int(g["up_nnz"])

    z = f.apply(g["rhs"])
    assert rel_err(z, g["apply_out"]) <= 1e-12
    ax = orc.bsr_spmv(n, bs, g["rp"], g["ci"], g["vals"], np.ones(n * bs))
    # A @ 1 cancels heavily (row sums of a diagonally dominant operator): scale
    # the error by |A| @ |1| instead of by the (small) result
    absax = orc.bsr_spmv(n, bs, g["rp"], g["ci"], np.abs(g["vals"]), np.ones(n * bs))
    assert np.abs(ax - g["spmv_ones"]).max() <= 1e-14 * absax.max()

    mv = lambda v: orc.bsr_spmv(n, bs, g["rp"], g["ci"], g["vals"], v)  # noqa: E731
    b = g["spmv_ones"]
    _, its, conv, rel, _ = orc.gmres(mv, b, f.apply, restart=30, rel_tol=1e-6)
    assert abs(its - int(g["gmres_iters"])) <= 1 and conv == bool(g["gmres_conv"])
    _, its, conv, rel, _ = orc.bicgstab(mv, b, f.apply, rel_tol=1e-6)
    assert abs(its - int(g["bicg_iters"])) <= 1 and conv == bool(g["bicg_conv"])


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(p)[:-4] for p in CASES])
def test_c_oracle_matches_reference_golden(path):
    """The C restatement (oracle/coracle.c) used at full size is pinned the same way."""
    from oracle import coracle
    g = load_golden(path)
    n, bs, k = int(g["n"]), int(g["bs"]), int(g["k"])
    cf = coracle.CFactors(n, bs, g["rp"], g["ci"], g["vals"], k)
    assert np.array_equal(cf.L_rp, g["L_rp"]) and np.array_equal(cf.L_ci, g["L_ci"])
    assert np.array_equal(cf.U_rp, g["U_rp"]) and np.array_equal(cf.U_ci, g["U_ci"])
    assert rel_err(cf.L_vals, g["L_vals"]) <= 1e-12
    assert rel_err(cf.U_vals, g["U_vals"]) <= 1e-12
    assert rel_err(cf.dinv, g["dinv"]) <= 1e-12
    assert np.array_equal(cf.lo_level_of_row, g["lo_level_of_row"])
    assert np.array_equal(cf.up_level_of_row, g["up_level_of_row"])
    assert cf.plnnz == int(g["lo_nnz"]) and cf.punnz == int(g["up_nnz"])
    assert rel_err(cf.apply(g["rhs"]), g["apply_out"]) <= 1e-12
    from oracle import cbaseline
    assert rel_err(cbaseline.PortApply(cf)(g["rhs"]), g["apply_out"]) <= 1e-12
    ax = coracle.bsr_spmv(n, bs, g["rp"], g["ci"], g["vals"], np.ones(n * bs))
    absax = coracle.bsr_spmv(n, bs, g["rp"], g["ci"], np.abs(g["vals"]), np.ones(n * bs))
    assert np.abs(ax - g["spmv_ones"]).max() <= 1e-14 * absax.max()


def test_c_oracle_errors():
    from oracle import coracle
    # singular leading 2x2 block (reference test_factor.py:145-155) -> code 2, row 0
    rp = np.array([0, 2, 4], np.int64)
    ci = np.array([0, 1, 0, 1], np.int64)
    blk = np.zeros((4, 2, 2))
    blk[0] = [[1.0, 2.0], [2.0, 4.0]]
    blk[2] = np.eye(2)
    blk[3] = np.eye(2)
    vals = blk.transpose(0, 2, 1).reshape(-1)
    with pytest.raises(coracle.COracleError) as exc:
        coracle.CFactors(2, 2, rp, ci, vals, 0)
    assert exc.value.code == 2 and exc.value.row == 0
    # missing diagonal -> structural, row 0
    with pytest.raises(coracle.COracleError) as exc:
        coracle.CFactors(2, 1, np.array([0, 1, 2], np.int64), np.array([1, 0], np.int64), np.ones(2), 0)
    assert exc.value.code == 1 and exc.value.row == 0


def test_block_invert_known_answers():
    # reference test_factor.py:20-48
    inv = orc.block_invert(np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert np.allclose(inv, [[-2.0, 1.0], [1.5, -0.5]], rtol=1e-14, atol=1e-14)
    assert orc.block_invert(np.array([[4.0]]))[0, 0] == 0.25
    b = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.allclose(orc.block_invert(b), b, atol=1e-15)
    with pytest.raises(orc.OracleSingularBlock):
        orc.block_invert(np.array([[1.0, 2.0], [2.0, 4.0]]))
    with pytest.raises(orc.OracleSingularBlock):
        orc.block_invert(np.array([[0.0]]))


def test_symbolic_known_answers():
    # reference test_symbolic.py:11-53
    grid = [[0, 1, 2], [0, 1, 3], [0, 2, 3], [1, 2, 3]]
    got = orc.symbolic_phase(4, grid, 1)
    added = {(i, j) for i, r in enumerate(got) for j in r} - {(i, j) for i, r in enumerate(grid) for j in r}
    assert added == {(1, 2), (2, 1)}
    tri = [sorted({max(i - 1, 0), i, min(i + 1, 6)}) for i in range(7)]
    for k in range(5):
        assert orc.symbolic_phase(7, tri, k) == tri
    arrow = [list(range(5))] + [sorted({0, i}) for i in range(1, 5)]
    assert sum(len(r) for r in orc.symbolic_phase(5, arrow, 1)) == 25
    with pytest.raises(orc.OracleStructuralError):
        orc.symbolic_phase(2, [[0, 1], [0]], 1)
