"""The reference's sub-stage entry points (blockiluk/__init__.py:51-86) on the GPU,
against the reference goldens and the oracle.

block_invert (factor.py:38-70), materialize (:83-121), point_ilu0_factorize
(:151-162), block_ilu0_factorize (:165-205), split_ldu (:230-289),
solve_unit_triangular (trisolve.py:121-145), apply_block_diagonal (:148-166).
"""

import os

import numpy as np
import pytest

from conftest import golden_files, load_golden, rel_err
from oracle import iluk_oracle as orc

pytestmark = pytest.mark.gpu

CASES = golden_files()
IDS = [os.path.basename(p)[:-4] for p in CASES]
TOL = 1e-12


@pytest.fixture(scope="module")
def b2(cuda_ok):
    import paper_1703_01325_b200 as mod
    return mod


def test_block_invert_known_answers_and_singular(b2):
    # reference test_factor.py:20-22
    assert np.allclose(b2.block_invert([[1.0, 2.0], [3.0, 4.0]]), [[-2.0, 1.0], [1.5, -0.5]], rtol=0, atol=1e-15)
    assert np.allclose(b2.block_invert([[4.0]]), [[0.25]])
    with pytest.raises(b2.SingularBlockError):
        b2.block_invert(np.zeros((3, 3)))
    with pytest.raises(b2.SingularBlockError):
        b2.block_invert([[1.0, 2.0], [2.0, 4.0]])
    with pytest.raises(b2.StructuralError):
        b2.block_invert(np.ones((2, 3)))
    rng = np.random.default_rng(0)
    for bs in range(1, 9):
        stack = rng.standard_normal((50, bs, bs)) + 3.0 * np.eye(bs)
        got = b2.block_invert(stack)
        want = np.stack([orc.block_invert(m) for m in stack])
        assert rel_err(got, want) <= 1e-13, bs


@pytest.mark.parametrize("path", CASES, ids=IDS)
def test_stage_pipeline_matches_reference(b2, path):
    """materialize -> block_ilu0_factorize -> split_ldu, stage by stage, equals
    the reference's factors; the split factors apply like build_preconditioner's."""
    g = load_golden(path)
    n, bs, k = int(g["n"]), int(g["bs"]), int(g["k"])
    a = b2.BcsrMatrix(bs, n, n, g["rp"], g["ci"], g["vals"])
    pat = b2.symbolic_phase(b2.PatternMatrix.from_csr_arrays(n, g["rp"], g["ci"]), k)
    assert np.array_equal(pat.to_csr_arrays()[0], g["P_rp"]) and np.array_equal(pat.to_csr_arrays()[1], g["P_ci"])
    ap = b2.materialize(a, pat)
    prp, pci, pv = orc.materialize(n, bs, g["rp"], g["ci"], g["vals"], pat.rows)
    assert np.array_equal(ap.row_ptr, prp) and np.array_equal(ap.col_idx, pci)
    assert np.array_equal(ap.values, pv)                 # a copy: bit-exact
    before = a.values.copy()
    fac = b2.block_ilu0_factorize(ap)
    assert fac is ap and np.array_equal(a.values, before)
    want_fv, _ = orc.block_ilu0(n, bs, prp, pci, pv)
    assert rel_err(ap.values, want_fv) <= TOL
    f = b2.split_ldu(ap)
    assert np.array_equal(f.L.row_ptr, g["L_rp"]) and np.array_equal(f.uprime.col_idx, g["U_ci"])
    assert rel_err(f.L.values, g["L_vals"]) <= TOL
    assert rel_err(f.uprime.values, g["U_vals"]) <= TOL
    assert rel_err(f.dinv, g["dinv"]) <= TOL
    assert rel_err(b2.apply_preconditioner(f, g["rhs"]), g["apply_out"]) <= TOL
    # the two triangular solves and the block diagonal, stage by stage (Alg. 7)
    y = b2.solve_unit_triangular(f.lower_op, f.lower_schedule, g["rhs"])
    z = b2.apply_block_diagonal(f.dinv, y)
    x = b2.solve_unit_triangular(f.upper_op, f.upper_schedule, z)
    assert rel_err(x, g["apply_out"]) <= TOL
    yo = orc.solve_unit_triangular(n * bs, *orc.csr_expand(n, bs, g["L_rp"], g["L_ci"], g["L_vals"]),
                                   orc.level_schedule(n * bs, *orc.csr_expand(n, bs, g["L_rp"], g["L_ci"],
                                                                               g["L_vals"])[:2], "lower")[1],
                                   g["rhs"])
    assert rel_err(y, yo) <= TOL
    assert rel_err(z, orc.apply_block_diagonal(g["dinv"], y)) <= 1e-14


def test_point_ilu0_known_answer_and_errors(b2):
    # reference test_factor.py:51-54: [[4, 2], [0.5, 2]] -> l21 = 0.125, u22 = 1.75
    a = b2.CsrMatrix(2, 2, [0, 2, 4], [0, 1, 0, 1], [4.0, 2.0, 0.5, 2.0])
    b2.point_ilu0_factorize(a)
    assert np.allclose(a.values, [4.0, 2.0, 0.125, 1.75], rtol=0, atol=1e-15)
    z = b2.CsrMatrix(2, 2, [0, 2, 4], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0])
    with pytest.raises(b2.FactorizationError) as ei:
        b2.point_ilu0_factorize(z)
    assert ei.value.row == 1
    nodiag = b2.CsrMatrix(2, 2, [0, 1, 2], [0, 0], [1.0, 1.0])
    with pytest.raises(b2.StructuralError):
        b2.point_ilu0_factorize(nodiag)
    # block singular diagonal reports its row (reference test_factor.py:145-155)
    blk = b2.BcsrMatrix(2, 2, 2, [0, 2, 4], [0, 1, 0, 1],
                        np.concatenate([np.eye(2).ravel(), np.eye(2).ravel(), np.eye(2).ravel(),
                                        np.eye(2).ravel()]))
    with pytest.raises(b2.SingularBlockError) as ei:
        b2.block_ilu0_factorize(blk)
    assert ei.value.row == 1


def test_materialize_and_split_errors(b2):
    a = b2.CsrMatrix(3, 3, [0, 2, 3, 5], [0, 2, 1, 0, 2], [1.0, 2.0, 3.0, 4.0, 5.0])
    with pytest.raises(b2.StructuralError, match=r"\(0, 2\)"):
        b2.materialize(a, b2.PatternMatrix(3, [[0], [1], [0, 2]]))
    with pytest.raises(b2.StructuralError):
        b2.split_ldu(b2.BcsrMatrix(1, 2, 2, [0, 1, 1], [0], [1.0]))
    sing = b2.BcsrMatrix(2, 2, 2, [0, 1, 2], [0, 1], np.concatenate([np.eye(2).ravel(), np.zeros(4)]))
    with pytest.raises(b2.SingularBlockError) as ei:
        b2.split_ldu(sing)
    assert ei.value.row == 1


def test_solve_unit_triangular_contract(b2):
    """Chain solves (reference test_trisolve.py:53-104 style), the schedule check
    and an untouched right-hand side."""
    n = 6
    rp = np.concatenate([[0], np.arange(n)])   # row i > 0 holds (i, i-1) = -1
    t = b2.TriangularOperand(b2.CsrMatrix(n, n, rp, np.arange(n - 1), np.full(n - 1, -1.0)), "lower")
    s = b2.build_level_schedule(t)
    b = np.ones(n)
    x = b2.solve_unit_triangular(t, s, b)
    assert np.allclose(x, np.arange(1, n + 1)) and np.array_equal(b, np.ones(n))
    other = b2.TriangularOperand(b2.CsrMatrix(n, n, rp, np.arange(n - 1), np.full(n - 1, -1.0)), "lower")
    with pytest.raises(b2.StructuralError):
        b2.solve_unit_triangular(other, s, b)
    with pytest.raises(ValueError):
        b2.solve_unit_triangular(t, s, np.ones(n + 1))
    with pytest.raises(ValueError):
        b2.apply_block_diagonal(np.ones((2, 2, 2)), np.ones(5))
