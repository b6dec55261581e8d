"""The drop-in surface on CPU: every name the reference package exports
(blockiluk/__init__.py:51-86) exists here, and the coupled ILU(k) oracle of the
reference's public API (symbolic.py:75-122) agrees with the two-phase pattern."""

import numpy as np

from conftest import golden_files, load_golden

REFERENCE_ALL = [   # blockiluk/__init__.py:51-86
    "BcsrMatrix", "BlockIlukFactors", "CsrMatrix", "FactorizationError", "LevelSchedule", "MatrixMarketError",
    "PatternMatrix", "SingularBlockError", "SolveStats", "SolverConfig", "StructuralError", "TriangularOperand",
    "apply_block_diagonal", "apply_preconditioner", "assemble_csr", "bcsr_from_csr", "block_ilu0_factorize",
    "block_invert", "build_level_schedule", "build_preconditioner", "coupled_iluk_oracle", "csr_expand",
    "csr_from_triplets", "extract_point_pattern", "gen_poisson_3d", "gmres", "point_ilu0_factorize",
    "read_matrix_market", "solve_unit_triangular", "split_ldu", "spmv", "strict_triangle", "symbolic_phase",
    "__version__",
]


def test_reference_all_is_exported():
    import paper_1703_01325_b200 as b2
    missing = [n for n in REFERENCE_ALL if n not in b2.__all__ or not hasattr(b2, n)]
    assert not missing, missing


def test_reference_module_paths():
    from paper_1703_01325_b200 import factor, symbolic, trisolve
    for mod, names in ((factor, ["block_invert", "materialize", "point_ilu0_factorize", "block_ilu0_factorize",
                                 "split_ldu", "build_preconditioner", "BlockIlukFactors"]),
                       (trisolve, ["solve_unit_triangular", "apply_block_diagonal", "apply_preconditioner",
                                   "build_level_schedule", "LevelSchedule", "TriangularOperand"]),
                       (symbolic, ["symbolic_phase", "coupled_iluk_oracle"])):
        for n in names:
            assert hasattr(mod, n), (mod.__name__, n)


def test_coupled_oracle_pattern_equals_symbolic_phase():
    """reference test_symbolic.py:86-95: the coupled single pass and the
    two-phase pipeline agree on the pattern, and on point ILU(k) values."""
    import paper_1703_01325_b200 as b2
    from oracle import iluk_oracle as orc
    for path in golden_files():
        g = load_golden(path)
        if int(g["bs"]) != 1 or int(g["n"]) > 150:
            continue
        n, k = int(g["n"]), int(g["k"])
        a = b2.CsrMatrix(n, n, g["rp"], g["ci"], g["vals"])
        fac, pat = b2.coupled_iluk_oracle(a, k)
        assert np.array_equal(pat.to_csr_arrays()[0], g["P_rp"]) and np.array_equal(pat.to_csr_arrays()[1],
                                                                                       g["P_ci"])
        prp, pci, pv = orc.materialize(n, 1, g["rp"], g["ci"], g["vals"], pat.rows)
        fv, _ = orc.block_ilu0(n, 1, prp, pci, pv)
        assert np.allclose(fac.values, fv, rtol=1e-12, atol=1e-14)
    # k = n equals Gaussian elimination fill (reference test_symbolic.py:76-84)
    d = np.array([[4.0, 1, 0, 1], [1, 4, 1, 0], [0, 1, 4, 1], [1, 0, 1, 4]])
    r, c = np.nonzero(d)
    a = b2.CsrMatrix(4, 4, np.concatenate([[0], np.cumsum(np.bincount(r, minlength=4))]), c, d[r, c])
    fac, pat = b2.coupled_iluk_oracle(a, 4)
    lu = np.zeros((4, 4))
    rows = np.repeat(np.arange(4), np.diff(fac.row_ptr))
    lu[rows, fac.col_idx] = fac.values
    lo = np.tril(lu, -1) + np.eye(4)
    assert np.allclose(lo @ np.triu(lu), d)
