"""Full-size parity (BASELINE configs[1..3]) against the C restatement of the
reference (oracle/coracle.c), plus size-independent properties at 128^3 ILU(2).

Bars: factors and preconditioned vectors <= 1e-12 relative (max-norm), point
level sets exact, BiCGSTAB iteration counts within +-1.
"""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b2(cuda_ok):
    import paper_1703_01325_b200 as mod
    return mod


@pytest.mark.parametrize("nx,k", [(64, 1), (128, 0)])
def test_fullsize_factors_and_apply_vs_c_oracle(b2, nx, k):
    from oracle import coracle
    n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, 3, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, k)
    cf = coracle.CFactors(n, bs, rp, ci, vals, k)
    assert np.array_equal(f.L.row_ptr, cf.L_rp) and np.array_equal(f.L.col_idx, cf.L_ci)
    assert np.array_equal(f.uprime.row_ptr, cf.U_rp) and np.array_equal(f.uprime.col_idx, cf.U_ci)
    assert rel_err(f.L.values, cf.L_vals) <= 1e-12
    assert rel_err(f.uprime.values, cf.U_vals) <= 1e-12
    assert rel_err(f.dinv, cf.dinv) <= 1e-12
    rhs = np.random.default_rng(1).standard_normal(n * bs)
    assert rel_err(b2.apply_preconditioner(f, rhs), cf.apply(rhs)) <= 1e-12
    if nx <= 64:   # point schedules of the zero-dropped expansions: exact
        assert np.array_equal(f.lower_schedule.level_of_row, cf.lo_level_of_row)
        assert np.array_equal(f.upper_schedule.level_of_row, cf.up_level_of_row)


def test_bicgstab_64cube_ilu1_iterations_vs_oracle(b2):
    """BASELINE configs[1]: 64^3 b3 ILU(1) + BiCGSTAB to 1e-6, iterations within +-1."""
    from oracle import coracle
    from oracle import iluk_oracle as orc
    n, bs, rp, ci, vals = b2.reservoir_block_grid(64, 64, 64, 3, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    b = b2.synthetic.ones_rhs(n, bs, rp, ci, vals)
    f = b2.build_preconditioner(a, 1)
    x, st = b2.bicgstab(a, b, M=f)
    cf = coracle.CFactors(n, bs, rp, ci, vals, 1)
    mv = lambda v: coracle.bsr_spmv(n, bs, rp, ci, vals, v)  # noqa: E731
    _, its, conv, rel, _ = orc.bicgstab(mv, b, cf.apply, rel_tol=1e-6)
    assert st.converged and conv
    assert abs(st.iterations - its) <= 1
    assert st.final_relative_residual <= 1e-6
    assert np.abs(x - 1.0).max() <= 1e-3


def test_ilu2_128cube_properties(b2):
    """128^3 b3 ILU(2): M x = b reconstructed with device SpMVs of the factors, and linearity."""
    import torch
    n, bs, rp, ci, vals = b2.reservoir_block_grid(128, 128, 128, 3, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, 2)
    b = torch.from_numpy(np.random.default_rng(7).standard_normal(n * bs)).cuda()
    x = b2.apply_preconditioner(f, b)
    # (I + L) D (I + U') x == b   with D = dinv^-1 (block diagonal)
    Lop = b2.DeviceOperator(f.L)
    Uop = b2.DeviceOperator(f.uprime)
    d = np.linalg.inv(f.dinv)                                 # (n, bs, bs) row-major
    dcm = np.ascontiguousarray(d.transpose(0, 2, 1)).reshape(-1)
    D = b2.BcsrMatrix(bs, n, n, np.arange(n + 1), np.arange(n), dcm)
    Dop = b2.DeviceOperator(D)
    t1 = x + Uop.matvec(x)
    t2 = Dop.matvec(t1)
    t3 = t2 + Lop.matvec(t2)
    res = float((t3 - b).abs().max() / b.abs().max())
    assert res <= 1e-10, res
    y1 = b2.apply_preconditioner(f, 2.0 * b)
    assert float((y1 - 2.0 * x).abs().max() / x.abs().max()) <= 1e-14
    f.status()
