"""Full-size parity (BASELINE configs[1..4]) against the C restatement of the
reference (oracle/coracle.c), and size-independent properties at 128^3 ILU(2).

Bars: factors and preconditioned vectors <= 1e-12 relative (max-norm), point
level sets exact, Krylov iteration counts within +-1 (BiCGSTAB and GMRES(30)
counts at 128^3 / 100^3 come from tests/golden/fullsize_iters.json, made by
tests/golden/make_fullsize_golden.py with the same oracle).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b2(cuda_ok):
    import paper_1703_01325_b200 as mod
    return mod


@pytest.mark.parametrize("nx,k", [(64, 1), (128, 0), (128, 1), (128, 2)])
def test_fullsize_factors_and_apply_vs_c_oracle(b2, nx, k):
    """BASELINE configs[1] and [2] (ILU(0), ILU(1), ILU(2) of 128^3): the planner's
    own kernel choice (with fill: four producer warps) against the C oracle."""
    from oracle import coracle
    n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, 3, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, k)
    if nx == 128:
        assert f.info["engine"] == 1
        assert f.info["sweep_warps"] == 3 * 4 + (4 if k >= 1 else 2)   # the planner: four producers with fill
    cf = coracle.CFactors(n, bs, rp, ci, vals, k)
    assert np.array_equal(f.L.row_ptr, cf.L_rp) and np.array_equal(f.L.col_idx, cf.L_ci)
    assert np.array_equal(f.uprime.row_ptr, cf.U_rp) and np.array_equal(f.uprime.col_idx, cf.U_ci)
    assert rel_err(f.L.values, cf.L_vals) <= 1e-12
    assert rel_err(f.uprime.values, cf.U_vals) <= 1e-12
    assert rel_err(f.dinv, cf.dinv) <= 1e-12
    for seed in (1, 2):
        rhs = np.random.default_rng(seed).standard_normal(n * bs)
        err = rel_err(b2.apply_preconditioner(f, rhs), cf.apply(rhs))
        print(f"{nx}^3 ILU({k}) apply rel err {err:.2e}")
        assert err <= 1e-12
    # point schedules of the zero-dropped expansions: exact
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


FULL = json.load(open(os.path.join(GOLDEN_DIR, "fullsize_iters.json")))


@pytest.mark.parametrize("name", sorted(FULL))
def test_fullsize_krylov_iterations_vs_oracle_golden(b2, name):
    """configs[2] BiCGSTAB + ILU(0) at 128^3, configs[3] GMRES(30) + ILU(1) at
    100^3 with 4x4 and 8x8 blocks: iteration counts within +-1 of the oracle's."""
    g = FULL[name]
    nx, bs, k = g["grid"], g["bs"], g["k"]
    n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, bs, seed=0)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    import torch
    b = torch.from_numpy(b2.synthetic.ones_rhs(n, bs, rp, ci, vals)).cuda()
    f = b2.build_preconditioner(a, k)
    solve = b2.bicgstab if g["solver"] == "bicgstab" else b2.gmres
    x, st = solve(a, b, M=f, cfg=b2.SolverConfig(restart=30, rel_tol=1e-6))
    print(name, "gpu", st.iterations, "oracle", g["iterations"])
    assert st.converged == g["converged"]
    assert abs(st.iterations - g["iterations"]) <= 1
    assert st.final_relative_residual <= 1e-6


def test_batch_systems_vs_oracle(b2):
    """BASELINE configs[4]: the 64-system batch (64^3 b3 ILU(1)) as the bench
    builds it -- one block-diagonal operator -- applied once; systems 0, 21, 42
    and 63 of the result against the C oracle of each system alone."""
    import torch
    from oracle import coracle
    mats = []
    for s in range(64):
        n, bs, rp, ci, vals = b2.reservoir_block_grid(64, 64, 64, 3, seed=s)
        mats.append(b2.BcsrMatrix(bs, n, n, rp, ci, vals))
    big = b2.block_diagonal(mats)
    f = b2.build_preconditioner(big, 1)
    m = n * bs
    rhs = np.random.default_rng(9).standard_normal(64 * m)
    z = b2.apply_preconditioner(f, torch.from_numpy(rhs).cuda()).cpu().numpy()
    f.status()
    for s in (0, 21, 42, 63):
        a = mats[s]
        cf = coracle.CFactors(a.num_block_rows, bs, a.row_ptr, a.col_idx, a.values, 1)
        assert rel_err(z[s * m:(s + 1) * m], cf.apply(rhs[s * m:(s + 1) * m])) <= 1e-12, s


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
