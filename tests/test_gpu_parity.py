"""GPU parity of the CUDA path against the reference (golden vectors) and the oracle.

Bars (BASELINE.json north star): patterns and level sets exact; L / D^-1 / U'
and preconditioned vectors within 1e-12 relative (max-norm, acceptance-01
style); Krylov iteration counts within +-1.
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


def _golden_matrix(b2, g):
    n, bs = int(g["n"]), int(g["bs"])
    return b2.BcsrMatrix(bs, n, n, g["rp"], g["ci"], g["vals"])


@pytest.mark.parametrize("path", CASES, ids=IDS)
def test_factors_apply_and_solvers_match_reference(b2, path):
    g = load_golden(path)
    k = int(g["k"])
    a = _golden_matrix(b2, g)
    f = b2.build_preconditioner(a, k)
    # factors: structure exact, values 1e-12
    assert np.array_equal(f.L.row_ptr, g["L_rp"]) and np.array_equal(f.L.col_idx, g["L_ci"])
    assert np.array_equal(f.uprime.row_ptr, g["U_rp"]) and np.array_equal(f.uprime.col_idx, g["U_ci"])
    assert rel_err(f.L.values, g["L_vals"]) <= TOL
    assert rel_err(f.uprime.values, g["U_vals"]) <= TOL
    assert rel_err(f.dinv, g["dinv"]) <= TOL
    # point-wise schedules on the zero-dropped expansions: exact
    assert np.array_equal(f.lower_schedule.level_of_row, g["lo_level_of_row"])
    assert np.array_equal(f.upper_schedule.level_of_row, g["up_level_of_row"])
    # preconditioned vector
    z = b2.apply_preconditioner(f, g["rhs"])
    assert rel_err(z, g["apply_out"]) <= TOL
    # SpMV
    ax = b2.spmv(a, np.ones(a.shape[0]))
    absax = orc.bsr_spmv(a.num_block_rows, a.block_size, g["rp"], g["ci"], np.abs(g["vals"]), np.ones(a.shape[0]))
    assert np.abs(ax - g["spmv_ones"]).max() <= 1e-14 * absax.max()
    # Krylov: iteration counts within +-1 and the same verdict
    b = g["spmv_ones"]
    x, st = b2.gmres(a, b, M=f, cfg=b2.SolverConfig(restart=30, rel_tol=1e-6))
    assert abs(st.iterations - int(g["gmres_iters"])) <= 1
    assert st.converged == bool(g["gmres_conv"])
    x, st = b2.bicgstab(a, b, M=f, cfg=b2.SolverConfig(rel_tol=1e-6))
    assert abs(st.iterations - int(g["bicg_iters"])) <= 1
    assert st.converged == bool(g["bicg_conv"])


@pytest.mark.parametrize("nx,bs,k", [(16, 3, 0), (12, 3, 2), (10, 4, 1), (8, 8, 1), (9, 2, 3), (7, 5, 2)])
def test_synthetic_vs_oracle(b2, nx, bs, k):
    n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, bs, seed=11)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, k)
    of = orc.build_preconditioner(n, bs, rp, ci, vals, k)
    assert rel_err(f.L.values, of.L_vals) <= TOL
    assert rel_err(f.uprime.values, of.U_vals) <= TOL
    assert rel_err(f.dinv, of.dinv) <= TOL
    rhs = np.random.default_rng(1).standard_normal(n * bs)
    assert rel_err(b2.apply_preconditioner(f, rhs), of.apply(rhs)) <= TOL


def test_apply_is_deterministic_and_async_torch_path(b2):
    import torch
    n, bs, rp, ci, vals = b2.reservoir_block_grid(24, 20, 16, 3, seed=2)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 1)
    rhs = torch.randn(n * bs, dtype=torch.float64, device="cuda")
    x1 = b2.apply_preconditioner(f, rhs)
    outs = [b2.apply_preconditioner(f, rhs) for _ in range(5)]
    f.status()
    for x in outs:
        assert torch.equal(x, x1)           # bitwise repeatable run to run
    xh = b2.apply_preconditioner(f, rhs.cpu().numpy())
    assert np.array_equal(xh, x1.cpu().numpy())
    # linearity to rounding
    r2 = torch.randn_like(rhs)
    lhs = b2.apply_preconditioner(f, 3.0 * rhs + r2)
    rhs_lin = 3.0 * x1 + b2.apply_preconditioner(f, r2)
    assert float((lhs - rhs_lin).abs().max() / rhs_lin.abs().max()) <= 1e-13


def test_factorization_errors_match_reference(b2):
    # singular leading block -> SingularBlockError with .row == 0 (reference test_factor.py:145-155)
    dense = np.zeros((4, 4))
    dense[:2, :2] = [[1.0, 2.0], [2.0, 4.0]]
    dense[2:, 2:] = np.eye(2)
    dense[2:, :2] = np.eye(2)
    trip = [(i, j, dense[i, j]) for i in range(4) for j in range(4) if dense[i, j] != 0.0 or i // 2 == j // 2]
    a = b2.bcsr_from_csr(b2.csr_from_triplets(4, 4, trip), 2)
    with pytest.raises(b2.SingularBlockError) as exc:
        b2.build_preconditioner(a, 0)
    assert exc.value.row == 0 and str(exc.value).startswith("factorize:")
    # zero pivot on the scalar path -> FactorizationError, row 0 (test_factor.py:190-203)
    a = b2.csr_from_triplets(2, 2, [(0, 0, 0.0), (0, 1, 1.0), (1, 0, 1.0), (1, 1, 1.0)])
    with pytest.raises(b2.FactorizationError) as exc:
        b2.build_preconditioner(a, 0)
    assert exc.value.row == 0 and str(exc.value).startswith("factorize:")
    # missing diagonal surfaces from the symbolic stage by name
    a = b2.csr_from_triplets(2, 2, [(0, 1, 1.0), (1, 0, 1.0)])
    with pytest.raises(b2.StructuralError) as exc:
        b2.build_preconditioner(a, 0)
    assert str(exc.value).startswith("symbolic-phase:")
    # singular block deeper in the matrix: the FIRST failing row is reported
    n, bs, rp, ci, vals = b2.reservoir_block_grid(6, 5, 4, 3, seed=1)
    vals = vals.copy()
    for row in (77, 31):      # an all-zero block row factors to an all-zero U_ii
        vals[rp[row] * 9:rp[row + 1] * 9] = 0.0
    with pytest.raises(b2.SingularBlockError) as exc:
        b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 0)
    assert exc.value.row == 31


def test_bad_lengths_and_callable_preconditioner(b2):
    n, bs, rp, ci, vals = b2.reservoir_block_grid(6, 6, 6, 3, seed=4)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, 1)
    with pytest.raises(ValueError):
        b2.apply_preconditioner(f, np.zeros(n * bs - 1))
    b = b2.spmv(a, np.ones(n * bs))
    # the reference idiom: an opaque callable M (gmres.py:85-87)
    x1, s1 = b2.gmres(a, b, M=lambda v: b2.apply_preconditioner(f, v), cfg=b2.SolverConfig(restart=30))
    x2, s2 = b2.gmres(a, b, M=f, cfg=b2.SolverConfig(restart=30))
    assert s1.iterations == s2.iterations and s1.converged and s2.converged
    assert np.allclose(x1, x2, rtol=0, atol=1e-12)
    assert np.allclose(x2, 1.0, atol=1e-4)
    _, s0 = b2.gmres(a, b, cfg=b2.SolverConfig(restart=30))
    assert s0.iterations > s2.iterations          # preconditioning helps
    with pytest.raises(ValueError):
        b2.gmres(a, np.zeros(n * bs + 1))
    # a failing user M surfaces as its own exception, a wrong-length result as ValueError
    class Boom(Exception):
        pass

    def bad(v):
        raise Boom("user preconditioner failed")
    with pytest.raises(Boom):
        b2.gmres(a, b, M=bad)
    with pytest.raises(Boom):
        b2.bicgstab(a, b, M=bad)
    with pytest.raises(ValueError, match="shape"):
        b2.gmres(a, b, M=lambda v: v[:-1])


def test_mutated_matrix_values_reach_the_solvers(b2):
    """A host matrix edited in place (e.g. a refreshed Jacobian) is re-read by
    spmv / gmres / bicgstab on every call (no identity-only caching)."""
    n, bs, rp, ci, vals = b2.reservoir_block_grid(6, 5, 4, 3, seed=8)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals.copy())
    x = np.random.default_rng(0).standard_normal(n * bs)
    y1 = b2.spmv(a, x)
    a.values[:] *= 2.0
    y2 = b2.spmv(a, x)
    assert np.allclose(y2, 2.0 * y1, rtol=1e-14, atol=0)
    b = b2.spmv(a, np.ones(n * bs))
    f = b2.build_preconditioner(a, 0)
    xs, st = b2.bicgstab(a, b, M=f)
    assert st.converged and np.abs(xs - 1.0).max() <= 1e-4


def test_out_argument_is_checked(b2):
    import torch
    n, bs, rp, ci, vals = b2.reservoir_block_grid(5, 5, 5, 3, seed=2)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 0)
    rhs = torch.ones(n * bs, dtype=torch.float64, device="cuda")
    for bad in (torch.empty(n * bs - 1, dtype=torch.float64, device="cuda"),
                torch.empty(n * bs, dtype=torch.float32, device="cuda"),
                torch.empty(n * bs, dtype=torch.float64),
                torch.empty(2 * n * bs, dtype=torch.float64, device="cuda")[::2]):
        with pytest.raises(ValueError):
            b2.apply_preconditioner(f, rhs, out=bad)
    big = torch.ones(2 * n * bs, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):   # overlapping the right-hand side
        b2.apply_preconditioner(f, big[: n * bs], out=big[n * bs // 2: n * bs // 2 + n * bs])


def test_applies_on_two_streams_are_serialised(b2):
    """One plan applied from two torch streams back to back: the library orders
    the second apply after the first (shared sweep workspace), results exact."""
    import torch
    n, bs, rp, ci, vals = b2.reservoir_block_grid(24, 24, 24, 3, seed=3)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 1)
    of = orc.build_preconditioner(n, bs, rp, ci, vals, 1)
    r1 = np.random.default_rng(1).standard_normal(n * bs)
    r2 = np.random.default_rng(2).standard_normal(n * bs)
    d1, d2 = torch.from_numpy(r1).cuda(), torch.from_numpy(r2).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for _ in range(4):
        with torch.cuda.stream(s1):
            o1 = b2.apply_preconditioner(f, d1)
        with torch.cuda.stream(s2):
            o2 = b2.apply_preconditioner(f, d2)
        outs.append((o1, o2))
    torch.cuda.synchronize()
    f.status()
    w1, w2 = of.apply(r1), of.apply(r2)
    for o1, o2 in outs:
        assert rel_err(o1.cpu().numpy(), w1) <= TOL and rel_err(o2.cpu().numpy(), w2) <= TOL


def test_gmres_known_answers(b2):
    # identity converges in one iteration (reference test_gmres.py:13-20)
    a = b2.csr_from_triplets(10, 10, [(i, i, 1.0) for i in range(10)])
    b = np.arange(1.0, 11.0)
    x, st = b2.gmres(a, b)
    assert st.converged and st.iterations == 1 and np.allclose(x, b, atol=1e-12)
    # zero rhs short-circuits
    x, st = b2.gmres(a, np.zeros(10))
    assert st.converged and st.iterations == 0 and not x.any()
    # iteration cap reported honestly
    from paper_1703_01325_b200.synthetic import poisson7_pattern
    rp, ci = poisson7_pattern(10, 10, 1)
    vals = np.where(ci == np.repeat(np.arange(100), np.diff(rp)), 6.0, -1.0)
    p = b2.CsrMatrix(100, 100, rp, ci, vals)
    x, st = b2.gmres(p, b2.spmv(p, np.ones(100)), cfg=b2.SolverConfig(max_iters=3, rel_tol=1e-14))
    assert not st.converged and st.iterations == 3
    # full pattern ILU(n) is exact LU: one preconditioned iteration (acceptance 09)
    rng = np.random.default_rng(909)
    dense = rng.standard_normal((20, 20)) + 20 * np.eye(20)
    a = b2.csr_from_triplets(20, 20, [(i, j, dense[i, j]) for i in range(20) for j in range(20)])
    f = b2.build_preconditioner(b2.bcsr_from_csr(a, 1), 20)
    _, st = b2.gmres(a, a.to_dense() @ rng.standard_normal(20), M=f)
    assert st.converged and st.iterations == 1


def _random_pattern_matrix(n, bs, seed):
    """A non-grid pattern (contiguous-range partition path): random sparse + diagonal."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        cols = set(rng.choice(n, size=min(n, 4), replace=False).tolist()) | {i}
        rows.append(sorted(cols))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.array([c for r in rows for c in r], np.int64)
    vals = rng.uniform(-1, 1, (len(ci), bs, bs))
    for i, r in enumerate(rows):
        d = rp[i] + r.index(i)
        vals[d] += np.eye(bs) * (2.0 * bs * len(r))
    return n, bs, rp, ci, np.ascontiguousarray(vals.transpose(0, 2, 1)).reshape(-1)


@pytest.mark.parametrize("engine", [0, 1])
@pytest.mark.parametrize("case", ["grid16_b3_k0", "grid12_b3_k2", "grid10_b4_k1", "grid9_b2_k3", "rand300_b3_k1",
                                  "rand200_b1_k0"])
def test_both_engines_match_oracle_and_are_repeatable(b2, monkeypatch, engine, case):
    """Each sweep engine, forced, against the oracle; bitwise repeatable applies."""
    import torch
    monkeypatch.setenv("BILUK_ENGINE", str(engine))
    kind, bsk, kk = case.split("_")
    bs, k = int(bsk[1:]), int(kk[1:])
    if kind.startswith("grid"):
        nx = int(kind[4:])
        n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, bs, seed=5)
    else:
        n, bs, rp, ci, vals = _random_pattern_matrix(int(kind[4:]), bs, seed=5)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, k)
    assert f.info["engine"] == engine
    of = orc.build_preconditioner(n, bs, rp, ci, vals, k)
    rhs = np.random.default_rng(3).standard_normal(n * bs)
    z = b2.apply_preconditioner(f, rhs)
    assert rel_err(z, of.apply(rhs)) <= TOL
    rt = torch.from_numpy(rhs).cuda()
    x1 = b2.apply_preconditioner(f, rt)
    for _ in range(3):
        assert torch.equal(b2.apply_preconditioner(f, rt), x1)
    f.status()


@pytest.mark.parametrize("bs", [5, 6, 7, 8])
@pytest.mark.parametrize("k", [0, 1, 2])
def test_large_blocks_match_oracle(b2, bs, k):
    """Block sizes 5..8 (the tiled sweep: several lanes per block row) against
    the oracle, bitwise repeatable."""
    import torch
    n, bs, rp, ci, vals = b2.reservoir_block_grid(9, 8, 7, bs, seed=11)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), k)
    assert f.info["engine"] == 0
    of = orc.build_preconditioner(n, bs, rp, ci, vals, k)
    rhs = np.random.default_rng(5).standard_normal(n * bs)
    assert rel_err(b2.apply_preconditioner(f, rhs), of.apply(rhs)) <= TOL
    rt = torch.from_numpy(rhs).cuda()
    x1 = b2.apply_preconditioner(f, rt)
    for _ in range(2):
        assert torch.equal(b2.apply_preconditioner(f, rt), x1)
    f.status()


@pytest.mark.parametrize("shape", [(5, 4, 3, 3), (16, 16, 16, 3), (17, 9, 13, 2), (24, 20, 16, 4), (20, 20, 20, 1),
                                   (33, 7, 5, 3)])
def test_grid_sweep_matches_oracle(b2, monkeypatch, shape):
    """The grid sweep (engine 2, opt-in: ILU(0) of a 7-point block grid) against
    the oracle, bitwise repeatable, on odd shapes and every block size it takes."""
    import torch
    monkeypatch.setenv("BILUK_ENGINE", "2")
    nx, ny, nz, bs = shape
    n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, ny, nz, bs, seed=7)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 0)
    assert f.info["engine"] == 2
    of = orc.build_preconditioner(n, bs, rp, ci, vals, 0)
    rhs = np.random.default_rng(4).standard_normal(n * bs)
    assert rel_err(b2.apply_preconditioner(f, rhs), of.apply(rhs)) <= TOL
    rt = torch.from_numpy(rhs).cuda()
    x1 = b2.apply_preconditioner(f, rt)
    for _ in range(3):
        assert torch.equal(b2.apply_preconditioner(f, rt), x1)
    f.status()


def test_grid_sweep_declines_other_patterns(b2, monkeypatch):
    """Engine 2 is only planned for a 7-point ILU(0) grid: fill or a random
    pattern falls back to the partitioned sweep."""
    monkeypatch.setenv("BILUK_ENGINE", "2")
    n, bs, rp, ci, vals = b2.reservoir_block_grid(8, 8, 8, 3, seed=1)
    assert b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 1).info["engine"] == 1
    n, bs, rp, ci, vals = _random_pattern_matrix(200, 3, seed=2)
    assert b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 0).info["engine"] == 1


@pytest.mark.parametrize("groups,nprod", [(3, 1), (2, 2), (2, 1), (3, 2), (3, 3), (3, 4)])
@pytest.mark.parametrize("case", ["grid16_b3_k0", "grid12_b3_k2", "grid10_b4_k1", "rand300_b3_k1"])
def test_partitioned_kernel_variants_match_oracle(b2, monkeypatch, groups, nprod, case):
    """Every instantiation of the partitioned sweep (compute groups x producer
    warps; the planner picks one producer only for large ILU(2)+) against the oracle."""
    monkeypatch.setenv("BILUK_ENGINE", "1")
    monkeypatch.setenv("BILUK_GROUPS", str(groups))
    monkeypatch.setenv("BILUK_NPROD", str(nprod))
    kind, bsk, kk = case.split("_")
    bs, k = int(bsk[1:]), int(kk[1:])
    if kind.startswith("grid"):
        nx = int(kind[4:])
        n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, bs, seed=6)
    else:
        n, bs, rp, ci, vals = _random_pattern_matrix(int(kind[4:]), bs, seed=6)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, k)
    assert f.info["engine"] == 1 and f.info["sweep_warps"] == groups * 4 + nprod
    of = orc.build_preconditioner(n, bs, rp, ci, vals, k)
    for seed in (3, 4):
        rhs = np.random.default_rng(seed).standard_normal(n * bs)
        assert rel_err(b2.apply_preconditioner(f, rhs), of.apply(rhs)) <= TOL
    f.status()


def test_sweep_dependency_timeout_is_reported_not_hung(b2, monkeypatch):
    """Fault injection: a record made to wait on a row published after it.  The
    partitioned sweep must time out (bounded waits, the hand-over passed on) and
    report BILUK_ETIMEOUT as CudaPathError -- not hang the GPU."""
    import torch
    monkeypatch.setenv("BILUK_ENGINE", "1")
    monkeypatch.setenv("BILUK_FAULT_GPOS", "1")
    n, bs, rp, ci, vals = b2.reservoir_block_grid(12, 12, 12, 3, seed=1)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    f = b2.build_preconditioner(a, 0)
    monkeypatch.delenv("BILUK_FAULT_GPOS")
    rhs = torch.from_numpy(np.random.default_rng(3).standard_normal(n * bs)).cuda()
    from paper_1703_01325_b200._native import CudaPathError
    with pytest.raises(CudaPathError, match="timed out"):
        b2.apply_preconditioner(f, rhs)
        torch.cuda.synchronize()
        f.status()
    # the plan recovers: a fresh plan of the same matrix is exact again
    g = b2.build_preconditioner(a, 0)
    of = orc.build_preconditioner(n, bs, rp, ci, vals, 0)
    assert rel_err(b2.apply_preconditioner(g, rhs.cpu().numpy()), of.apply(rhs.cpu().numpy())) <= TOL


@pytest.mark.parametrize("k", [0, 1])
def test_block_diagonal_batch_equals_independent_systems(b2, k):
    """A batch applied as one block-diagonal operator equals each system alone."""
    mats, rhs = [], []
    for s in range(3):
        n, bs, rp, ci, vals = b2.reservoir_block_grid(7 + s, 6, 5, 3, seed=20 + s)
        mats.append((n, bs, rp, ci, vals))
        rhs.append(np.random.default_rng(s).standard_normal(n * bs))
    big = b2.block_diagonal([b2.BcsrMatrix(bs, n, n, rp, ci, vals) for n, bs, rp, ci, vals in mats])
    f = b2.build_preconditioner(big, k)
    z = b2.apply_preconditioner(f, np.concatenate(rhs))
    off = 0
    for (n, bs, rp, ci, vals), r in zip(mats, rhs):
        want = orc.build_preconditioner(n, bs, rp, ci, vals, k).apply(r)
        assert rel_err(z[off:off + n * bs], want) <= TOL
        off += n * bs


@pytest.mark.parametrize("k", [0, 1])
def test_batched_bicgstab_equals_independent_solves(b2, k):
    """Batched BiCGSTAB: each system iterates as if alone (same x, same count) and
    its count is within +-1 of the oracle's; a zero right-hand side stops at once."""
    shapes = [(7, 6, 5), (9, 4, 6), (5, 5, 5), (8, 7, 3)]
    mats, rhs = [], []
    for s, (nx, ny, nz) in enumerate(shapes):
        n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, ny, nz, 3, seed=40 + s)
        mats.append(b2.BcsrMatrix(bs, n, n, rp, ci, vals))
        r = np.random.default_rng(s).standard_normal(n * bs)
        rhs.append(np.zeros_like(r) if s == 2 else r)
    big = b2.block_diagonal(mats)
    seg = np.concatenate([[0], np.cumsum([m.num_block_rows for m in mats])])
    cfg = b2.SolverConfig(rel_tol=1e-9)
    assert np.array_equal(big.batch_segments, seg)
    xb, stats = b2.bicgstab_batched(big, np.concatenate(rhs), M=b2.build_preconditioner(big, k), cfg=cfg)
    assert len(stats) == len(mats)
    for i, (m, r) in enumerate(zip(mats, rhs)):
        xs, st = b2.bicgstab(m, r, M=b2.build_preconditioner(m, k), cfg=cfg)
        part = xb[seg[i] * 3:seg[i + 1] * 3]
        assert stats[i].converged == st.converged
        if i == 2:
            assert stats[i].iterations == 0 and stats[i].converged and not np.any(part)
            continue
        # the batch's sweep sums may round differently from the single system's
        # (record layout), so x agrees to rounding -- or to the tolerance when
        # that rounding moves the stopping test by one iteration
        assert abs(stats[i].iterations - st.iterations) <= 1
        assert rel_err(part, xs) <= (1e-10 if stats[i].iterations == st.iterations else 1e-6)
        n, bs = m.num_block_rows, 3
        f = orc.build_preconditioner(n, bs, m.row_ptr, m.col_idx, m.values, k)
        _, its, conv, _, _ = orc.bicgstab(lambda v: orc.bsr_spmv(n, bs, m.row_ptr, m.col_idx, m.values, v), r,
                                          precond=f.apply, rel_tol=1e-9)
        assert conv and abs(its - stats[i].iterations) <= 1


def test_batched_bicgstab_rejects_coupled_segments(b2):
    n, bs, rp, ci, vals = b2.reservoir_block_grid(6, 5, 4, 3, seed=3)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    with pytest.raises(ValueError):
        b2.bicgstab_batched(a, np.ones(n * bs), [0, n // 2, n])


def test_sweep_timing_hooks(b2):
    """biluk_plan_set_timing / sweep_ms: the sweep kernel alone, both engines."""
    import torch
    n, bs, rp, ci, vals = b2.reservoir_block_grid(20, 18, 16, 3, seed=5)
    a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
    rhs = torch.randn(n * bs, dtype=torch.float64, device="cuda")
    for k in (0, 2):
        f = b2.build_preconditioner(a, k)
        ref = b2.apply_preconditioner(f, rhs)
        f.set_sweep_timing(True)
        x = b2.apply_preconditioner(f, rhs)
        ms = f.sweep_ms()
        f.set_sweep_timing(False)
        assert 0.0 < ms < 1000.0
        assert torch.equal(x, ref)          # timing does not change the result
        with pytest.raises(ValueError):
            f.sweep_ms()                    # off again


def test_apply_many_pipelined_equals_single_applies(b2):
    """apply_preconditioner_many (host in/out, overlapped copies) == per-RHS applies, bitwise."""
    import torch
    n, bs, rp, ci, vals = b2.reservoir_block_grid(14, 12, 10, 3, seed=8)
    f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 0)
    rhs = np.random.default_rng(3).standard_normal((5, n * bs))
    got = b2.apply_preconditioner_many(f, rhs)
    assert tuple(got.shape) == (5, n * bs) and not got.is_cuda
    for j in range(5):
        assert np.array_equal(got[j].numpy(), b2.apply_preconditioner(f, rhs[j]))
    one = b2.apply_preconditioner_many(f, torch.from_numpy(rhs[:1]).pin_memory())
    assert np.array_equal(one[0].numpy(), got[0].numpy())
    with pytest.raises(ValueError):
        b2.apply_preconditioner_many(f, rhs[:, :-1])
    with pytest.raises(ValueError):
        b2.apply_preconditioner_many(f, torch.from_numpy(rhs).cuda())


def _bsr_from_dense_blocks(b2, nb, bs, blocks):
    """BcsrMatrix from {(i, j): (bs, bs) block} (column-major inside each block)."""
    rp, ci, vals = [0], [], []
    for i in range(nb):
        for j in sorted(c for (r, c) in blocks if r == i):
            ci.append(j)
            vals.extend(np.asarray(blocks[(i, j)], dtype=np.float64).T.reshape(-1))
        rp.append(len(ci))
    return b2.BcsrMatrix(bs, nb, nb, np.array(rp), np.array(ci), np.array(vals))


@pytest.mark.parametrize("engine", ["0", "1"])
def test_edge_shapes_match_oracle(b2, monkeypatch, engine):
    """One block row; a block-diagonal matrix (one level); an arrowhead whose
    first row and column touch every row (a long row, a long column); a 1x1
    scalar system."""
    monkeypatch.setenv("BILUK_ENGINE", engine)
    rng = np.random.default_rng(77)
    cases = []
    d = rng.standard_normal((3, 3)) + 4 * np.eye(3)
    cases.append((_bsr_from_dense_blocks(b2, 1, 3, {(0, 0): d}), [0, 2]))
    diag = {(i, i): rng.standard_normal((2, 2)) + 3 * np.eye(2) for i in range(50)}
    cases.append((_bsr_from_dense_blocks(b2, 50, 2, diag), [0, 1]))
    arrow = {(i, i): rng.standard_normal((3, 3)) + 40 * np.eye(3) for i in range(60)}
    for i in range(1, 60):
        arrow[(0, i)] = 0.1 * rng.standard_normal((3, 3))
        arrow[(i, 0)] = 0.1 * rng.standard_normal((3, 3))
    cases.append((_bsr_from_dense_blocks(b2, 60, 3, arrow), [0, 1]))
    cases.append((b2.csr_from_triplets(1, 1, [(0, 0, 2.5)]), [0, 3]))
    for a, ks in cases:
        nb = a.num_block_rows if hasattr(a, "num_block_rows") else a.num_rows
        bs = a.block_size if hasattr(a, "block_size") else 1
        for k in ks:
            f = b2.build_preconditioner(a, k)
            of = orc.build_preconditioner(nb, bs, a.row_ptr, a.col_idx, a.values, k)
            rhs = rng.standard_normal(nb * bs)
            assert rel_err(b2.apply_preconditioner(f, rhs), of.apply(rhs)) <= TOL


def test_rows_too_long_for_the_sweep_fail_clearly(b2, monkeypatch):
    """A row whose sweep tile cannot be staged raises NotImplementedError naming the row length."""
    monkeypatch.setenv("BILUK_ENGINE", "0")
    rng = np.random.default_rng(5)
    arrow = {(i, i): rng.standard_normal((3, 3)) + 40 * np.eye(3) for i in range(400)}
    for i in range(1, 400):
        arrow[(0, i)] = 0.1 * rng.standard_normal((3, 3))
        arrow[(i, 0)] = 0.1 * rng.standard_normal((3, 3))
    with pytest.raises(NotImplementedError, match="off-diagonal blocks"):
        b2.build_preconditioner(_bsr_from_dense_blocks(b2, 400, 3, arrow), 0)
