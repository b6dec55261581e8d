"""Matrix Market ingestion, the Poisson source and the sweep harness's report contract (CPU),
plus one GPU sweep."""

import numpy as np
import pytest

import paper_1703_01325_b200 as b2
from paper_1703_01325_b200 import harness


def _write(tmp_path, text, name="m.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_matrix_market_general_symmetric_and_duplicates(tmp_path):
    gen = _write(tmp_path, "%%MatrixMarket matrix coordinate real general\n% comment\n\n3 3 4\n"
                           "1 1 2.0\n3 2 -1.5\n1 1 0.5\n2 3 4\n")
    a = b2.read_matrix_market(gen)
    dense = np.zeros((3, 3))
    for i in range(3):
        dense[i, a.col_idx[a.row_ptr[i]:a.row_ptr[i + 1]]] = a.values[a.row_ptr[i]:a.row_ptr[i + 1]]
    assert np.array_equal(dense, [[2.5, 0, 0], [0, 0, 4.0], [0, -1.5, 0]])   # duplicates summed
    sym = _write(tmp_path, "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 3\n2 1 -1\n", "s.mtx")
    s = b2.read_matrix_market(sym)
    assert s.row_ptr.tolist() == [0, 2, 3] and s.col_idx.tolist() == [0, 1, 0]   # strict triangle mirrored
    assert s.values.tolist() == [3.0, -1.0, -1.0]


@pytest.mark.parametrize("text,line", [
    ("", 1),
    ("%%MatrixMarket matrix array real general\n1 1\n1\n", 1),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", 1),
    ("%%MatrixMarket matrix coordinate real general\n% only comments\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n", 4),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n% trailing\n", 4),
])
def test_matrix_market_errors_name_the_line(tmp_path, text, line):
    with pytest.raises(b2.MatrixMarketError) as exc:
        b2.read_matrix_market(_write(tmp_path, text))
    assert exc.value.line == line and str(exc.value).startswith(f"line {line}: ")
    assert isinstance(exc.value, ValueError)


def test_poisson_operator_known_answer():
    a = b2.gen_poisson_3d(3, 2, 2)
    assert a.num_rows == 12
    row0 = a.col_idx[a.row_ptr[0]:a.row_ptr[1]].tolist()
    assert row0 == [0, 1, 3, 6] and a.values[a.row_ptr[0]:a.row_ptr[1]].tolist() == [6.0, -1.0, -1.0, -1.0]
    assert np.all(np.diff(a.row_ptr) >= 4) and np.all(np.diff(a.row_ptr) <= 7)
    with pytest.raises(b2.StructuralError):
        b2.gen_poisson_3d(0, 2, 2)


def test_report_contract_roundtrip_and_table():
    recs = [harness.BenchRecord(1, 0, 1, 0.5, 0.25, 10, True, 1e-7),
            harness.BenchRecord(1, 0, 4, 0.5, 0.125, 10, True, 1e-7),
            harness.BenchRecord(2, 1, 1, 0.1, 0.3, 3, False, 2e-3)]
    text = harness.emit_report(recs, "csv")
    assert text.splitlines()[0] == ",".join(harness.CSV_HEADER)
    assert harness.parse_records_csv(text) == recs
    table = harness.emit_report(recs).splitlines()
    assert table[0].split() == ["block_size", "k", "threads", "setup_s", "solve_s", "iterations", "converged",
                                "residual", "speedup"]
    assert table[3].split()[-1] == "2.00" and table[4].startswith("-")   # speedup vs 1 thread; section rule
    with pytest.raises(ValueError):
        harness.emit_report([])
    with pytest.raises(ValueError):
        harness.parse_records_csv("a,b\n")


@pytest.mark.parametrize("kw", [{}, {"poisson": (2, 2, 2), "mtx_path": "x"}, {"poisson": (2, 2, 2), "block_sizes": [0]},
                                {"poisson": (2, 2, 2), "k_levels": [-1]}, {"poisson": (2, 2, 2), "threads": []},
                                {"poisson": (2, 2, 2), "output": "json"}])
def test_plan_validation(kw):
    with pytest.raises(ValueError):
        harness.BenchPlan(**kw)


def test_cli_parser():
    args = harness.build_parser().parse_args(["--poisson", "4", "4", "4", "--block-sizes", "1,2", "--format", "csv"])
    assert args.block_sizes == [1, 2] and args.k_levels == [0] and args.restart == 20 and args.tol == 1e-6
    with pytest.raises(SystemExit):
        harness.build_parser().parse_args(["--poisson", "4", "4", "4", "--block-sizes", "a"])


@pytest.mark.gpu
def test_sweep_on_gpu_matches_oracle_iterations(cuda_ok, capsys):
    from oracle import iluk_oracle as orc
    plan = harness.BenchPlan(poisson=(6, 6, 6), block_sizes=[1, 3, 5], k_levels=[0, 1], threads=[1, 2],
                             solver=b2.SolverConfig(restart=30))
    recs = harness.run_bench(plan)
    assert "skipping block size 5" in capsys.readouterr().err
    assert [(r.block_size, r.k, r.threads) for r in recs] == [(1, 0, 1), (1, 0, 2), (1, 1, 1), (1, 1, 2),
                                                             (3, 0, 1), (3, 0, 2), (3, 1, 1), (3, 1, 2)]
    assert all(r.converged for r in recs)
    a = b2.gen_poisson_3d(6, 6, 6)
    b = harness._rhs(a, "ones-solution", 0)
    for r in recs[::2]:
        blk = b2.bcsr_from_csr(a, r.block_size)
        f = orc.build_preconditioner(blk.num_block_rows, r.block_size, blk.row_ptr, blk.col_idx, blk.values, r.k)
        mv = lambda v: orc.bsr_spmv(blk.num_block_rows, r.block_size, blk.row_ptr, blk.col_idx, blk.values, v)
        _, its, conv, _, _ = orc.gmres(mv, b, precond=f.apply, restart=30)
        assert conv and abs(its - r.iterations) <= 1
    assert harness.main(["--poisson", "4", "4", "4", "--block-sizes", "1,2", "--format", "csv"]) == 0


@pytest.mark.parametrize("fmt", ["csv", "table"])
def test_reports_match_reference_golden(fmt):
    """Byte-identical to the reference's emit_report (tests/golden/make_harness_golden.py)."""
    import os
    recs = [harness.BenchRecord(1, 0, 1, 0.5, 0.25, 10, True, 1e-7),
            harness.BenchRecord(1, 0, 4, 0.5, 0.125, 10, True, 1e-7),
            harness.BenchRecord(2, 1, 1, 0.1, 0.3, 3, False, 2e-3),
            harness.BenchRecord(4, 2, 1, 1.0 / 3.0, 0.0, 0, True, 0.0)]
    path = os.path.join(os.path.dirname(__file__), "golden", f"harness_report_{fmt}.txt")
    with open(path) as fh:
        assert harness.emit_report(recs, fmt) == fh.read()
