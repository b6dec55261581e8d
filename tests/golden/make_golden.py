"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (needs /root/reference, read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Each file holds one (matrix, k) case: the BSR
input, and the reference's outputs for it -- the ILU(k) pattern
(symbolic_phase), L / D^-1 / U' (build_preconditioner), the point-wise level
schedules of both triangles, apply_preconditioner on a seeded vector, spmv of
ones, GMRES(30) to 1e-6, and BiCGSTAB (the repo's definition,
oracle/iluk_oracle.py:bicgstab) run on top of the reference's own spmv and
apply_preconditioner.  Nothing here is used at run time on the GPU box: the
committed .npz files are the fixtures.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")

import blockiluk as ref  # noqa: E402  (the reference, read-only)
from helpers import random_sparse_csr  # noqa: E402  (reference test helper)

import importlib.util  # noqa: E402

_spec = importlib.util.spec_from_file_location(
    "_synth", os.path.join(ROOT, "paper_1703_01325_b200", "synthetic.py"))
synth = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(synth)
_spec = importlib.util.spec_from_file_location("_oracle", os.path.join(ROOT, "oracle", "iluk_oracle.py"))
oracle = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(oracle)


def dump(name, a, k, rhs_seed=1):
    bs, n = a.block_size, a.num_block_rows
    f = ref.build_preconditioner(a, k)
    pat = ref.symbolic_phase(ref.extract_point_pattern(a), k)
    prp = np.zeros(n + 1, np.int64)
    prp[1:] = np.cumsum(pat.row_lengths)
    pci = np.array([j for r in pat.rows for j in r], np.int64)
    rhs = np.random.default_rng(rhs_seed).standard_normal(n * bs)
    z = ref.apply_preconditioner(f, rhs)
    apt = ref.csr_expand(a)
    ones = np.ones(n * bs)
    ax = ref.spmv(apt, ones)
    b = ax.copy()
    M = lambda v: ref.apply_preconditioner(f, v)  # noqa: E731
    gx, gst = ref.gmres(a, b, M=M, cfg=ref.SolverConfig(restart=30, rel_tol=1e-6))
    bx, bit, bconv, brel, bhist = oracle.bicgstab(lambda v: ref.spmv(apt, v), b, M, rel_tol=1e-6)
    out = dict(
        n=n, bs=bs, k=k, rp=a.row_ptr, ci=a.col_idx, vals=a.values,
        P_rp=prp, P_ci=pci,
        L_rp=f.L.row_ptr, L_ci=f.L.col_idx, L_vals=f.L.values,
        dinv=f.dinv,
        U_rp=f.uprime.row_ptr, U_ci=f.uprime.col_idx, U_vals=f.uprime.values,
        lo_level_of_row=f.lower_schedule.level_of_row, lo_num_levels=f.lower_schedule.num_levels,
        up_level_of_row=f.upper_schedule.level_of_row, up_num_levels=f.upper_schedule.num_levels,
        lo_nnz=f.lower_op.matrix.nnz, up_nnz=f.upper_op.matrix.nnz,
        rhs=rhs, apply_out=z, spmv_ones=ax,
        gmres_x=gx, gmres_iters=gst.iterations, gmres_conv=gst.converged,
        gmres_rel=gst.final_relative_residual, gmres_hist=np.array(gst.residual_history),
        bicg_x=bx, bicg_iters=bit, bicg_conv=bconv, bicg_rel=brel,
    )
    path = os.path.join(HERE, f"{name}_k{k}.npz")
    np.savez_compressed(path, **out)
    print(f"{path}: n={n} bs={bs} k={k} nnzP={pci.size} gmres={gst.iterations} "
          f"bicg={bit} lo_levels={f.lower_schedule.num_levels}")


def synth_bsr(nx, ny, nz, bs, seed=0):
    n, bs, rp, ci, vals = synth.reservoir_block_grid(nx, ny, nz, bs, seed=seed)
    return ref.BcsrMatrix(bs, n, n, rp, ci, vals)


def main():
    for k in (0, 1, 2):
        dump("synth4x4x4_b3", synth_bsr(4, 4, 4, 3), k)
    for k in (0, 1, 2):
        dump("synth8x8x8_b3", synth_bsr(8, 8, 8, 3), k)
    dump("synth5x4x3_b2", synth_bsr(5, 4, 3, 2, seed=3), 1)
    dump("synth3x3x3_b4", synth_bsr(3, 3, 3, 4, seed=4), 2)
    dump("synth3x3x2_b8", synth_bsr(3, 3, 2, 8, seed=5), 1)
    dump("synth4x3x3_b5", synth_bsr(4, 3, 3, 5, seed=6), 1)
    # reblocked scalar Poisson: in-block zeros -> point schedules shallower than block ones
    for k in (0, 1, 3):
        dump("poisson4x3x2_b2", ref.bcsr_from_csr(ref.gen_poisson_3d(4, 3, 2), 2), k)
    dump("poisson6x6x6_b4", ref.bcsr_from_csr(ref.gen_poisson_3d(6, 6, 6), 4), 1)
    # scalar path (bs = 1: point kernel with division, factor.py:124-148)
    rng = np.random.default_rng(47)
    a = random_sparse_csr(rng, 40)
    for k in (0, 1, 2):
        dump("random40_b1", ref.bcsr_from_csr(a, 1), k)
    dump("poisson5x5x5_b1", ref.bcsr_from_csr(ref.gen_poisson_3d(5, 5, 5), 1), 2)


if __name__ == "__main__":
    main()
