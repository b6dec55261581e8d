timeout 900 python - <<'PY' 2>&1 | tail -30
import os, sys, time
sys.path.insert(0, '.')
import torch
import bench
import paper_1703_01325_b200 as b2
os.environ["BILUK_KRYLOV_DEBUG"] = "1"
for name, (nxc, bsc, kc, solver) in list(bench.CONFIGS.items())[:2]:
    ncf, bsf, rpf, cif, vf = b2.reservoir_block_grid(nxc, nxc, nxc, bsc, seed=0)
    af = b2.BcsrMatrix(bsf, ncf, ncf, rpf, cif, vf)
    ff = b2.build_preconditioner(af, kc)
    op = b2.DeviceOperator(af)
    bb = torch.from_numpy(b2.synthetic.ones_rhs(ncf, bsf, rpf, cif, vf)).cuda()
    cfgf = b2.SolverConfig(restart=30, rel_tol=1e-6)
    for r in range(4):
        torch.cuda.synchronize(); t2 = time.perf_counter()
        _, stf = b2.bicgstab(op, bb, M=ff, cfg=cfgf)
        torch.cuda.synchronize(); print(name, r, round((time.perf_counter() - t2) * 1e3, 2), "ms", flush=True)
PY
