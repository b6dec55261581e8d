import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_1703_01325_b200 as b2
from test_gpu_parity import _bsr_from_dense_blocks
rng = np.random.default_rng(77)
d = rng.standard_normal((3, 3)) + 4 * np.eye(3)
cases = {"one": _bsr_from_dense_blocks(b2, 1, 3, {(0, 0): d})}
diag = {(i, i): rng.standard_normal((2, 2)) + 3 * np.eye(2) for i in range(50)}
cases["diag"] = _bsr_from_dense_blocks(b2, 50, 2, diag)
arrow = {(i, i): rng.standard_normal((3, 3)) + 40 * np.eye(3) for i in range(300)}
for i in range(1, 300):
    arrow[(0, i)] = 0.1 * rng.standard_normal((3, 3)); arrow[(i, 0)] = 0.1 * rng.standard_normal((3, 3))
cases["arrow"] = _bsr_from_dense_blocks(b2, 300, 3, arrow)
cases["scalar"] = b2.csr_from_triplets(1, 1, [(0, 0, 2.5)])
for eng in ("0", "1"):
    os.environ["BILUK_ENGINE"] = eng
    for name, a in cases.items():
        for k in (0, 1):
            try:
                f = b2.build_preconditioner(a, k)
                inf = f.info
                print(eng, name, k, "ok", {x: inf[x] for x in ("engine", "sweep_ctas", "sweep_warps", "sweep_stages", "stage_bytes") if x in inf})
            except Exception as e:
                print(eng, name, k, "ERR", str(e)[:120])
