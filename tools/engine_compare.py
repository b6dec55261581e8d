"""Apply time of both sweep engines over the BASELINE configs (GPU).

    python tools/engine_compare.py [NX_BS_K ...]      (default: the BASELINE configs)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CASES = [(16, 3, 0), (64, 3, 1), (128, 3, 0), (128, 3, 1), (128, 3, 2), (100, 4, 1), (100, 8, 1)]


def main():
    import torch
    import paper_1703_01325_b200 as b2
    cases = [tuple(int(v) for v in c.split("_")) for c in sys.argv[1:]] or CASES
    for nx, bs, k in cases:
        n, bs_, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, bs, seed=0)
        a = b2.BcsrMatrix(bs, n, n, rp, ci, vals)
        rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
        out = torch.empty_like(rhs)
        res = {"case": f"{nx}^3 b{bs} k{k}"}
        for eng in (0, 1):
            os.environ["BILUK_ENGINE"] = str(eng)
            f = b2.build_preconditioner(a, k)
            for _ in range(3):
                b2.apply_preconditioner(f, rhs, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                b2.apply_preconditioner(f, rhs, out=out)
            e1.record()
            torch.cuda.synchronize()
            f.status()
            us = e0.elapsed_time(e1) / 10 * 1e3
            inf = f.info
            res[f"e{eng}_us"] = round(us, 1)
            res[f"e{eng}_GBps"] = round(inf["apply_bytes"] / us / 1e3, 1)
            if eng == 1:
                res["records"] = inf["records"]
                res["parts"] = inf["parts"]
            del f
            torch.cuda.empty_cache()
        os.environ.pop("BILUK_ENGINE", None)
        print(res, flush=True)


if __name__ == "__main__":
    main()
