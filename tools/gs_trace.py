"""Per-record stamps of the grid sweep (engine 2): where does a level's time go?

    python tools/gs_trace.py [nx] [--out file.npz]
Stamps (globaltimer ns): 0 bulk copy issued, 5 record done (thread 0),
6 halo stored by the halo warp, 7 flags (U' bit | level << 10); then clock64
stages of thread 0 for the first 16384 records.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_01325_b200 as b2  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 128
os.environ["BILUK_ENGINE"] = "2"
n, bs, rp, ci, vals = b2.reservoir_block_grid(nx, nx, nx, 3, seed=0)
f = b2.build_preconditioner(b2.BcsrMatrix(bs, n, n, rp, ci, vals), 0)
rhs = torch.from_numpy(np.random.default_rng(1).standard_normal(n * bs)).cuda()
out = torch.empty_like(rhs)
for _ in range(3):
    b2.apply_preconditioner(f, rhs, out=out)
tr = f.set_trace(True)
b2.apply_preconditioner(f, rhs, out=out)
torch.cuda.synchronize()
f.status()
t = tr.cpu().numpy()[: f.info["records"]].astype(np.int64)
t0 = t[:, 0][t[:, 0] > 0].min()
s = (t[:, :7] - t0) / 1e3
print("span us", s[:, 5].max())
rec_int = []
parts = f.info["parts"]
# per part (records are contiguous per part): interval between consecutive ends
nrec = t.shape[0] // parts
for c in range(parts):
    e = s[c * nrec:(c + 1) * nrec, 5]
    rec_int.append(np.diff(e))
ri = np.concatenate(rec_int)
print(f"  record interval: p10 {np.percentile(ri, 10):.3f} med {np.median(ri):.3f} p90 {np.percentile(ri, 90):.3f}")
full = tr.cpu().numpy().astype(np.int64)
dbg = full[f.info["records"]:f.info["records"] + 16384]
dbg = dbg[dbg[:, 0] > 0]
dd = np.diff(dbg, axis=1)
for j, nm in enumerate(["record wait", "inputs+blocks staged", "halo wait", "hand-over wait", "chain",
                        "global stores+arrives", "prefetch issue"]):
    print(f"  cycles {nm}: med {np.median(dd[:, j]):.0f} p90 {np.percentile(dd[:, j], 90):.0f}")
gap = dbg[1:, 0] - dbg[:-1, 7]
print(f"  cycles loop back: med {np.median(gap[(gap > 0) & (gap < 1e6)]):.0f}")
if "--out" in sys.argv:
    np.savez_compressed(sys.argv[sys.argv.index("--out") + 1], trace=t)
