"""Critical path of the partitioned ILU(0) sweep from a trace (tools/trace_psweep.py --out).

    python tools/critpath.py gpurun_out/ptrace_k0.npz

For the grid-column partition (py x pz parts of nx x nx columns, part c =
b * py + a, psweep_plan.cpp partition_columns) the L record j of part (a, b) holds level y0 + z0 + j and depends
on the same part's record j - 1 and on level - 1 of parts (a-1, b), (a, b-1);
U' mirrors it.  Walking back from the last record, every step is charged to
what the record waited on last: its own previous record (the chain), its
bulk copy landing, or a cross-part dependency.
"""
import sys

import numpy as np


def load(path, nx=128):
    z = np.load(path)
    tr = z["trace"]
    info = dict(zip([str(k) for k in z["keys"]], z["info"]))
    py, pz = int(info["split_y"]), int(info["split_z"])
    cta = (tr[:, 6] >> 32).astype(np.int64)
    fl = tr[:, 7]
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    t = (tr[:, :6] - t0) / 1e3
    # column j belongs to part floor(j * p / nx): part a starts at ceil(a * nx / p)
    yb = [-(-nx * i // py) for i in range(py + 1)]
    zb = [-(-nx * i // pz) for i in range(pz + 1)]
    L, U = {}, {}
    for c in range(py * pz):
        m = np.where(cta == c)[0]
        a, b = c % py, c // py
        up = (fl[m] & 1) != 0
        l0 = yb[a] + zb[b]
        u0 = (nx - yb[a + 1]) + (nx - zb[b + 1])
        for j, r in enumerate(m[~up]):
            L[(c, l0 + j)] = t[r]
        for j, r in enumerate(m[up]):
            U[(c, u0 + j)] = t[r]
    return L, U, py, pz


def walk(R, py, pz, upstream):
    last = max(R, key=lambda k: R[k][5])
    cur = last
    acc = {"chain": [0, 0.0], "prep": [0, 0.0], "landing": [0, 0.0], "dependency": [0, 0.0]}
    while True:
        c, l = cur
        a, b = c % py, c // py
        ups = [(cc, l - 1) for cc in upstream(a, b) if (cc, l - 1) in R]
        own = (c, l - 1) if (c, l - 1) in R else None
        if own is None and not ups:
            break
        r = R[cur]
        oe = R[own][5] if own else -1e9
        ue = max((R[k][5] for k in ups), default=-1e9)
        if r[4] <= oe + 0.05 or (own and r[3] <= oe):
            prev, kind = own, "chain"            # ready in time: the hand-over chain
        elif ue > oe - 0.05 and r[3] > r[2] + 0.05:
            prev, kind = max(ups, key=lambda k: R[k][5]), "dependency"
        elif own is not None and r[1] > oe:
            prev, kind = own, "landing"          # its bulk copy had not landed
        else:
            prev, kind = (own if own else max(ups, key=lambda k: R[k][5])), "prep"
        acc[kind][0] += 1
        acc[kind][1] += r[5] - R[prev][5]
        cur = prev
    return R[last][5] - R[cur][4], acc


def main(path):
    L, U, py, pz = load(path)
    def upL(a, b):
        return ([b * py + a - 1] if a > 0 else []) + ([(b - 1) * py + a] if b > 0 else [])
    def upU(a, b):
        return ([b * py + a + 1] if a + 1 < py else []) + ([(b + 1) * py + a] if b + 1 < pz else [])
    for name, R, up in (("L", L, upL), ("U'", U, upU)):
        span, acc = walk(R, py, pz, up)
        print(f"{name}: critical path {span:.1f} us: " + "; ".join(
            f"{k} {n} steps {tt:.1f} us ({tt / max(1, n):.3f})" for k, (n, tt) in acc.items()))
    lend = max(v[5] for v in L.values())
    ustart = min(v[4] for v in U.values())
    print(f"L end {lend:.1f}  first U' start {ustart:.1f}  U' end {max(v[5] for v in U.values()):.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
