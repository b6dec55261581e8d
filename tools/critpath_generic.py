"""Critical path of the partitioned sweep from a trace, for contiguous-row
partitions (parts depend on the parts just before them in the L sweep and just
after them in U').  Record levels come from the header flags (>> 10).

    python tools/critpath_generic.py gpurun_out/ptrace_k2.npz [reach]
"""
import sys

import numpy as np


def main(path, reach=4):
    z = np.load(path)
    tr = z["trace"]
    cta = (tr[:, 6] >> 32).astype(np.int64)
    fl = tr[:, 7].astype(np.int64)
    lev, up = fl >> 10, fl & 1
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    t = (tr[:, :6] - t0) / 1e3
    for sweep in (0, 1):
        idx = np.where(up == sweep)[0]
        # per (part, level): the last record of that part at that level
        last = {}
        for r in idx:
            k = (cta[r], lev[r])
            if k not in last or t[r, 5] > t[last[k], 5]:
                last[k] = r
        prev_own = {}
        for c in np.unique(cta[idx]):
            rs = idx[cta[idx] == c]
            for a, b in zip(rs[:-1], rs[1:]):
                prev_own[b] = a
        end = idx[np.argmax(t[idx, 5])]
        cur = end
        acc = {"chain": [0, 0.0], "prep": [0, 0.0], "landing": [0, 0.0], "dependency": [0, 0.0]}
        while True:
            c, l = cta[cur], lev[cur]
            own = prev_own.get(cur)
            sgn = -1 if sweep == 0 else 1
            ups = [last[(c + sgn * d, l - 1)] for d in range(1, reach + 1) if (c + sgn * d, l - 1) in last]
            if own is None and not ups:
                break
            r = t[cur]
            oe = t[own, 5] if own is not None else -1e9
            ue = max((t[u, 5] for u in ups), default=-1e9)
            if own is not None and (r[4] <= oe + 0.05 or r[3] <= oe):
                prev, kind = own, "chain"
            elif ups and ue > oe - 0.05 and r[3] > r[2] + 0.05:
                prev, kind = max(ups, key=lambda u: t[u, 5]), "dependency"
            elif own is not None and r[1] > oe:
                prev, kind = own, "landing"
            else:
                prev, kind = (own if own is not None else max(ups, key=lambda u: t[u, 5])), "prep"
            acc[kind][0] += 1
            acc[kind][1] += r[5] - t[prev, 5]
            cur = prev
        span = t[end, 5] - t[cur, 4]
        print(("L" if sweep == 0 else "U'") + f": critical path {span:.1f} us: " + "; ".join(
            f"{k} {n} steps {tt:.1f} us ({tt / max(1, n):.3f})" for k, (n, tt) in acc.items()))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4)
