"""Independent systems spread over ranks (BASELINE configs[4]).

A single system is never split (block-Jacobi or halo exchange would change
the preconditioner).  With G ranks, rank g solves the contiguous shard
[g*S/G, (g+1)*S/G) of the S systems -- no collective on the data path; one
all_gather of the per-system statistics at the end, and the elapsed time is
the max over ranks.  ``run_sharded`` is the driver bench.py uses; the local
solve is a callable, so the sharding / gathering / reduction logic runs (and
is tested) on CPU with the gloo backend as well.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass


@dataclass
class SystemResult:
    system: int
    rank: int
    iterations: int
    converged: bool
    rel_residual: float
    setup_s: float
    solve_s: float


def shard(num_systems: int, world: int, rank: int) -> range:
    """Contiguous, balanced shard of system indices owned by ``rank`` (any S, G)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return range(rank * num_systems // world, (rank + 1) * num_systems // world)


def gather_results(local: list, dist=None) -> list:
    """All ranks' results, ordered by system index (one all_gather_object)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return sorted(local, key=lambda r: r.system)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, [asdict(r) for r in local])
    out = [SystemResult(**d) for part in parts for d in part]
    return sorted(out, key=lambda r: r.system)


def max_over_ranks(values, dist=None, device=None):
    """Element-wise max of a list of floats over ranks (one all_reduce)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in values]
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def run_sharded(num_systems: int, solve_local, dist=None, device=None):
    """Shard ``num_systems`` over the ranks of ``dist`` and solve this rank's share.

    ``solve_local(indices) -> (list[SystemResult], timings: dict[str, float])``
    solves the given global system indices on this rank (the seeds follow the
    global index, so the union over ranks is the same batch for any G).
    Returns (every rank's results by system, timings max-reduced over ranks).
    """
    world = dist.get_world_size() if dist is not None and dist.is_initialized() else 1
    rank = dist.get_rank() if dist is not None and dist.is_initialized() else 0
    mine = shard(num_systems, world, rank)
    local, timings = solve_local(list(mine))
    keys = sorted(timings)
    red = max_over_ranks([timings[k] for k in keys], dist, device)
    return gather_results(local, dist), dict(zip(keys, red))
