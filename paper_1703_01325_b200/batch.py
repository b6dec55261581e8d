"""Independent systems spread over ranks (BASELINE configs[4]).

A single system is never split (block-Jacobi or halo exchange would change
the preconditioner).  With G ranks, rank g solves the contiguous shard
[g*S/G, (g+1)*S/G) of the S systems -- no collective on the data path; one
all_gather of the per-system statistics at the end, and the wall time is the
max over ranks.  The solver itself is a plain function so the sharding and
gathering logic is testable on CPU (gloo) without a GPU.
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
    """Contiguous, balanced shard of system indices owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return range(rank * num_systems // world, (rank + 1) * num_systems // world)


def run_shard(num_systems: int, world: int, rank: int, solve_one) -> list:
    """Solve this rank's systems; ``solve_one(index) -> SystemResult``."""
    return [solve_one(i) for i in shard(num_systems, world, rank)]


def gather_results(local: list, dist=None) -> list:
    """All ranks' results, ordered by system index (one all_gather_object)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return sorted(local, key=lambda r: r.system)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, [asdict(r) for r in local])
    out = [SystemResult(**d) for part in parts for d in part]
    return sorted(out, key=lambda r: r.system)


def device_solver(nx: int, bs: int, k: int, rel_tol: float = 1e-6, method: str = "bicgstab"):
    """solve_one for the GPU: seeded synthetic system -> ILU(k) -> Krylov (b = A 1)."""
    import time

    import torch

    from . import BcsrMatrix, bicgstab, build_preconditioner, gmres, SolverConfig
    from .synthetic import ones_rhs, reservoir_block_grid

    rank = torch.distributed.get_rank() if torch.distributed.is_initialized() else 0

    def solve_one(i: int) -> SystemResult:
        n, b_, rp, ci, vals = reservoir_block_grid(nx, nx, nx, bs, seed=i)
        a = BcsrMatrix(b_, n, n, rp, ci, vals)
        rhs = torch.from_numpy(ones_rhs(n, b_, rp, ci, vals)).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = build_preconditioner(a, k)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        solver = bicgstab if method == "bicgstab" else gmres
        cfg = SolverConfig(rel_tol=rel_tol, restart=30)
        _, st = solver(a, rhs, M=f, cfg=cfg)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        return SystemResult(i, rank, st.iterations, st.converged, st.final_relative_residual, t1 - t0, t2 - t1)

    return solve_one
