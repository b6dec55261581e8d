"""N > 1 host logic on CPU: sharding of independent systems and the stats
gather over a world_size-2 gloo group (no GPU; the solver is a stand-in)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1703_01325_b200.batch import SystemResult, gather_results, run_shard, shard


def test_shard_covers_every_system_once():
    for num in (1, 7, 64, 65):
        for world in (1, 2, 3, 4, 8):
            seen = [i for r in range(world) for i in shard(num, world, r)]
            assert seen == list(range(num))
            sizes = [len(shard(num, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def fake_solve(i):
        return SystemResult(system=i, rank=rank, iterations=10 + i, converged=True, rel_residual=1e-7,
                            setup_s=0.0, solve_s=0.001 * i)

    local = run_shard(64, world, rank, fake_solve)
    everything = gather_results(local, dist)
    t = torch.tensor([sum(r.solve_s for r in local)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)      # wall time = max over ranks
    if rank == 0:
        torch.save({"systems": [r.system for r in everything], "ranks": [r.rank for r in everything],
                    "iters": [r.iterations for r in everything], "tmax": float(t.item())}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_gather(tmp_path):
    out = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = torch.load(out)
    assert res["systems"] == list(range(64))
    assert res["ranks"] == [0] * 32 + [1] * 32
    assert res["iters"] == [10 + i for i in range(64)]
    assert res["tmax"] == pytest.approx(sum(0.001 * i for i in range(32, 64)))
