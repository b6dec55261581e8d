"""N > 1 host logic on CPU: the batch driver bench.py uses (``batch.run_sharded``:
shard -> local solve -> all_gather of the per-system statistics -> MAX-reduce of
the timings) over a world_size-2 gloo group.  The local solve is a stand-in
(no GPU); batch sizes that do not divide by the world size are covered."""

import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1703_01325_b200.batch import SystemResult, run_sharded, shard


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


def _fake_solve_local(rank):
    def solve_local(indices):
        # seeds follow the global index (as bench.py generates system i with seed i)
        res = [SystemResult(system=i, rank=rank, iterations=10 + i, converged=True, rel_residual=1e-7,
                            setup_s=0.0, solve_s=0.001 * i) for i in indices]
        return res, {"apply_ms": float(len(indices)), "solve_s": sum(r.solve_s for r in res)}
    return solve_local


def _worker(rank, world, port, num, out_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    everything, timings = run_sharded(num, _fake_solve_local(rank), dist)
    if rank == 0:
        torch.save({"systems": [r.system for r in everything], "ranks": [r.rank for r in everything],
                    "iters": [r.iterations for r in everything], "timings": timings}, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("num", [64, 7])
def test_gloo_world2_run_sharded(tmp_path, num):
    out = str(tmp_path / "res.pt")
    mp.spawn(_worker, args=(2, _free_port(), num, out), nprocs=2, join=True)
    res = torch.load(out)
    half = num // 2
    assert res["systems"] == list(range(num))
    assert res["ranks"] == [0] * half + [1] * (num - half)
    assert res["iters"] == [10 + i for i in range(num)]
    # timings are the max over ranks
    assert res["timings"]["apply_ms"] == float(num - half)
    assert res["timings"]["solve_s"] == pytest.approx(sum(0.001 * i for i in range(half, num)))


def test_run_sharded_single_process():
    everything, timings = run_sharded(5, _fake_solve_local(0), None)
    assert [r.system for r in everything] == list(range(5))
    assert timings["apply_ms"] == 5.0
