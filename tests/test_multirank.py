"""Multi-rank host logic of bench.py on CPU (gloo, world size 2).

The GPU path shards independent pairs over ranks with no data-path
collective; what must hold across processes is the
seed partition, the max-over-ranks timing reduction and rank-0-only output
of the reference arm.  Runs here without a GPU.
"""

import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as tmp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        pairs = 16
        seeds = list(range(bench.rank_seed0(rank, pairs), bench.rank_seed0(rank, pairs) + pairs))
        gathered = [None] * world
        dist.all_gather_object(gathered, seeds)
        # rank r reports (step ms, e2e ms, fields ms); the slowest rank must win each entry
        mine = [10.0 + rank, 50.0 - rank, 3.0 * (rank + 1)]
        red = bench.max_over_ranks(mine, world, "cpu")
        out[rank] = (gathered, red)
    finally:
        dist.destroy_process_group()


def test_seed_partition_and_max_reduction():
    world = 2
    port = _free_port()
    mgr = tmp.Manager()
    out = mgr.dict()
    tmp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        gathered, red = out[rank]
        flat = [s for part in gathered for s in part]
        assert sorted(flat) == list(range(32)) and len(set(flat)) == 32     # disjoint, complete
        assert red == [11.0, 50.0, 6.0]


def test_reference_arm_is_rank0_only(capsys):
    sys.path.insert(0, ROOT)
    import bench

    class A:
        steps, warmup, size, pairs = 1, 0, 64, 1

    bench.run_reference(A, rank=1, world=2)        # must return at once without work or output
    assert capsys.readouterr().out == ""
