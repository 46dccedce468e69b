"""bench.py's multi-rank host logic on CPU with gloo, world size 2 (no GPU).

Every rank solves its own endgames (weak scaling): seeds differ per
rank, the timed region is the max over ranks, and the reported value counts every rank's
games."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    args = type("A", (), {"workload": "libratus", "seed": 2100, "batch": 4})()
    r, local, w = bench.dist_env()
    spec, boards, p1, p2 = bench.workload(args, r)
    gathered = [None] * world
    dist.all_gather_object(gathered, boards.tolist())
    ms = bench.max_over_ranks(10.0 + 5.0 * r, w)
    out[rank] = {"env": (r, local, w), "boards": gathered, "ms": ms,
                 "value": bench.throughput(args.batch, w, 7, ms)}
    dist.barrier()
    dist.destroy_process_group()


def bench_grads():
    import bench
    return bench.GRADS_PER_STEP


def test_two_ranks_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        assert res[rank]["env"] == (rank, rank, world)
        assert res[rank]["ms"] == 15.0                      # max over ranks
        assert res[rank]["value"] == pytest.approx(bench_grads() * 4 * 2 * 7 / 0.015)
    b0, b1 = (np.array(b) for b in res[0]["boards"])
    assert b0.shape == b1.shape == (4, 5)
    assert not np.array_equal(b0, b1)                         # independent endgames per rank
    assert res[0]["boards"] == res[1]["boards"]


def test_single_rank_defaults():
    import bench
    assert bench.max_over_ranks(3.5, 1) == 3.5
    assert bench.throughput(296, 1, 10, 1000.0) == bench.GRADS_PER_STEP * 296 * 10


def _uid_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1810_03063_b200 import binding
    uid = bytes(range(128)) if rank == 0 else None
    out[rank] = binding.broadcast_uid(uid)
    dist.destroy_process_group()


def test_nccl_uid_broadcast_gloo():
    """Row 8's host plumbing: rank 0's NCCL unique id reaches every rank."""
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_uid_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0] == res[1] == bytes(range(128))
