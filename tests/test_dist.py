"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 bench path:
independent instances per rank (weak scaling, no data-path collective) and
the max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    ids = bench.instance_ids(rank, 5)
    t = bench.max_over_ranks(10.0 + rank)  # each rank reports its own time
    got = [None] * ws
    dist.all_gather_object(got, ids)
    q.put((rank, t, got))
    dist.destroy_process_group()


def test_two_rank_weak_scaling_helpers():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, got in res:
        assert t == 11.0  # max over ranks
        flat = [i for ids in got for i in ids]
        assert len(set(flat)) == len(flat) == 10  # disjoint instances per rank


def test_single_rank_identity():
    assert bench.max_over_ranks(3.5) == 3.5
    assert bench.instance_ids(0, 3) == [0, 1, 2]
