"""world_size-2 gloo run of the N>1 plumbing: env sharding + the
episode-statistics all-gather (the path's only collective)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1904_01201_b200.dist import EnvShard, gather_records
    shard = EnvShard(n_total=7, world=world, rank=rank)
    # records encode the global env id so the gathered order can be checked
    ids = torch.arange(shard.lo, shard.hi, dtype=torch.float64)
    rec = torch.stack([ids, ids * 2, ids + 0.5, -ids, ids ** 2], dim=1)
    out = gather_records(rec, world)
    if rank == 0:
        q.put(out.numpy().tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_gather_records_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = [row[0] for row in out]
    assert ids == list(range(7))
    assert all(row[1] == 2 * row[0] and row[4] == row[0] ** 2 for row in out)
