"""World-size-2 checks of the multi-rank path on CPU (gloo), as the bench
runs it under torchrun with nccl: the Shard layout, max-over-ranks timing and
the final ordering check's digest gather.  The per-rank element order is the
oracle's shard -> shuffle order (P/tests/test_iterator.cpp:191-210: the union
of all shards is the input multiset), digested with the K7 definition that
the GPU parity tests pin against the kernel.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_per_rank, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from tests.oracle_lib import Oracle
    orc = Oracle()
    lay = bench.shard_layout(world, rank, n_per_rank)
    pos = orc.shard_positions(lay["global_count"], world, rank)
    assert pos.size == lay["resident"]
    ids = pos[orc.shuffle_order(pos.size, 300, orc.shuffle_seed(1, 42))]
    digest = torch.tensor([np.int64(np.uint64(orc.order_digest(ids[:8 * 64])).view(np.int64))])
    digests = bench.gather_digests(digest, world)
    ms_max = bench.max_over_ranks(10.0 + rank, world, "cpu")
    gathered = [torch.zeros(lay["resident"], dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(ids))
    if rank == 0:
        out.put({"digests": digests, "ms_max": ms_max, "all": torch.cat(gathered).numpy().tolist()})
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_layout_timing_and_order_check(orc):
    world, n_per_rank = 2, 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_per_rank, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["ms_max"] == 11.0  # max over ranks, not rank 0's own
    assert sorted(res["all"]) == list(range(world * n_per_rank))  # union of shards = input
    for r in range(world):
        pos = orc.shard_positions(world * n_per_rank, world, r)
        ids = pos[orc.shuffle_order(pos.size, 300, orc.shuffle_seed(1, 42))]
        assert res["digests"][r] == f"{orc.order_digest(ids[:8 * 64]):016x}"
    assert res["digests"][0] != res["digests"][1]
