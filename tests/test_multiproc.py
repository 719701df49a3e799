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


def test_bench_gpus_n_launches_n_ranks():
    """`bench.py --gpus N` outside torchrun re-runs itself as N ranks
    (torch.distributed.run, 127.0.0.1); rank 0 sees the whole group, the
    max over ranks and every rank's digest, plus the golden order digests
    of that world size."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--probe-launch",
                          "--config", "cfg3"], capture_output=True, text=True, env=env, cwd=root, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["ms_max"] == 2.0
    assert line["per_rank"] == [f"{0:016x}", f"{1001:016x}"]
    assert None not in line["expected"] and line["expected"][0] != line["expected"][1]


def test_bench_rejects_world_size_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--probe-launch"],
                         capture_output=True, text=True, env=env, cwd=root, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=2" in out.stderr


def test_golden_order_check_table_matches_the_oracle(orc):
    """tests/golden/order_check.json (what bench.py compares each rank's
    device digest with) recomputed from the oracle for a sample of keys."""
    import json
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(here, "golden"))
    import make_order_check as m
    table = json.load(open(os.path.join(here, "golden", "order_check.json")))["entries"]
    for config, world, rank in [("cfg2", 1, 0), ("cfg3", 8, 5), ("cfg5", 4, 3), ("cfg1", 2, 1), ("cfg4", 1, 0),
                                ("cfg4r", 2, 1), ("cfg4b", 1, 0)]:
        n = m.SIZES[config]
        assert table[f"{config}/n{n}/w{world}/r{rank}"] == f"{m.expected(orc, config, world, rank, n):016x}"


def test_bench_launch_tiling_puts_the_window_on_group_boundaries():
    """bench.py honours --steps/--warmup exactly: the chosen tiling has launch
    boundaries at both ends of the timed window (simulated group starts,
    same rule as DevicePipeline::GroupRange)."""
    import bench

    def starts(d, head, bpe, upto):
        out, e = set(), 0
        while e * bpe <= upto:
            k = 0
            while k < bpe:
                out.add(e * bpe + k)
                k += head if (e == 0 and head and k == 0) else d
            e += 1
        return out

    for w, k, gmax, bpe in [(5, 20, 21, 256), (32, 512, 21, 256), (3, 7, 16, 256), (16, 16, 16, 256), (5, 300, 21, 256),
                            (7, 1000, 21, 100), (4, 4, 1, 10)]:
        d, head = bench.launch_tiling_for(w, k, gmax, bpe)
        st = starts(d, head, bpe, w + k + bpe)
        assert w in st and (w + k) in st, (w, k, d, head)
        assert 1 <= d <= gmax
    assert bench.launch_tiling_for(5, 20, 21, 256) == (20, 5)
    assert bench.launch_tiling_for(32, 512, 21, 256) == (16, 0)
