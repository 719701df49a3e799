"""The multi-rank bench path on the one GPU of the test box: two torchrun
ranks (gloo for the 8-byte collectives, DP_BENCH_ONE_GPU=1) each run the
cfg2 / cfg3 pipeline on its own shard(2, rank) with sharded residency (and
cfg5 with block residency of its record files).  The final
ordering check's per-rank K7 digests must equal the oracle's digest of
shard(2, rank) -> shuffle(10k, 42) for that rank.  The
ranks' kernels never wait on one another (no data-path collective)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,port", [("cfg2", 29533), ("cfg3", 29535)])
def test_two_rank_bench_order_check_matches_oracle(orc, config, port):
    """cfg2 (crop) and cfg3 (resize, "1/2/4/8 GPUs via Shard") on two ranks."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n = 8192
    env = dict(os.environ, DP_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "32",
           "--warmup", "16", "--elements-per-gpu", str(n), "--config", config]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["batches_in_window"] == 32
    digests = line["order_check"]["per_rank"]
    for r in range(2):
        pos = orc.shard_positions(2 * n, 2, r)
        # the bench graph repeats above the batch: epoch 0's shuffle is salted
        # MixSeeds(base, 0) (RepeatIterator::MakeChild, runtime.cpp:1175-1177)
        ids = pos[orc.shuffle_order(pos.size, 10000, orc.shuffle_seed(orc.mix_seeds(1, 0), 42))]
        assert digests[r] == f"{orc.order_digest(ids[:8 * 256]):016x}", r


def test_two_rank_cfg5_block_residency_order_check(orc):
    """cfg5 on two ranks: each holds only the record files of its
    shard(2, rank) of the interleave's inputs; its digest equals the oracle's
    interleave (closed form) -> shuffle(10k, 42) of those files."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n, files = 8192, 32  # per rank: 32 files of 256 records
    env = dict(os.environ, DP_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29534", os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "32",
           "--warmup", "16", "--elements-per-gpu", str(n), "--config", "cfg5"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["batches_in_window"] == 32 and line["e2e"]["value"] > 0
    digests = line["order_check"]["per_rank"]
    for r in range(2):
        inter = orc.interleave_order(np.arange(r, 2 * files, 2), 4, n // files)
        ids = inter[orc.shuffle_order(inter.size, 10000, orc.shuffle_seed(orc.mix_seeds(1, 0), 42))]
        assert digests[r] == f"{orc.order_digest(ids[:8 * 256]):016x}", r


def test_self_launched_two_ranks_full_size_order_check():
    """the driver's own command shape, `bench.py --gpus 2`
    with no torchrun around it, spawns two ranks; at the full cfg3 size
    (65,536 images per rank) each rank's digest equals the golden oracle
    digest (tests/golden/order_check.json) and the line says so."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["DP_BENCH_ONE_GPU"] = "1"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "20", "--warmup",
                          "5", "--config", "cfg3"], capture_output=True, text=True, env=env, cwd=ROOT, timeout=1200)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["comm"]["world_size"] == 2
    assert line["steps"] == 20 and line["warmup"] == 5 and line["batches_in_window"] == 20
    assert line["order_check"]["ok"] is True, line["order_check"]
