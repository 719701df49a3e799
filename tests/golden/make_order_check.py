"""Generates tests/golden/order_check.json: the expected K7 order digest of
each rank's first 8 batches for every bench.py configuration at 1, 2, 4 and
8 GPUs (the "final ordering check").

Computed with the oracle restatement (oracle/restate.c, pinned against the
compiled reference by tests/test_oracle.py) and numpy; tests/test_oracle.py
recomputes a subset.  bench.py compares each rank's device digest with this
table after the timed region, so the bench never executes oracle code.

    python tests/golden/make_order_check.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.oracle_lib import Oracle  # noqa: E402

WORLDS = (1, 2, 4, 8)
FIRST_BATCHES = 8


def expected(orc, config, world, rank, n):
    """The values the bench digests for rank `rank` of `world` (bench.py run_ours)."""
    o = Oracle.order_digest
    salt0 = orc.mix_seeds(1, 0)  # repeat(-1) above the batch: epoch 0 is salted MixSeeds(base, 0)
    if config in ("cfg2", "cfg3", "cfg2u8", "cfg2rrc", "cfg3e"):
        pos = orc.shard_positions(world * n, world, rank) if world > 1 else np.arange(n)
        ids = pos[orc.shuffle_order(pos.size, 10000, orc.shuffle_seed(salt0, 42))]
        return o(ids[:FIRST_BATCHES * 256])
    if config == "cfg5":
        files = 32
        inter = orc.interleave_order(np.arange(rank, files * world, world), 4, n // files)
        ids = inter[orc.shuffle_order(inter.size, 10000, orc.shuffle_seed(salt0, 42))]
        return o(ids[:FIRST_BATCHES * 256])
    if config == "cfg1":
        pos = np.arange(rank, FIRST_BATCHES * 1024 * world, world, dtype=np.int64)[:FIRST_BATCHES * 1024]
        return o(pos * 3 + 1)
    # token configs: every rank holds its own 1M sequences (seed 4 + rank)
    lens = orc.lengths(n, 1024, 4 + rank)
    kept = orc.filter_len_le(lens, 512)
    if config == "cfg4":
        return o(lens[kept[:FIRST_BATCHES * 128]].astype(np.uint32))
    if config == "cfg4r":
        acc, pos = 0, 0
        for j in range(FIRST_BATCHES):
            rows = lens[kept[j * 128:(j + 1) * 128]].astype(np.int64)
            splits = np.concatenate([[0], np.cumsum(rows)])
            acc = (acc + o(splits, pos)) % 2 ** 64
            pos += splits.size
        return acc
    if config == "cfg4b":
        order = kept[orc.shuffle_order(kept.size, 10000, orc.shuffle_seed(salt0, 42))]
        batches = orc.bucket_by_length(lens, order, [128, 256, 384], [256, 128, 96, 64])
        acc, pos = 0, 0
        for b in batches[:FIRST_BATCHES]:
            acc = (acc + o(lens[b].astype(np.uint32), pos)) % 2 ** 64
            pos += b.size
        return acc
    raise KeyError(config)


SIZES = {"cfg1": 1 << 28, "cfg2": 65536, "cfg3": 65536, "cfg5": 65536, "cfg2u8": 65536, "cfg2rrc": 65536,
         "cfg3e": 65536, "cfg4": 1_000_000, "cfg4r": 1_000_000,
         "cfg4b": 1_000_000}


def main():
    orc = Oracle()
    table = {"generator": "tests/golden/make_order_check.py (oracle restatement)",
             "digest": "K7: sum_i SplitMix64Next(v_i ^ (i * 0x9E3779B97F4A7C15)) over each rank's first 8 batches "
                       "(ids; cfg1 values; cfg4/cfg4b row lengths; cfg4r row splits), positions running across "
                       "the batches",
             "entries": {}}
    for config, n in SIZES.items():
        for world in WORLDS:
            for rank in range(world):
                key = f"{config}/n{n}/w{world}/r{rank}"
                table["entries"][key] = f"{expected(orc, config, world, rank, n):016x}"
                print(key, table["entries"][key], flush=True)
    with open(os.path.join(HERE, "order_check.json"), "w") as f:
        json.dump(table, f, indent=1)


if __name__ == "__main__":
    main()
