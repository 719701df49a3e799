"""Generates tests/golden/token_digests.json: whole-epoch output digests of
the BASELINE.json token configurations at full size (1M sequences, len
U[1,1024], seed 4) for tests/test_gpu_fullsize.py:

  cfg4   filter(len <= 512) -> padded_batch(128, pad 0): every padded batch
         matrix (rows x Lmax int32, row major) back to back, and the lengths
  cfg4r  filter(len <= 512) -> batch(128) (ragged): the values back to back,
         and each batch's int64 row splits
  cfg4b  filter -> shuffle(10000, 42) -> bucket_by_length(128/256/384;
         256/128/96/64): the padded bucket batches back to back, and lengths

digest = K7's position hash (SplitMix64Next(w ^ p * 0x9E3779B97F4A7C15))
summed over the words, p running across the epoch.  Orders, filter and
bucketing come from the oracle restatement (pinned against the compiled
reference by tests/test_oracle.py); tokens from the synthetic formula.

    python tests/golden/make_token_digests.py
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.oracle_lib import Oracle  # noqa: E402

N, SEED, MAX_LEN, KEEP, BATCH = 1_000_000, 4, 1024, 512, 128
GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix(z):
    with np.errstate(over="ignore"):
        z = z + GOLD
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def digest(words, first):
    """sum over i of SplitMix64Next(words[i] ^ (first + i) * golden) mod 2^64"""
    w = np.ascontiguousarray(words).astype(np.uint64)
    with np.errstate(over="ignore"):
        p = np.arange(first, first + w.size, dtype=np.uint64) * GOLD
        return int(splitmix(w ^ p).sum(dtype=np.uint64))


def row_tokens(rows, lens, offs_unused=None):
    """tokens of the given sequence indices (concatenated) -- the synthetic formula."""
    l = lens[rows].astype(np.int64)
    i = np.repeat(rows.astype(np.uint64), l)
    starts = np.concatenate([[0], np.cumsum(l)[:-1]])
    j = (np.arange(int(l.sum()), dtype=np.int64) - np.repeat(starts, l)).astype(np.uint64)
    with np.errstate(over="ignore"):
        s = np.uint64(SEED) ^ ((i << np.uint64(20)) | j)
        return (splitmix(s) & np.uint64(0x7FFFFFFF)).astype(np.uint32)


def padded_digest(batches, lens):
    """batches: list of position arrays -> (digest of padded matrices, digest of lengths, total words)"""
    acc = accl = pos = posl = 0
    for b in batches:
        l = lens[b].astype(np.int64)
        lm = int(l.max())
        mat = np.zeros((b.size, lm), np.uint32)
        mask = np.arange(lm)[None, :] < l[:, None]
        mat[mask] = row_tokens(b, lens)
        acc = (acc + digest(mat.reshape(-1), pos)) % 2 ** 64
        accl = (accl + digest(l.astype(np.uint32), posl)) % 2 ** 64
        pos += mat.size
        posl += b.size
    return acc, accl, pos


def main():
    orc = Oracle()
    lens = orc.lengths(N, MAX_LEN, SEED)
    kept = orc.filter_len_le(lens, KEEP)
    out = {"generator": "tests/golden/make_token_digests.py (oracle restatement + the synthetic token formula)",
           "n": N, "seed": SEED, "max_len": MAX_LEN, "keep": KEEP, "cases": {}}
    t = time.time()
    batches = [kept[k:k + BATCH] for k in range(0, kept.size, BATCH)]
    d, dl, words = padded_digest(batches, lens)
    out["cases"]["cfg4"] = {"batches": len(batches), "words": words, "tokens": f"{d:016x}", "lengths": f"{dl:016x}"}
    print("cfg4", out["cases"]["cfg4"], f"{time.time() - t:.0f}s", flush=True)
    t = time.time()
    acc = accs = pos = poss = 0
    for b in batches:
        toks = row_tokens(b, lens)
        acc = (acc + digest(toks, pos)) % 2 ** 64
        pos += toks.size
        splits = np.concatenate([[0], np.cumsum(lens[b].astype(np.int64))])
        accs = (accs + digest(splits, poss)) % 2 ** 64
        poss += splits.size
    out["cases"]["cfg4r"] = {"batches": len(batches), "tokens": pos, "values": f"{acc:016x}", "splits": f"{accs:016x}"}
    print("cfg4r", out["cases"]["cfg4r"], f"{time.time() - t:.0f}s", flush=True)
    t = time.time()
    order = kept[orc.shuffle_order(kept.size, 10000, orc.shuffle_seed(1, 42))]
    bb = orc.bucket_by_length(lens, order, [128, 256, 384], [256, 128, 96, 64])
    d, dl, words = padded_digest(bb, lens)
    out["cases"]["cfg4b"] = {"batches": len(bb), "words": words, "tokens": f"{d:016x}", "lengths": f"{dl:016x}"}
    print("cfg4b", out["cases"]["cfg4b"], f"{time.time() - t:.0f}s", flush=True)
    with open(os.path.join(HERE, "token_digests.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
