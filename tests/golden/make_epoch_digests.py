"""Generates tests/golden/epoch_digests.json: whole-epoch output digests of
the BASELINE.json image configurations at full size, for the GPU parity
test tests/test_gpu_fullsize.py (full-size parity must cover
every output byte, not samples).

Per case: the element order of one epoch (the oracle's reservoir shuffle /
interleave restatement, pinned against the compiled reference by
tests/test_oracle.py), then every image through the oracle's map chain
(oracle/chain.c) with the K7 position hash summed over the epoch's u32 words
(the device side runs dp_k_word_digest over each batch).  ~1-2 minutes on 8
host threads.

    python tests/golden/make_epoch_digests.py
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.oracle_lib import MEAN, STD, Oracle  # noqa: E402

CROP = [["random_crop", 224, 224, 7, True], ["normalize", list(MEAN), list(STD)]]
RESIZE = [["resize", 224, 224], ["normalize", list(MEAN), list(STD)]]
RRC = [["random_crop", 160, 160, 7, True], ["resize", 224, 224], ["normalize", list(MEAN), list(STD)]]
EVAL = [["resize", 256, 256], ["center_crop", 224, 224], ["normalize", list(MEAN), list(STD)]]

CASES = {
    # name: (source, n, hw, steps)
    "cfg2": ("tensor_slices", 65536, 256, CROP),
    "cfg3": ("tensor_slices", 65536, 320, RESIZE),
    "cfg5": ("interleave", 65536, 256, CROP),   # 32 files x 2048 records, cycle 4, parallel 4
    "cfg2rrc": ("tensor_slices", 65536, 256, RRC),   # RandomResizedCrop (K10)
    "cfg3e": ("tensor_slices", 65536, 320, EVAL),    # ResNet eval (K10)
}


def epoch_ids(orc, source, n):
    """Epoch 0 of <source> -> shuffle(10000, seed 42), base seed 1, no repeat."""
    seed = orc.shuffle_seed(1, 42)
    if source == "tensor_slices":
        return orc.shuffle_order(n, 10000, seed)
    inter = orc.interleave_order(np.arange(32), 4, n // 32)
    return inter[orc.shuffle_order(inter.size, 10000, seed)]


def main():
    orc = Oracle()
    only = sys.argv[1:]  # case names to (re)compute; the others are kept from the existing file
    path = os.path.join(HERE, "epoch_digests.json")
    old = json.load(open(path))["cases"] if only and os.path.exists(path) else {}
    out = {"generator": "tests/golden/make_epoch_digests.py (oracle restatement: shuffle / interleave order + "
                        "oracle/chain.c map chain)",
           "digest": "pixels: sum over the epoch's output u32 words w at running position p of "
                     "SplitMix64Next(w ^ p * 0x9E3779B97F4A7C15) mod 2^64; ids: the same over the int64 ids",
           "cases": {}}
    for name, (source, n, hw, steps) in CASES.items():
        if only and name not in only:
            if name in old:
                out["cases"][name] = old[name]
            continue
        t = time.time()
        ids = epoch_ids(orc, source, n)
        pix = orc.epoch_image_digest([tuple(s) for s in steps], ids, hw, hw)
        out["cases"][name] = {"source": source, "n": n, "hw": hw, "steps": steps, "shuffle": [10000, 42],
                              "base_seed": 1, "batch": 256, "ids": f"{Oracle.order_digest(ids):016x}",
                              "pixels": f"{pix:016x}"}
        print(name, out["cases"][name]["ids"], out["cases"][name]["pixels"], f"{time.time() - t:.1f}s", flush=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
