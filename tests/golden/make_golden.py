"""Generates tests/golden/golden.json from the COMPILED REFERENCE.

Runs oracle/_ref/libdpref.so -- the reference's own sources from
/root/reference/proj/src compiled in place by oracle/Makefile -- through its
operator API (ops::*, Optimize, MakeIterator/GetNext with seed_override) and
records known answers.  Needs /root/reference at build time only; the JSON is
committed so the CPU and GPU suites never read /root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from tests.oracle_lib import Oracle, Reference  # noqa: E402

SHUFFLE_CASES = [
    # (n, buffer, seed, base_seed)
    (1, 1, 42, 1), (5, 1, 42, 1), (5, 8, 7, 1), (5, 8, 7, 2), (10, 10, 3, 1), (11, 10, 3, 1),
    (100, 7, 0, 5), (1000, 1000, 9, 1), (1000, 999, 9, 1), (1000, 1001, 9, 1), (4097, 64, 123, 77),
    (20000, 10000, 42, 1), (65536, 10000, 42, 1), (100000, 3, 5, 9), (30000, 30000, 1, 1),
    (70000, 60000, 11, 3), (333, 32, 2**63 + 5, 2**40 + 1), (1025, 31, 8, 8), (1025, 33, 8, 8),
]
INTERLEAVE_CASES = [
    # (num_sources, cycle, records, parallel, shard_k, shard_g)
    (1, 1, 1, 1, 0, 0), (5, 2, 3, 1, 0, 0), (5, 2, 3, 2, 0, 0), (13, 4, 7, 1, 0, 0), (13, 4, 7, 4, 0, 0),
    (8, 3, 1, 3, 0, 0), (2, 4, 3, 1, 0, 0), (64, 4, 16, 4, 8, 3), (64, 4, 16, 1, 8, 7), (17, 4, 5, 2, 8, 0),
]


def main():
    orc, ref = Oracle(), Reference.load()
    if ref is None:
        sys.exit("compiled reference unavailable (needs /root/reference)")
    g = {"generator": "tests/golden/make_golden.py over oracle/_ref/libdpref.so (reference runtime)",
         "digest": "fnv: h=0xcbf29ce484222325; h=(h^v)*0x100000001b3 over int64 values (SURVEY.md Appendix A)"}

    cfg1 = {}
    for n in (1_000_000, 1 << 20, 1, 1023, 1024, 1025):
        vals, sizes, kind = ref.range_map_batch(n, batch=1024)
        cfg1[str(n)] = {"root_kind": kind, "num_batches": int(sizes.size), "last_batch": int(sizes[-1]),
                        "sum": int(vals.sum()), "fnv": f"{orc.fnv_digest(vals):016x}"}
    g["cfg1_range_map_batch_1024"] = cfg1

    sh = []
    for (n, b, seed, base) in SHUFFLE_CASES:
        ids = ref.shuffle_ids(n, b, seed=seed, base_seed=base)
        sh.append({"n": n, "buffer": b, "seed": seed, "base_seed": base, "first": ids[:8].tolist(),
                   "last": ids[-4:].tolist(), "fnv": f"{orc.fnv_digest(ids):016x}"})
    big = ref.shuffle_ids(1_000_000, 10000, seed=42, base_seed=1)
    sh.append({"n": 1_000_000, "buffer": 10000, "seed": 42, "base_seed": 1, "first": big[:8].tolist(),
               "last": big[-4:].tolist(), "fnv": f"{orc.fnv_digest(big):016x}"})
    g["shuffle"] = sh

    unseeded = ref.shuffle_ids(5000, 100, seed=None, base_seed=3, has_seed=False)
    g["shuffle_unseeded"] = {"n": 5000, "buffer": 100, "base_seed": 3, "fnv": f"{orc.fnv_digest(unseeded):016x}"}

    rep = []
    for optimize in (False, True):
        ids = ref.shuffle_ids(3000, 500, seed=42, base_seed=1, epochs=3, optimize=optimize)
        rep.append({"n": 3000, "buffer": 500, "seed": 42, "base_seed": 1, "epochs": 3, "optimize": optimize,
                    "fnv": f"{orc.fnv_digest(ids):016x}"})
    g["shuffle_repeat"] = rep

    shs = []
    for (k, gg) in ((2, 0), (2, 1), (8, 3), (8, 7)):
        ids = ref.shuffle_ids(50000, 10000, seed=42, base_seed=1, shard=(k, gg))
        shs.append({"n": 50000, "buffer": 10000, "seed": 42, "base_seed": 1, "shard": [k, gg],
                    "count": int(ids.size), "fnv": f"{orc.fnv_digest(ids):016x}"})
    g["shard_shuffle"] = shs

    il = []
    for (m, c, L, p, k, gg) in INTERLEAVE_CASES:
        ids = ref.interleave_ids(m, c, L, parallel=p, shard=(k, gg) if k else None)
        il.append({"num_sources": m, "cycle": c, "records": L, "parallel": p, "shard": [k, gg],
                   "count": int(ids.size), "first": ids[:8].tolist(), "fnv": f"{orc.fnv_digest(ids):016x}"})
    ids = ref.interleave_ids(64, 4, 32, parallel=4, shard=(8, 5), shuffle_buffer=100, shuffle_seed=42)
    il.append({"num_sources": 64, "cycle": 4, "records": 32, "parallel": 4, "shard": [8, 5], "shuffle": [100, 42],
               "count": int(ids.size), "first": ids[:8].tolist(), "fnv": f"{orc.fnv_digest(ids):016x}"})
    g["interleave"] = il

    row_len, toks, sizes = ref.filter_batch_tokens(3000, max_keep=512, batch=128)
    g["cfg4_filter_batch"] = {"n": 3000, "max_keep": 512, "batch": 128, "len_seed": 4, "max_len": 1024,
                              "tok_seed": 4, "rows": int(row_len.size), "num_batches": int(sizes.size),
                              "last_batch": int(sizes[-1]), "fnv_row_lengths": f"{orc.fnv_digest(row_len):016x}",
                              "fnv_tokens": f"{orc.fnv_digest(toks):016x}",
                              "fnv_batch_sizes": f"{orc.fnv_digest(sizes):016x}"}

    def words_fnv(pix):
        w = np.ascontiguousarray(pix).view(np.uint32).astype(np.int64)
        return f"{orc.fnv_digest(w):016x}"

    img = []
    for (mode, n, in_hw, buf, batch, shard) in ((0, 600, (256, 256), 256, 64, None),
                                                 (2, 300, (256, 256), 100, 32, None),
                                                 (1, 200, (320, 320), 0, 48, None),
                                                 (1, 300, (320, 320), 64, 32, (4, 1))):
        ids, pix, sizes = ref.image_pipeline(mode, n, in_hw, (224, 224), shuffle_buffer=buf, batch=batch,
                                             shard=shard)
        img.append({"mode": mode, "n": n, "in_hw": list(in_hw), "out_hw": [224, 224], "shuffle_buffer": buf,
                    "shuffle_seed": 42, "batch": batch, "shard": list(shard) if shard else None,
                    "udf_seed": 7, "pix_seed": 0x5EED, "base_seed": 1, "batch_sizes": sizes.tolist(),
                    "fnv_ids": f"{orc.fnv_digest(ids):016x}", "fnv_pixels": words_fnv(pix)})
    g["image_pipelines"] = img

    # interleave over readers of unequal lengths (record files of different
    # sizes): the sequential order, and the parallel one where it agrees (no
    # empty reader -- see DESIGN.md 6d)
    rng = np.random.default_rng(21)
    ivar = []
    for case in range(24):
        m, c = int(rng.integers(1, 14)), int(rng.integers(1, 6))
        lens = rng.integers(0 if case % 3 == 0 else 1, 9, m)
        shard = [int(x) for x in rng.choice([[0, 0], [2, 1], [3, 0]])]
        p = 1 if case % 3 == 0 else c
        ids = ref.interleave_var_ids(lens, c, p, tuple(shard) if shard[0] else None)
        ivar.append({"lengths": lens.tolist(), "cycle": c, "parallel": p, "shard": shard,
                     "order": ids.tolist()})
    g["interleave_var"] = ivar

    # value filters (keep_even / keep_odd after an affine map), unoptimized and
    # optimized (map_filter_fusion), with and without a shuffle after them
    vf = []
    for (n, a, b, odd, buf) in ((1000, 3, 1, 0, 0), (1000, 3, 1, 1, 0), (5000, -7, 2, 0, 300), (777, 1, 0, 1, 50)):
        for opt in (0, 1):
            vals, graph = ref.filter_values(n, a, b, odd, buf, opt)
            vf.append({"n": n, "a": a, "b": b, "odd": odd, "shuffle": buf, "optimize": opt,
                       "count": int(vals.size), "first": vals[:6].tolist(), "fnv": f"{orc.fnv_digest(vals):016x}",
                       "graph": graph})
    g["value_filters"] = vf

    ser = []
    for which in range(6):  # pipeline shapes: oracle/ref_shim.cpp ref_serialize_pipeline
        b, fp = ref.serialize_pipeline(which)
        ser.append({"which": which, "dpg1_hex": b.hex(), "fingerprint": fp})
    g["serialize"] = ser
    g["checkpoint"] = [{"which": w, "k": k, "dpc1_hex": ref.checkpoint_after(w, k).hex()}
                       for (w, k) in ((1, 1), (2, 5), (2, 0), (3, 0))]

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
