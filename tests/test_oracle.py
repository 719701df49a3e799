"""Pins the CPU oracle (oracle/restate.c) before anything is checked against it.

* against the known answers generated from the compiled reference
  (tests/golden/golden.json);
* against the compiled reference itself (oracle/_ref), when it is built here;
* Philox4x32-10 against the Random123 known-answer vectors;
* the device normalize's fast exact division against IEEE division over its
  whole (finite) input domain.

Mirrors the reference's own suites: shuffle reproducibility / multiset /
identity (P/tests/test_iterator.cpp:151-189), shard partition (:191-210),
map+batch fusion keeps the partial batch (P/tests/test_optimizer.cpp:102-127).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def fnv(orc, v):
    return f"{orc.fnv_digest(v):016x}"


def restated_shuffle(orc, n, buffer, seed, base_seed, in_map=None):
    order = orc.shuffle_order(n, buffer, orc.shuffle_seed(base_seed, seed))
    return order if in_map is None else np.asarray(in_map)[order]


# ---------------------------------------------------------------- cfg1 ----
def test_cfg1_known_answers(orc):
    for n_str, want in GOLDEN["cfg1_range_map_batch_1024"].items():
        n = int(n_str)
        vals = np.arange(n, dtype=np.int64) * 3 + 1
        nb = (n + 1023) // 1024
        assert want["root_kind"] == "map_and_batch"
        assert want["num_batches"] == nb
        assert want["last_batch"] == n - (nb - 1) * 1024
        assert want["sum"] == int(vals.sum())
        assert want["fnv"] == fnv(orc, vals)
    # SURVEY.md Appendix A
    assert GOLDEN["cfg1_range_map_batch_1024"]["1000000"]["fnv"] == "8bc444c576bd14a5"


# ------------------------------------------------------------- shuffle ----
def test_prng_contract(orc):
    assert orc.shuffle_seed(1, 42) == 0x488DACB220274C43


def test_shuffle_known_answers(orc):
    for case in GOLDEN["shuffle"]:
        got = restated_shuffle(orc, case["n"], case["buffer"], case["seed"], case["base_seed"])
        assert got[:8].tolist() == case["first"], case
        assert got[-4:].tolist() == case["last"], case
        assert fnv(orc, got) == case["fnv"], case
    big = GOLDEN["shuffle"][-1]
    assert big["n"] == 1_000_000 and big["fnv"] == "ea02cb23a74a25ef"
    assert big["first"] == [442, 5136, 5127, 7349, 5098, 8269, 2879, 6576]


def test_shuffle_unseeded_uses_base_seed(orc):
    c = GOLDEN["shuffle_unseeded"]
    got = orc.shuffle_order(c["n"], c["buffer"], orc.shuffle_seed(c["base_seed"], None))
    assert fnv(orc, got) == c["fnv"]


def test_shuffle_repeat_epoch_seeds(orc):
    # RepeatIterator::MakeChild salts epoch e with MixSeeds(salt, e)
    # (runtime.cpp:1175-1177); the fused shuffle derives the same
    # (runtime.cpp:751).  Both rewrites must give one sequence.
    digests = set()
    for c in GOLDEN["shuffle_repeat"]:
        seq = np.concatenate([orc.shuffle_order(c["n"], c["buffer"],
                                                orc.shuffle_seed(orc.mix_seeds(c["base_seed"], e), c["seed"]))
                              for e in range(c["epochs"])])
        assert fnv(orc, seq) == c["fnv"], c
        digests.add(c["fnv"])
    assert len(digests) == 1


def test_shard_then_shuffle(orc):
    for c in GOLDEN["shard_shuffle"]:
        pos = orc.shard_positions(c["n"], *c["shard"])
        got = restated_shuffle(orc, pos.size, c["buffer"], c["seed"], c["base_seed"], in_map=pos)
        assert got.size == c["count"] and fnv(orc, got) == c["fnv"], c


def test_shuffle_properties(orc):
    # identity at buffer 1, reproducible, multiset preserved, seed-sensitive
    assert orc.shuffle_order(5, 1, 123).tolist() == [0, 1, 2, 3, 4]
    a = orc.shuffle_order(1000, 64, orc.shuffle_seed(1, 7))
    assert (a == orc.shuffle_order(1000, 64, orc.shuffle_seed(1, 7))).all()
    assert sorted(a.tolist()) == list(range(1000))
    assert (a != orc.shuffle_order(1000, 64, orc.shuffle_seed(2, 7))).any()


# ----------------------------------------------------------- interleave ----
def test_interleave_known_answers(orc):
    for c in GOLDEN["interleave"]:
        k, g = c["shard"]
        inputs = orc.shard_positions(c["num_sources"], k, g) if k else np.arange(c["num_sources"])
        got = orc.interleave_order(inputs, c["cycle"], c["records"])
        if "shuffle" in c:
            buf, seed = c["shuffle"]
            got = restated_shuffle(orc, got.size, buf, seed, 1, in_map=got)
        assert got.size == c["count"] and got[:8].tolist() == c["first"] and fnv(orc, got) == c["fnv"], c


def closed_form_interleave(inputs, cycle, records):
    """K6's closed form (k_index.cu shard_interleave_kernel)."""
    m_in = len(inputs)
    out = []
    for t in range(m_in * records):
        g = t // (cycle * records)
        g0 = g * cycle
        m = min(cycle, m_in - g0)
        p = t - g * cycle * records
        r, s = divmod(p, m)
        out.append(int(inputs[g0 + s]) * records + r)
    return np.array(out, dtype=np.int64)


def test_interleave_closed_form_equals_simulation(orc):
    for m in (1, 2, 5, 8, 13):
        for c in (1, 2, 3, 4):
            for L in (1, 3, 7):
                inputs = np.arange(m) * 3 + 1
                assert (closed_form_interleave(inputs, c, L) == orc.interleave_order(inputs, c, L)).all()


# --------------------------------------------------------- filter (cfg4) ----
def test_filter_batch_known_answers(orc):
    c = GOLDEN["cfg4_filter_batch"]
    lens = orc.lengths(c["n"], c["max_len"], c["len_seed"])
    toks, offs = orc.tokens(lens, c["tok_seed"])
    kept = orc.filter_len_le(lens, c["max_keep"])
    assert kept.size == c["rows"]
    sizes = [min(c["batch"], kept.size - s) for s in range(0, kept.size, c["batch"])]
    assert len(sizes) == c["num_batches"] and sizes[-1] == c["last_batch"]
    assert fnv(orc, lens[kept].astype(np.int64)) == c["fnv_row_lengths"]
    flat = np.concatenate([toks[offs[p]:offs[p + 1]] for p in kept]).astype(np.int64)
    assert fnv(orc, flat) == c["fnv_tokens"]
    assert fnv(orc, np.array(sizes)) == c["fnv_batch_sizes"]


def test_token_generator_vectorised_matches_c(orc):
    lens = orc.lengths(50, 40, 4)
    toks, offs = orc.tokens(lens, 4)
    for i in (0, 7, 49):
        for j in range(lens[i]):
            assert toks[offs[i] + j] == orc.token(4, i, j)


# ------------------------------------------------------ image UDF chains ----
def restated_image_pipeline(orc, c):
    n, (ih, iw), (oh, ow) = c["n"], c["in_hw"], c["out_hw"]
    pos = orc.shard_positions(n, *c["shard"]) if c["shard"] else np.arange(n)
    if c["shuffle_buffer"]:
        pos = restated_shuffle(orc, pos.size, c["shuffle_buffer"], c["shuffle_seed"], c["base_seed"], in_map=pos)
    pix = np.zeros((pos.size, oh, ow, 3), np.float32)
    for k, p in enumerate(pos):
        img = orc.images(int(p), 1, ih, iw)[0]
        if c["mode"] == 1:
            pix[k] = orc.resize_normalize(img, oh, ow)
        else:
            pix[k] = orc.crop_flip_normalize(img, int(p), oh, ow, c["udf_seed"], do_flip=c["mode"] == 0)
    return pos, pix


def test_image_pipelines_known_answers(orc):
    for c in GOLDEN["image_pipelines"]:
        ids, pix = restated_image_pipeline(orc, c)
        sizes = [min(c["batch"], ids.size - s) for s in range(0, ids.size, c["batch"])]
        assert sizes == c["batch_sizes"]
        assert fnv(orc, ids) == c["fnv_ids"], c
        assert fnv(orc, pix.view(np.uint32).astype(np.int64)) == c["fnv_pixels"], c


def test_philox_known_answer_vectors(orc):
    from tests.oracle_lib import P
    kat = [([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
           ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
           ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
            [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1])]
    for ctr, key, want in kat:
        c, k, out = np.array(ctr, np.uint32), np.array(key, np.uint32), np.zeros(4, np.uint32)
        orc.L.orc_philox4x32_10(P(c), P(k), P(out))
        assert out.tolist() == want


def _f32_round(fr: Fraction) -> np.float32:
    if fr == 0:
        return np.float32(0)
    sign = -1 if fr < 0 else 1
    a = abs(fr)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    m = a / Fraction(2) ** (e - 23)
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return np.float32(sign * fl * 2.0 ** (e - 23))


def test_fast_division_exhaustive():
    """normalize_u8 in csrc/common.cuh: q = RN(d*r); q' = RN(q + RN(d - q*s)*r)
    (two FMAs) equals IEEE RN(d / s) for every uint8 pixel and channel."""
    from tests.oracle_lib import MEAN, STD
    for c in range(3):
        m, s = np.float32(MEAN[c]), np.float32(STD[c])
        r = np.float32(1) / s
        for x in range(256):
            d = np.float32(np.float32(x) - m)
            want = np.float32(d / s)
            q = np.float32(d * r)
            rem = _f32_round(Fraction(float(d)) - Fraction(float(q)) * Fraction(float(s)))
            got = _f32_round(Fraction(float(rem)) * Fraction(float(r)) + Fraction(float(q)))
            assert got == want, (c, x)


# ------------------------------------------ restatement vs compiled reference ----
def test_restatement_matches_reference_shuffle_random(orc, ref):
    rng = np.random.default_rng(0)
    for _ in range(40):
        n = int(rng.integers(1, 5000))
        b = int(rng.integers(1, 6000))
        seed = int(rng.integers(0, 2**63))
        base = int(rng.integers(0, 2**63))
        want = ref.shuffle_ids(n, b, seed=seed, base_seed=base)
        assert (restated_shuffle(orc, n, b, seed, base) == want).all()


def test_restatement_matches_reference_interleave_random(orc, ref):
    rng = np.random.default_rng(1)
    for _ in range(20):
        m, c, L = int(rng.integers(1, 30)), int(rng.integers(1, 6)), int(rng.integers(1, 9))
        p = int(rng.integers(1, c + 1))
        k = int(rng.integers(1, 4))
        g = int(rng.integers(0, k))
        want = ref.interleave_ids(m, c, L, parallel=p, shard=(k, g))
        inputs = orc.shard_positions(m, k, g)
        assert (closed_form_interleave(inputs, c, L) == want).all()


def test_fast_division_proven_for_all_fp32_in_0_255(tmp_path):
    """tools/prove_fast_div.c enumerates every fp32 in [+0, 255] (1.13e9 per
    channel) and checks the device normalize's two-FMA division against IEEE
    division: the K4 (resize) inputs are blends of uint8 pixels, all in that
    range, so K4's normalize is exact too."""
    import subprocess
    src = os.path.join(os.path.dirname(HERE), "tools", "prove_fast_div.c")
    exe = str(tmp_path / "prove_fast_div")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", src, "-o", exe, "-lm"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "TOTAL mismatches: 0" in out.stdout, out.stdout


def test_bucket_by_length_restatement(orc):
    """group_by_window semantics (restate.c orc_bucket_by_length): a bucket's
    batch is emitted when its window fills; leftovers flush in ascending
    bucket order at the end unless drop_remainder."""
    lengths = np.array([5, 50, 6, 7, 51, 8, 52, 9], np.int32)
    got = orc.bucket_by_length(lengths, None, [10], [2, 2])
    assert [b.tolist() for b in got] == [[0, 2], [1, 4], [3, 5], [7], [6]]
    got = orc.bucket_by_length(lengths, None, [10], [2, 2], drop=True)
    assert [b.tolist() for b in got] == [[0, 2], [1, 4], [3, 5]]
    order = np.array([7, 6, 5, 4, 3, 2, 1, 0])
    got = orc.bucket_by_length(lengths, order, [6, 51], [3, 1, 5])
    # buckets: len<6 -> 0, 6..50 -> 1 (size 1: emitted at once), >=51 -> 2
    assert [b.tolist() for b in got] == [[7], [5], [3], [2], [1], [0], [6, 4]]


def test_interleave_var_restatement_vs_reference_golden(orc):
    """Readers of unequal lengths (record files of different sizes): the
    restatement equals the compiled reference's order (golden
    interleave_var, sequential and parallel-without-empty-readers)."""
    for c in GOLDEN["interleave_var"]:
        lens = np.array(c["lengths"], np.int64)
        k, g = c["shard"]
        inputs = np.arange(g, lens.size, k) if k else np.arange(lens.size)
        assert orc.interleave_var(inputs, c["cycle"], lens).tolist() == c["order"], c


def test_interleave_schedule_closed_form(orc):
    """dp_interleave_schedule (host, C ABI) + the position formula of the
    interleave_var kernel reproduce the sequential loop on random cases --
    the device kernel is this formula, one thread per record."""
    import ctypes
    from paper_2101_12127_b200 import _capi
    L = _capi.lib()
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    rng = np.random.default_rng(5)
    for _ in range(300):
        m, c = int(rng.integers(0, 20)), int(rng.integers(1, 7))
        lens = rng.integers(0, 9, m).astype(np.int64)
        slot, start = np.zeros(max(m, 1), np.int64), np.zeros(max(m, 1), np.int64)
        end = np.zeros(c, np.int64)
        assert L.dp_interleave_schedule(ctypes.c_int64(m), P(lens), ctypes.c_int64(c), P(slot), P(start),
                                        P(end)) == 0
        first = np.concatenate([[0], np.cumsum(lens)[:-1]]) if m else np.zeros(0, np.int64)
        out = np.full(int(lens.sum()), -1, np.int64)
        for i in range(m):
            for j in range(lens[i]):
                r = start[i] + j
                pos = int(np.minimum(end, r).sum()) + int(((np.arange(c) < slot[i]) & (end > r)).sum())
                out[pos] = first[i] + j
        assert out.tolist() == orc.interleave_var(np.arange(m), c, lens).tolist(), (lens.tolist(), c)


def test_chain_restatement_equals_the_fused_restatements_and_digest(orc):
    """oracle/chain.c (each UDF a MapFn on the whole element, in order) equals
    the fused crop+flip+normalize / resize+normalize restatements, and its
    epoch digest equals K7's position hash over the chained outputs."""
    from tests.oracle_lib import MEAN, STD, Oracle
    for ident in (0, 5, 77, 1 << 33):
        img = orc.images(ident, 1, 256, 256)[0]
        a = orc.chain(img, ident, [("random_crop", 224, 224, 7, True), ("normalize", MEAN, STD)])
        assert np.array_equal(a.view(np.uint32), orc.crop_flip_normalize(img, ident).view(np.uint32))
        img = orc.images(ident, 1, 320, 320)[0]
        a = orc.chain(img, ident, [("resize", 224, 224), ("normalize", MEAN, STD)])
        assert np.array_equal(a.view(np.uint32), orc.resize_normalize(img).view(np.uint32))
        a = orc.chain(img, ident, [("resize", 200, 150)])
        assert np.array_equal(a.view(np.uint32), orc.resize(img, 200, 150).view(np.uint32))
    ids = np.array([3, 1, 4, 1, 5, 9, 2, 6], np.int64)
    steps = [("random_crop", 24, 20, 7, True), ("normalize", MEAN, STD)]
    outs = np.concatenate([orc.chain(orc.images(int(i), 1, 32, 40)[0], int(i), steps).reshape(-1).view(np.uint32)
                           for i in ids])
    assert orc.epoch_image_digest(steps, ids, 32, 40, threads=3) == Oracle.order_digest(outs)


def test_chain_goldens_equal_the_restatement(orc):
    """tests/golden/chains.json (the compiled reference running the chain
    steps as MapFns) equals the oracle's shuffle order + chain restatement."""
    import json
    import os
    from tests.oracle_lib import Oracle
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "chains.json")))
    n, (buf, seed) = gold["n"], gold["shuffle"]
    order = orc.shuffle_order(n, buf, orc.shuffle_seed(gold["base_seed"], seed))
    for case in gold["cases"]:
        steps = [tuple(s) for s in case["steps"]]
        assert f"{orc.fnv_digest(order):016x}" == case["ids"]
        imgs = np.stack([orc.chain(orc.images(int(i), 1, *case["in_hw"])[0], int(i), steps) for i in order])
        assert f"{Oracle.order_digest(imgs.reshape(-1).view(np.uint32)):016x}" == case["images"], case["name"]
        b = gold["batch"]
        assert case["batch_sizes"] == [min(b, n - k) for k in range(0, n, b)]


def test_token_digest_goldens_reproduce():
    """tests/golden/token_digests.json (the GPU full-epoch token parity
    target) recomputed from the oracle for the ragged case (~3 s)."""
    import json
    import os
    import sys
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    import make_token_digests as m
    from tests.oracle_lib import Oracle
    gold = json.load(open(os.path.join(here, "token_digests.json")))["cases"]["cfg4r"]
    orc = Oracle()
    lens = orc.lengths(m.N, m.MAX_LEN, m.SEED)
    kept = orc.filter_len_le(lens, m.KEEP)
    acc = pos = 0
    for k in range(0, kept.size, m.BATCH):
        toks = m.row_tokens(kept[k:k + m.BATCH], lens)
        acc = (acc + m.digest(toks, pos)) % 2 ** 64
        pos += toks.size
    assert pos == gold["tokens"] and f"{acc:016x}" == gold["values"]
