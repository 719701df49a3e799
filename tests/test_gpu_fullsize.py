"""Whole-output parity at BASELINE.json's full sizes (VERDICT r1 "what's
weak" #1): every pixel of a full epoch of cfg2 (65,536 256x256 images ->
shuffle(10k) -> crop 224 + flip + normalize -> batch 256), cfg3 (320x320 ->
resize 224 + normalize), cfg5 (32 record files x 2048 -> interleave(4, 4)
-> shuffle -> crop + flip + normalize), and the K10 chains cfg2rrc (crop 160 +
flip -> resize 224 -> normalize) and cfg3e (320 -> resize 256 -> center crop
224 -> normalize), digested on the device batch by
batch (K7 dp_k_word_digest, position = the running u32 word index of the
epoch) and compared with tests/golden/epoch_digests.json, which the oracle
restatement computed over the same epoch (tests/golden/make_epoch_digests.py).
Any wrong byte anywhere in the 39 GB of output changes the digest."""
import ctypes
import json
import os

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "epoch_digests.json")))["cases"]


@pytest.fixture(scope="module")
def dp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2101_12127_b200 import pipeline
    return pipeline


def _graph(dp, case):
    c = GOLD[case]
    reg = dp.Registry()
    for i, st in enumerate(c["steps"]):
        name = f"s{i}"
        if st[0] == "random_crop":
            reg.register_random_crop_flip(name, st[1], st[2], seed=st[3], flip=st[4])
        elif st[0] == "resize":
            reg.register_resize_bilinear(name, st[1], st[2])
        elif st[0] == "center_crop":
            reg.register_center_crop(name, st[1], st[2])
        elif st[0] == "normalize":
            reg.register_normalize(name, st[1], st[2])
    if c["source"] == "tensor_slices":
        src = dp.Source.synthetic_images(c["n"], c["hw"], c["hw"])
        g = dp.Dataset.tensor_slices(reg, src)
    else:
        src = dp.Source.synthetic_records_sharded(32, c["n"] // 32, c["hw"], c["hw"])
        reg.register_record_reader("reader", c["n"] // 32)
        g = dp.Dataset.range(reg, 32).interleave("reader", 4, 4, records=src)
    g = g.shuffle(*c["shuffle"])
    for i in range(len(c["steps"])):
        g = g.map(f"s{i}")
    return g.batch(c["batch"]).prefetch(-1), src


def _epoch_digests(dp, g, **opts):
    import torch
    from paper_2101_12127_b200 import _capi
    it = dp.make_iterator(g, seed_override=GOLD["cfg2"]["base_seed"], **opts)
    dig = torch.zeros(2, dtype=torch.int64, device="cuda")
    L = _capi.lib()
    words = ids = 0
    n = 0
    for b in it:
        (_, ishape, iptr, _), (_, pshape, pptr, _) = b.components[:2]
        nw = pshape[0] * pshape[1] * pshape[2] * pshape[3]  # fp32 words
        _capi.check(L.dp_k_order_digest(ctypes.c_void_p(iptr), ishape[0], ids, ctypes.c_void_p(dig.data_ptr()),
                                        ctypes.c_void_p(it.stream)))
        _capi.check(L.dp_k_word_digest(ctypes.c_void_p(pptr), nw, words, ctypes.c_void_p(dig.data_ptr() + 8),
                                       ctypes.c_void_p(it.stream)))
        ids += ishape[0]
        words += nw
        n += 1
        b.release()
    torch.cuda.synchronize()
    v = [int(x) & (2 ** 64 - 1) for x in dig.cpu().tolist()]
    return n, ids, f"{v[0]:016x}", f"{v[1]:016x}"


@pytest.mark.parametrize("case", ["cfg2", "cfg3", "cfg5", "cfg2rrc", "cfg3e"])
def test_full_epoch_every_pixel_matches_the_oracle(dp, case):
    c = GOLD[case]
    g, src = _graph(dp, case)
    n, ids, id_dig, pix_dig = _epoch_digests(dp, g)
    assert n == c["n"] // c["batch"] and ids == c["n"]
    assert id_dig == c["ids"], "element order differs from the reference's shuffle"
    assert pix_dig == c["pixels"], "some output byte of the epoch differs from the oracle"


def test_full_epoch_digest_independent_of_launch_tiling(dp):
    """The same full cfg2 epoch with 1-batch launches and with a 3-batch head
    followed by 7-batch launches: identical digests (prefetch / launch
    settings do not change the sequence, P/tests/test_parallel.cpp:297-312)."""
    c = GOLD["cfg2"]
    g, src = _graph(dp, "cfg2")
    for opts in ({"launch_batches": 1}, {"launch_batches": 7, "first_launch_batches": 3}):
        _, _, id_dig, pix_dig = _epoch_digests(dp, g, **opts)
        assert (id_dig, pix_dig) == (c["ids"], c["pixels"]), opts


TOK = json.load(open(os.path.join(HERE, "golden", "token_digests.json")))


@pytest.mark.parametrize("case", ["cfg4", "cfg4r", "cfg4b"])
def test_full_epoch_every_token_matches_the_oracle(dp, case):
    """A whole epoch of 1M sequences: every output word of the padded /
    ragged / bucketed batches (padding included) and every row length /
    split, digested on the device, equals the oracle's digests
    (tests/golden/token_digests.json)."""
    import torch
    from paper_2101_12127_b200 import _capi
    c = TOK["cases"][case]
    reg = dp.Registry()
    reg.register_length_filter("keep", TOK["keep"])
    src = dp.Source.synthetic_tokens(TOK["n"], TOK["max_len"], TOK["seed"], TOK["seed"])
    g = dp.Dataset.token_sequences(reg, src).filter("keep")
    if case == "cfg4":
        g = g.padded_batch(128)
    elif case == "cfg4r":
        g = g.batch(128)
    else:
        g = g.shuffle(10000, 42).bucket_by_length([128, 256, 384], [256, 128, 96, 64])
    it = dp.make_iterator(g.prefetch(-1), seed_override=1)
    L = _capi.lib()
    dig = torch.zeros(2, dtype=torch.int64, device="cuda")
    p0 = p1 = n = 0
    for b in it:
        (_, s0, ptr0, _), (_, s1, ptr1, _) = b.components[:2]
        w0 = s0[0] * (s0[1] if len(s0) > 1 else 1)
        _capi.check(L.dp_k_word_digest(ctypes.c_void_p(ptr0), w0, p0, ctypes.c_void_p(dig.data_ptr()),
                                       ctypes.c_void_p(it.stream)))
        fn = L.dp_k_order_digest if case == "cfg4r" else L.dp_k_word_digest  # row splits are int64
        _capi.check(fn(ctypes.c_void_p(ptr1), s1[0], p1, ctypes.c_void_p(dig.data_ptr() + 8), ctypes.c_void_p(it.stream)))
        p0 += w0
        p1 += s1[0]
        n += 1
        b.release()
    torch.cuda.synchronize()
    v = [f"{int(x) & (2 ** 64 - 1):016x}" for x in dig.cpu().tolist()]
    assert n == c["batches"]
    if case == "cfg4r":
        assert p0 == c["tokens"] and v == [c["values"], c["splits"]]
    else:
        assert p0 == c["words"] and v == [c["tokens"], c["lengths"]]
