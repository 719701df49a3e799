"""End-to-end parity of the operator API on the GPU, through the C ABI
(include/dpcuda_pipeline.h): graphs built with the ops:: builders, optimized,
iterated with GetNext, compared with the oracle restatement and with the
golden vectors generated from the compiled reference.

Mirrors the reference's suites: P/tests/test_iterator.cpp (sticky EOF,
partial batch, shuffle reproducibility / multiset / identity, shard
partition), P/tests/test_optimizer.cpp (fusion preserves the sequence,
shuffle+repeat), P/tests/acceptance/acceptance_main.cpp #9 (determinism).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))


@pytest.fixture(scope="module")
def dp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2101_12127_b200 import pipeline
    return pipeline


def fnv(orc, v):
    return f"{orc.fnv_digest(np.asarray(v, dtype=np.int64)):016x}"


def drain(it, comps=(0,)):
    """All batches, copied to host (each Batch released right after)."""
    out = []
    while (b := it.get_next()) is not None:
        out.append([b.numpy(c) for c in comps])
        b.release()
    return out


def image_registry(dp, mode, crop=(224, 224), seed=7):
    reg = dp.Registry()
    if mode == 1:
        reg.register_resize_bilinear("resize", *crop)
    else:
        reg.register_random_crop_flip("crop", crop[0], crop[1], seed=seed, flip=(mode == 0))
    reg.register_normalize("norm")
    return reg


# ------------------------------------------------------------------ cfg1 ----
def test_cfg1_through_the_operator_api(dp, orc):
    reg = dp.Registry()
    reg.register_affine("affine(3,1)", 3, 1)
    g, _ = dp.Dataset.range(reg, 1_000_000).map("affine(3,1)").batch(1024).optimize()
    assert g.root_kind == "map_and_batch"
    it = dp.make_iterator(g, seed_override=1)
    batches = [b[0] for b in drain(it)]
    want = GOLDEN["cfg1_range_map_batch_1024"]["1000000"]
    assert len(batches) == want["num_batches"] == 977 and batches[-1].size == want["last_batch"] == 576
    vals = np.concatenate(batches)
    assert int(vals.sum()) == want["sum"] and fnv(orc, vals) == want["fnv"]
    assert it.get_next() is None and it.get_next() is None  # sticky EOF
    assert it.kernel_launches >= 1


def test_from_memory_batch_partial_and_drop(dp):
    reg = dp.Registry()
    src = dp.Dataset.from_memory(reg, [1, 2, 3, 4, 5])
    got = [b[0].tolist() for b in drain(dp.make_iterator(src.batch(2)))]
    assert got == [[1, 2], [3, 4], [5]]
    got = [b[0].tolist() for b in drain(dp.make_iterator(src.batch(2, drop_remainder=True)))]
    assert got == [[1, 2], [3, 4]]


def test_unfused_map_batch_equals_fused(dp):
    reg = dp.Registry()
    reg.register_affine("times2", 2, 0)
    g = dp.Dataset.from_memory(reg, list(range(1, 8))).map("times2").batch(3)
    fused, _ = g.optimize()
    assert fused.root_kind == "map_and_batch" and g.root_kind == "batch"
    a = [b[0].tolist() for b in drain(dp.make_iterator(g))]
    b = [b[0].tolist() for b in drain(dp.make_iterator(fused))]
    assert a == b == [[2, 4, 6], [8, 10, 12], [14]]


# ------------------------------------------------------------- shuffle ----
def shuffle_ids(dp, n, buffer, seed, base_seed, shard=None, repeat=None, optimize=False):
    reg = dp.Registry()
    g = dp.Dataset.range(reg, n)
    if shard:
        g = g.shard(*shard)
    g = g.shuffle(buffer, seed)
    if repeat:
        g = g.repeat(repeat)
    g = g.batch(4096)
    if optimize:
        g, _ = g.optimize()
    return np.concatenate([b[0] for b in drain(dp.make_iterator(g, seed_override=base_seed))])


def test_value_filters_equal_the_reference(dp, orc):
    """keep_even / keep_odd after an affine map, unoptimized and optimized
    (map_filter_fusion), with a shuffle after the filter: the emitted values
    equal the compiled reference's (golden value_filters)."""
    for c in GOLDEN["value_filters"]:
        reg = dp.Registry()
        reg.register_standard_predicates()
        f = reg.register_affine(f"affine({c['a']},{c['b']})", c["a"], c["b"])
        g = dp.Dataset.from_memory(reg, range(c["n"])).map(f).filter("keep_odd" if c["odd"] else "keep_even")
        if c["shuffle"]:
            g = g.shuffle(c["shuffle"], 42)
        g = g.batch(64)
        if c["optimize"]:
            g = g.optimize()[0]
        vals = np.concatenate([b[0] for b in drain(dp.make_iterator(g, seed_override=1))])
        assert vals.size == c["count"] and vals[:6].tolist() == c["first"] and fnv(orc, vals) == c["fnv"], c
    # range source, a conjunction of terms, a filter between two maps
    reg = dp.Registry()
    reg.register_affine("x2", 2, 0)
    reg.register_affine("p5", 1, 5)
    reg.register_value_filter("window", [("ge", 100), ("lt", 900), ("mod_ne", 3, 1)])
    g = dp.Dataset.range(reg, 1000).map("x2").filter("window").map("p5").batch(50)
    got = np.concatenate([b[0] for b in drain(dp.make_iterator(g, seed_override=1))])
    x = np.arange(1000) * 2
    want = x[(x >= 100) & (x < 900) & (np.fmod(x, 3) != 1)] + 5
    assert got.tolist() == want.tolist()
    with pytest.raises(dp.DpError):  # a value predicate on images
        reg2 = image_registry(dp, 0, crop=(32, 32))
        reg2.register_standard_predicates()
        src = dp.Source.synthetic_images(10, 48, 48)
        dp.make_iterator(dp.Dataset.tensor_slices(reg2, src).filter("keep_even").map("crop").map("norm").batch(4))


def test_unbatched_pipelines(dp, orc):
    """No batch stage: GetNext delivers single elements, as MapIterator /
    ShuffleIterator roots do (int64 values on the host; images as (id,
    device tensor[h, w, 3]))."""
    reg = image_registry(dp, 0, crop=(32, 32))
    reg.register_affine("aff", 3, 1)
    reg.register_standard_predicates()

    def elems(g, comps=(0,), **kw):
        it = dp.make_iterator(g, seed_override=1, **kw)
        out = []
        while (b := it.get_next()) is not None:
            out.append([b.numpy(c) for c in comps])
            b.release()
        return out

    got = [int(e[0]) for e in elems(dp.Dataset.range(reg, 10000).map("aff"))]
    assert got == (np.arange(10000) * 3 + 1).tolist()
    got = [int(e[0]) for e in elems(dp.Dataset.from_memory(reg, np.arange(5000) * 7).shuffle(300, 42).map("aff"))]
    order = orc.shuffle_order(5000, 300, orc.shuffle_seed(1, 42))
    assert got == (order * 7 * 3 + 1).tolist()
    got = [int(e[0]) for e in elems(dp.Dataset.range(reg, 3000).map("aff").filter("keep_even").repeat(2))]
    x = np.arange(3000) * 3 + 1
    assert got == x[x % 2 == 0].tolist() * 2
    # images: single (id, image) elements equal the rows of the batched pipeline
    src = dp.Source.synthetic_images(300, 48, 48)
    base = dp.Dataset.tensor_slices(reg, src).shuffle(100, 5).map("crop").map("norm")
    single = elems(base, comps=(0, 1))
    batched = drain(dp.make_iterator(base.batch(64), seed_override=1), comps=(0, 1))
    ids = np.concatenate([b[0] for b in batched])
    pix = np.concatenate([b[1] for b in batched])
    assert [int(e[0]) for e in single] == ids.tolist()
    assert all(np.array_equal(e[1], pix[r]) for r, e in enumerate(single))
    # single token sequences (device views into internal ragged batches)
    reg.register_length_filter("short", 40)
    tsrc = dp.Source.synthetic_tokens(2000, 80, 5, 5)
    seqs = elems(dp.Dataset.token_sequences(reg, tsrc).filter("short").shuffle(300, 9))
    lens_all = orc.lengths(2000, 80, 5)
    toks, offs = orc.tokens(lens_all, 5)
    kept = orc.filter_len_le(lens_all, 40)
    order = kept[orc.shuffle_order(kept.size, 300, orc.shuffle_seed(1, 9))]
    assert len(seqs) == order.size
    assert all(np.array_equal(e[0], toks[offs[p]:offs[p + 1]]) for e, p in zip(seqs, order))
    # checkpoint in the middle of an unbatched, repeated pipeline
    g = dp.Dataset.range(reg, 5000).shuffle(700, 2).map("aff").repeat(3)
    full = [int(e[0]) for e in elems(g)]
    it = dp.make_iterator(g, seed_override=1)
    for _ in range(7777):
        it.get_next().release()
    rest = []
    r_it = dp.restore(g, it.save())
    while (b := r_it.get_next()) is not None:
        rest.append(int(b.numpy(0)))
        b.release()
    assert rest == full[7777:]


def test_pipeline_spec_runs_like_the_builders(dp, tmp_path):
    """A pipeline description (the reference's text format with device UDFs)
    iterates exactly like the ops:: graph; tools/dpbench.py runs it."""
    spec = """
        source images count=600 h=64 w=64 seed=0x5EED
        shuffle buffer=200 seed=42
        map crop h=48 w=48 seed=7 flip=true
        map normalize
        batch size=50
        prefetch buffer=AUTO
        epochs 2
    """
    reg = dp.Registry()
    g, info = dp.Dataset.from_spec(reg, spec)
    reg2 = image_registry(dp, 0, crop=(48, 48))
    want = dp.Dataset.tensor_slices(reg2, dp.Source.synthetic_images(600, 64, 64)).shuffle(200, 42).map("crop") \
        .map("norm").batch(50).prefetch(-1)
    a = drain(dp.make_iterator(g.optimize()[0], seed_override=3), comps=(0, 1))
    b = drain(dp.make_iterator(want.optimize()[0], seed_override=3), comps=(0, 1))
    assert len(a) == len(b) == 12
    assert all(np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1]) for x, y in zip(a, b))
    import subprocess
    import sys
    path = tmp_path / "p.txt"
    path.write_text(spec)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "dpbench.py"), str(path)],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "epoch 2: 600 elements" in out.stdout and "median epoch" in out.stdout


def test_shuffle_order_matches_reference(dp, orc):
    for c in GOLDEN["shuffle"]:
        got = shuffle_ids(dp, c["n"], c["buffer"], c["seed"], c["base_seed"])
        assert got[:8].tolist() == c["first"] and fnv(orc, got) == c["fnv"], c


def test_shuffle_properties(dp):
    assert shuffle_ids(dp, 5, 1, 42, 1).tolist() == [0, 1, 2, 3, 4]  # identity at buffer 1
    a = shuffle_ids(dp, 5000, 64, 7, 1)
    assert (a == shuffle_ids(dp, 5000, 64, 7, 1)).all()  # reproducible
    assert (a != shuffle_ids(dp, 5000, 64, 7, 2)).any()  # base seed matters
    assert sorted(a.tolist()) == list(range(5000))  # multiset


def test_shuffle_repeat_fused_and_unfused(dp, orc):
    for c in GOLDEN["shuffle_repeat"]:
        got = shuffle_ids(dp, c["n"], c["buffer"], c["seed"], c["base_seed"], repeat=c["epochs"],
                          optimize=c["optimize"])
        assert got.size == c["n"] * c["epochs"] and fnv(orc, got) == c["fnv"], c


def test_shard_then_shuffle(dp, orc):
    for c in GOLDEN["shard_shuffle"]:
        got = shuffle_ids(dp, c["n"], c["buffer"], c["seed"], c["base_seed"], shard=c["shard"])
        assert got.size == c["count"] and fnv(orc, got) == c["fnv"], c


def test_shard_partitions_the_input(dp):
    for k in (1, 2, 3, 8):
        seen = []
        for i in range(k):
            reg = dp.Registry()
            g = dp.Dataset.range(reg, 1001).shard(k, i).batch(100)
            part = np.concatenate([b[0] for b in drain(dp.make_iterator(g))])
            assert (part % k == i).all()
            seen.append(part)
        assert sorted(np.concatenate(seen).tolist()) == list(range(1001))


# -------------------------------------------------------- image configs ----
def test_golden_image_pipelines_through_the_operator_api(dp, orc):
    for c in GOLDEN["image_pipelines"]:
        reg = image_registry(dp, c["mode"])
        src = dp.Source.synthetic_images(c["n"], *c["in_hw"])
        g = dp.Dataset.tensor_slices(reg, src)
        if c["shard"]:
            g = g.shard(*c["shard"])
        if c["shuffle_buffer"]:
            g = g.shuffle(c["shuffle_buffer"], c["shuffle_seed"])
        first = "resize" if c["mode"] == 1 else "crop"
        g = g.map(first, 8).map("norm", 8).batch(c["batch"]).prefetch(-1)
        g, report = g.optimize()
        assert "map_map_fusion" in report and "map_batch_fusion" in report
        batches = drain(dp.make_iterator(g, seed_override=c["base_seed"]), comps=(0, 1))
        assert [b[0].size for b in batches] == c["batch_sizes"]
        ids = np.concatenate([b[0] for b in batches])
        pix = np.concatenate([b[1] for b in batches])
        assert fnv(orc, ids) == c["fnv_ids"]
        assert fnv(orc, pix.view(np.uint32).astype(np.int64)) == c["fnv_pixels"], c


def test_cfg2_shape_value_parity_20k(dp, orc):
    """N = 20,000 >= 2 x buffer, so fill and drain phases both run."""
    n, buf, b = 20_000, 10_000, 256
    reg = image_registry(dp, 0)
    src = dp.Source.synthetic_images(n, 256, 256)
    g, _ = (dp.Dataset.tensor_slices(reg, src).shuffle(buf, 42).map("crop").map("norm").batch(b).prefetch(4)
            .optimize())
    it = dp.make_iterator(g, seed_override=1)
    order = orc.shuffle_order(n, buf, orc.shuffle_seed(1, 42))
    rng = np.random.default_rng(0)
    check = set(rng.choice((n + b - 1) // b, 12, replace=False).tolist()) | {0, (n + b - 1) // b - 1}
    k = 0
    for j, bt in enumerate(it):
        ids = bt.numpy(0)
        assert (ids == order[k:k + ids.size]).all()
        if j in check:
            pix = bt.numpy(1)
            for r in rng.choice(ids.size, 3, replace=False):
                img = orc.images(int(ids[r]), 1, 256, 256)[0]
                want = orc.crop_flip_normalize(img, int(ids[r]))
                assert np.array_equal(pix[r].view(np.uint32), want.view(np.uint32))
        k += ids.size
        bt.release()
    assert k == n


@pytest.mark.parametrize("mode,hw", [(0, 256), (1, 320)])
def test_full_size_image_epoch(dp, orc, mode, hw):
    """cfg2 / cfg3 at BASELINE.json's full size (65,536 images of 256x256 /
    320x320 resident in HBM, shuffle(10k, 42), batch 256): the epoch's ids are
    exactly the reference's shuffle order (so a permutation of the dataset)
    and sampled images of every 16th batch equal the oracle bit for bit."""
    n, buf, b = 65536, 10_000, 256
    reg = image_registry(dp, mode)
    src = dp.Source.synthetic_images(n, hw, hw)
    op = "resize" if mode == 1 else "crop"
    g, _ = dp.Dataset.tensor_slices(reg, src).shuffle(buf, 42).map(op).map("norm").batch(b).prefetch(-1).optimize()
    order = orc.shuffle_order(n, buf, orc.shuffle_seed(1, 42))
    assert np.array_equal(np.sort(order), np.arange(n))
    it = dp.make_iterator(g, seed_override=1)
    rng = np.random.default_rng(mode)
    k = 0
    for j, bt in enumerate(it):
        ids = bt.numpy(0)
        assert np.array_equal(ids, order[k:k + ids.size])
        if j % 16 == 0:
            pix = bt.numpy(1)
            for r in rng.choice(ids.size, 2, replace=False):
                img = orc.images(int(ids[r]), 1, hw, hw)[0]
                want = orc.resize_normalize(img) if mode == 1 else orc.crop_flip_normalize(img, int(ids[r]))
                assert np.array_equal(pix[r].view(np.uint32), want.view(np.uint32))
        k += ids.size
        bt.release()
    assert k == n
    del it, g, src


def test_consumer_may_hold_batches(dp):
    """Holding every Element (the reference returns owned copies) grows the
    slot ring instead of overwriting held batches."""
    reg = image_registry(dp, 0, crop=(32, 32))
    src = dp.Source.synthetic_images(300, 64, 64)
    g, _ = dp.Dataset.tensor_slices(reg, src).map("crop").map("norm").batch(16).optimize()
    it = dp.make_iterator(g, seed_override=1)
    held = list(it)
    assert len(held) == 19
    ids = np.concatenate([h.numpy(0) for h in held])
    assert ids.tolist() == list(range(300))


@pytest.mark.parametrize("launch_batches", [1, 3, 4])
def test_group_lease_keeps_held_batches_intact(dp, launch_batches):
    """One lease per launch group: a batch held anywhere in a group (first,
    middle, last) keeps the whole group's slot from being rewritten while
    the iterator runs on through later groups and a second epoch; the other
    batches are dropped as they come, so the rest of the ring is reused."""
    reg = image_registry(dp, 0, crop=(24, 24))
    src = dp.Source.synthetic_images(640, 32, 32)
    g, _ = dp.Dataset.tensor_slices(reg, src).shuffle(200, 9).map("crop").map("norm").batch(16).repeat(2).prefetch(2).optimize()
    ref = drain(dp.make_iterator(g, seed_override=3, launch_batches=launch_batches), comps=(0, 1))
    assert len(ref) == 80
    it = dp.make_iterator(g, seed_override=3, launch_batches=launch_batches)
    held, k = {}, 0
    while (b := it.get_next()) is not None:
        if k % 7 in (0, 3) or k == 39:
            held[k] = b
        else:
            np.testing.assert_array_equal(b.numpy(1), ref[k][1])
            b.release()
        k += 1
    assert k == 80
    for k, b in held.items():  # read only now, after 80 batches went past
        np.testing.assert_array_equal(b.numpy(0), ref[k][0])
        np.testing.assert_array_equal(b.numpy(1), ref[k][1])
        b.release()


def test_concurrent_get_next_callers(dp):
    """PipelineIterator::GetNext is thread-safe for concurrent callers
    (runtime.hpp:53-55): 4 threads draining one iterator get every batch
    exactly once, each batch intact; two iterators run side by side."""
    import threading
    reg = image_registry(dp, 0, crop=(32, 32))
    src = dp.Source.synthetic_images(2000, 48, 48)
    g, _ = dp.Dataset.tensor_slices(reg, src).shuffle(500, 3).map("crop").map("norm").batch(20).optimize()
    ref = [b[0] for b in drain(dp.make_iterator(g, seed_override=5))]
    ref_pix = {tuple(b[0].tolist()): b[1] for b in drain(dp.make_iterator(g, seed_override=5), comps=(0, 1))}
    it = dp.make_iterator(g, seed_override=5)
    got, errors, lock = [], [], threading.Lock()

    def worker():
        try:
            while (b := it.get_next()) is not None:
                ids, pix = b.numpy(0), b.numpy(1)
                b.release()
                with lock:
                    got.append((ids, pix))
        except Exception as ex:  # surfaced below
            errors.append(ex)

    threads = [threading.Thread(target=worker) for _ in range(4)]
    other = dp.make_iterator(g, seed_override=5)
    for t in threads:
        t.start()
    side = [b[0] for b in drain(other)]  # a second iterator meanwhile
    for t in threads:
        t.join()
    assert not errors
    assert len(got) == len(ref) == 100
    assert sorted(tuple(x.tolist()) for x, _ in got) == sorted(tuple(x.tolist()) for x in ref)
    for ids, pix in got:
        assert np.array_equal(pix, ref_pix[tuple(ids.tolist())])
    assert all(np.array_equal(a, b) for a, b in zip(side, ref))


def test_resize_alone_and_normalize_alone(dp, orc):
    """resize without normalize (fp32) and normalize without a crop: the
    restatement's rounded ops, bit for bit."""
    imgs = orc.images(0, 40, 50, 70)
    src = dp.Source.images_from_host(imgs)
    reg = dp.Registry()
    reg.register_resize_bilinear("rs", 33, 41)
    reg.register_normalize("norm")
    out = drain(dp.make_iterator(dp.Dataset.tensor_slices(reg, src).shuffle(16, 1).map("rs").batch(8),
                                 seed_override=2), comps=(0, 1))
    for b in out:
        for r, i in enumerate(b[0]):
            assert np.array_equal(b[1][r].view(np.uint32), orc.resize(imgs[i], 33, 41).view(np.uint32))
    out = drain(dp.make_iterator(dp.Dataset.tensor_slices(reg, src).map("norm").batch(16), seed_override=2),
                comps=(0, 1))
    mean = np.array([123.675, 116.28, 103.53], np.float32)
    std = np.array([58.395, 57.12, 57.375], np.float32)
    want = (imgs.astype(np.float32) - mean) / std  # IEEE fp32 subtract + divide
    got = np.concatenate([b[1] for b in out])
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_cast_u8_to_f32(dp, orc):
    """The Map library's cast (u8 -> fp32, exact): alone, after a random
    crop + flip (the cropped, flipped window as floats) and after a resize;
    also through the pipeline text format (`map cast`)."""
    imgs = orc.images(0, 24, 48, 64)
    src = dp.Source.images_from_host(imgs)
    reg = dp.Registry()
    reg.register_cast("cast")
    reg.register_random_crop_flip("crop", 32, 40, seed=9, flip=True)
    reg.register_resize_bilinear("rs", 30, 44)
    base = dp.Dataset.tensor_slices(reg, src).shuffle(10, 4)
    alone = drain(dp.make_iterator(base.map("cast").batch(8), seed_override=1), comps=(0, 1))
    crop = drain(dp.make_iterator(base.map("crop").map("cast").batch(8), seed_override=1), comps=(0, 1))
    rs = drain(dp.make_iterator(base.map("rs").map("cast").batch(8), seed_override=1), comps=(0, 1))
    for a, c, r in zip(alone, crop, rs):
        for k, i in enumerate(a[0]):
            assert np.array_equal(a[1][k], imgs[i].astype(np.float32))
            oy, ox, fl = orc.crop_params(9, int(i), 48, 64, 32, 40)
            win = imgs[i][oy:oy + 32, ox:ox + 40]
            assert np.array_equal(c[1][k], (win[:, ::-1] if fl else win).astype(np.float32))
            assert np.array_equal(r[1][k].view(np.uint32), orc.resize(imgs[i], 30, 44).view(np.uint32))
    g, _ = dp.Dataset.from_spec(dp.Registry(), "source images count=24 h=48 w=64\nmap cast\nbatch size=8\n")
    out = drain(dp.make_iterator(g, seed_override=1), comps=(0, 1))
    pix = orc.images(0, 24, 48, 64)
    assert all(np.array_equal(b[1][k], pix[int(i)].astype(np.float32)) for b in out for k, i in enumerate(b[0]))


def test_pinned_host_token_source_equals_device_source(dp, orc):
    """Token sequences in pinned host memory (read over PCIe by the filter,
    padded / ragged and bucket kernels) give the same batches as the same
    sequences in HBM, with host_output on and off."""
    lens = orc.lengths(3000)
    toks, _ = orc.tokens(lens)
    reg = dp.Registry()
    reg.register_length_filter("len<=512", 512)
    outs = []
    for pinned, host in ((False, False), (True, False), (True, True)):
        src = dp.Source.tokens_from_host(lens, toks, pinned=pinned)
        base = dp.Dataset.token_sequences(reg, src).filter("len<=512")
        got = []
        for g in (base.padded_batch(64), base.batch(50), base.shuffle(300, 5).bucket_by_length([200], [32, 16])):
            it = dp.make_iterator(g, seed_override=1, host_output=host)
            while (b := it.get_next()) is not None:
                if host:
                    b.wait()
                got.append([b.numpy(0), b.numpy(1)])
                b.release()
        outs.append(got)
    for other in outs[1:]:
        assert len(other) == len(outs[0])
        assert all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) for a, b in zip(outs[0], other))


def test_host_output_equals_device_output(dp):
    reg = image_registry(dp, 0, crop=(64, 64))
    src = dp.Source.synthetic_images(200, 96, 96)
    g, _ = dp.Dataset.tensor_slices(reg, src).shuffle(50, 3).map("crop").map("norm").batch(32).optimize()
    dev = drain(dp.make_iterator(g, seed_override=9), comps=(0, 1))
    host = drain(dp.make_iterator(g, seed_override=9, host_output=True), comps=(0, 1))
    assert len(dev) == len(host)
    for a, b in zip(dev, host):
        assert (a[0] == b[0]).all() and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("op", ["crop", "resize", "resize_k4", "rrc"])
def test_pinned_host_source_equals_device_source(dp, orc, op):
    """Images in pinned host memory (end-to-end runs) go through the same
    TMA kernels as HBM-resident ones (K3 crop, K10 resize / RandomResizedCrop
    chain: cp.async.bulk reads host memory over PCIe) and give the same bits,
    also with the TMA path disabled (generic kernels' 16-byte loads)."""
    imgs = orc.images(0, 64, 80, 80)
    reg = (image_registry(dp, 0, crop=(48, 48)) if op == "crop" else
           image_registry(dp, 1, crop=(60, 60)) if op == "resize_k4" else  # 4:3: K4's TMA path
           image_registry(dp, 1, crop=(56, 56)))
    reg.register_random_crop_flip("c40", 40, 40, seed=3, flip=True)
    if op == "rrc":
        imgs = orc.images(0, 64, 64, 64)
    a_src = dp.Source.images_from_host(imgs)
    b_src = dp.Source.images_pinned_host(imgs)
    out = []
    for src, tma in ((a_src, "1"), (b_src, "1"), (b_src, "0")):
        os.environ["DP_DEV_TMA_HOST"] = tma
        try:
            d = dp.Dataset.tensor_slices(reg, src).shuffle(20, 1)
            d = d.map("crop") if op == "crop" else d.map("c40").map("resize") if op == "rrc" else d.map("resize")
            g, _ = d.map("norm").batch(10).optimize()
            out.append(drain(dp.make_iterator(g, seed_override=2), comps=(0, 1)))
        finally:
            del os.environ["DP_DEV_TMA_HOST"]
    for a, b, c in zip(*out):
        assert (a[0] == b[0]).all() and np.array_equal(a[1], b[1]) and np.array_equal(a[1], c[1])


def test_from_file_records_equal_tensor_slices(dp, orc, tmp_path):
    """from_file (graph.hpp:137, FromFileIterator runtime.cpp:416-474) over
    record files holding raw HWC images, decoded on the device by decode_raw:
    the record ordinal is the element id, so the pipeline equals tensor_slices
    over the same images bit for bit."""
    imgs = orc.images(5, 90, 72, 64)
    paths = [str(tmp_path / "a.rec"), str(tmp_path / "b.rec")]
    dp.write_record_file(paths[0], [im.tobytes() for im in imgs[:37]])
    dp.write_record_file(paths[1], [im.tobytes() for im in imgs[37:]])
    out = []
    for mode in (0, 1):
        reg = image_registry(dp, mode, crop=(48, 40))
        reg.register_decode_raw("decode", 72, 64)
        a = dp.Dataset.from_file(reg, paths).map("decode")
        b = dp.Dataset.tensor_slices(reg, dp.Source.images_from_host(imgs))
        res = []
        for d in (a, b):
            op = "crop" if mode == 0 else "resize"
            g, _ = d.shuffle(30, 4).map(op).map("norm").batch(16).optimize()
            res.append(drain(dp.make_iterator(g, seed_override=6), comps=(0, 1)))
        assert len(res[0]) == len(res[1]) == 6
        for x, y in zip(*res):
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
        # a map under the shuffle commutes with it (randomness keyed by element id)
        g, _ = a.map(op).shuffle(30, 4).map("norm").batch(16).optimize()
        for x, y in zip(drain(dp.make_iterator(g, seed_override=6), comps=(0, 1)), res[1]):
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
        out.append(res[0])
    # wrong decode shape / missing decode are rejected at MakeIterator
    reg = image_registry(dp, 0, crop=(48, 40))
    reg.register_decode_raw("decode_bad", 70, 64)
    with pytest.raises(dp.DpError) as e:
        dp.make_iterator(dp.Dataset.from_file(reg, paths).map("decode_bad").map("crop").map("norm").batch(8))
    assert e.value.code == dp.ERR["MalformedInput"]
    with pytest.raises(dp.DpError):
        dp.make_iterator(dp.Dataset.from_file(reg, paths).batch(8))


# ------------------------------------------------------------------ cfg4 ----
def test_cfg4_filter_padded_batch(dp, orc):
    c = GOLDEN["cfg4_filter_batch"]
    reg = dp.Registry()
    reg.register_length_filter("len<=512", c["max_keep"])
    src = dp.Source.synthetic_tokens(c["n"], c["max_len"], c["len_seed"], c["tok_seed"])
    g = dp.Dataset.token_sequences(reg, src).filter("len<=512").padded_batch(c["batch"], padding_value=0)
    batches = drain(dp.make_iterator(g, seed_override=1), comps=(0, 1))
    sizes = [b[1].size for b in batches]
    assert len(sizes) == c["num_batches"] and sizes[-1] == c["last_batch"]
    lens = np.concatenate([b[1] for b in batches])
    toks = np.concatenate([b[0][r, :b[1][r]] for b in batches for r in range(b[1].size)])
    for b in batches:  # padding is 0 past each row's length; width = the batch's max length
        assert b[0].shape[1] == b[1].max()
        for r in range(b[1].size):
            assert (b[0][r, b[1][r]:] == 0).all()
    assert fnv(orc, lens) == c["fnv_row_lengths"] and fnv(orc, toks) == c["fnv_tokens"]
    assert fnv(orc, sizes) == c["fnv_batch_sizes"]


def test_full_size_cfg4_epoch(dp, orc):
    """cfg4 at full size (1M sequences, len U[1,1024], filter len <= 512,
    padded_batch 128): every batch's row lengths are the reference filter's
    kept sequences in order, padding is 0 to the batch max, and sampled rows
    of every 64th batch hold the oracle's tokens."""
    n, max_keep, b = 1_000_000, 512, 128
    lens = orc.lengths(n)
    kept = orc.filter_len_le(lens, max_keep)
    reg = dp.Registry()
    reg.register_length_filter("len<=512", max_keep)
    src = dp.Source.synthetic_tokens(n, 1024, 4, 4)
    g = dp.Dataset.token_sequences(reg, src).filter("len<=512").padded_batch(b)
    it = dp.make_iterator(g, seed_override=1)
    rng = np.random.default_rng(4)
    k = j = 0
    for bt in it:
        toks, got = bt.numpy(0), bt.numpy(1)
        want = lens[kept[k:k + got.size]]
        assert np.array_equal(got, want) and toks.shape == (got.size, want.max())
        if j % 64 == 0:
            assert all((toks[r, got[r]:] == 0).all() for r in range(got.size))
            for r in rng.choice(got.size, 2, replace=False):
                i = int(kept[k + r])
                assert toks[r, :got[r]].tolist() == [orc.token(4, i, c) for c in range(int(got[r]))]
        k += got.size
        j += 1
        bt.release()
    assert k == kept.size and j == (kept.size + b - 1) // b


@pytest.mark.parametrize("kind", ["ragged", "bucket"])
def test_full_size_cfg4r_cfg4b_epoch(dp, orc, kind):
    """cfg4r (the reference graph: filter -> ragged batch 128) and cfg4b
    (filter -> shuffle(10k, 42) -> bucket_by_length) at full size (1M
    sequences): row lengths / bucket membership follow the oracle batch for
    batch over the whole epoch; sampled rows hold the oracle's tokens."""
    n, max_keep = 1_000_000, 512
    lens = orc.lengths(n)
    kept = orc.filter_len_le(lens, max_keep)
    reg = dp.Registry()
    reg.register_length_filter("len<=512", max_keep)
    src = dp.Source.synthetic_tokens(n, 1024, 4, 4)
    g = dp.Dataset.token_sequences(reg, src).filter("len<=512")
    if kind == "ragged":
        g = g.batch(128)
        expect = [kept[i:i + 128] for i in range(0, kept.size, 128)]
    else:
        bounds, sizes = [128, 256, 384], [256, 128, 96, 64]
        g = g.shuffle(10000, 42).bucket_by_length(bounds, sizes)
        order = kept[orc.shuffle_order(kept.size, 10000, orc.shuffle_seed(1, 42))]
        expect = orc.bucket_by_length(lens, order, bounds, sizes)
    it = dp.make_iterator(g, seed_override=1)
    rng = np.random.default_rng(5)
    j = 0
    for bt in it:
        pos = expect[j]
        if kind == "ragged":
            vals, splits = bt.numpy(0), bt.numpy(1)
            got = np.diff(splits)
            rows = [vals[splits[r]:splits[r + 1]] for r in range(got.size)]
        else:
            toks, got = bt.numpy(0), bt.numpy(1)
            assert toks.shape == (pos.size, lens[pos].max())
            rows = [toks[r, :got[r]] for r in range(got.size)]
        assert np.array_equal(got, lens[pos])
        if j % 64 == 0:
            for r in rng.choice(got.size, 2, replace=False):
                assert rows[r].tolist() == [orc.token(4, int(pos[r]), c) for c in range(int(got[r]))]
        j += 1
        bt.release()
    assert j == len(expect)


def test_cfg4_reference_graph_filter_then_ragged_batch(dp, orc):
    """The reference's own cfg4 graph, Filter(len <= 512) -> Batch(128), as
    is: a batch of variable-length sequences comes out ragged (values back
    to back + int64 row splits) and equals the compiled reference's lists
    (golden cfg4_filter_batch: row lengths, tokens, batch sizes)."""
    c = GOLDEN["cfg4_filter_batch"]
    reg = dp.Registry()
    reg.register_length_filter("len<=512", c["max_keep"])
    src = dp.Source.synthetic_tokens(c["n"], c["max_len"], c["len_seed"], c["tok_seed"])
    g = dp.Dataset.token_sequences(reg, src).filter("len<=512").batch(c["batch"]).prefetch(-1)
    batches = drain(dp.make_iterator(g, seed_override=1), comps=(0, 1))
    sizes = [b[1].size - 1 for b in batches]
    lens = np.concatenate([np.diff(b[1]) for b in batches])
    toks = np.concatenate([b[0] for b in batches])
    assert all(b[1][0] == 0 and b[1][-1] == b[0].size for b in batches)
    assert len(sizes) == c["num_batches"] and sizes[-1] == c["last_batch"]
    assert fnv(orc, lens) == c["fnv_row_lengths"] and fnv(orc, toks) == c["fnv_tokens"]
    assert fnv(orc, sizes) == c["fnv_batch_sizes"]
    # drop_remainder, shuffle, repeat above, checkpoint
    g = dp.Dataset.token_sequences(reg, src).filter("len<=512").shuffle(999, 4).batch(100, drop_remainder=True)
    g = g.repeat(2)
    full = drain(dp.make_iterator(g, seed_override=3), comps=(0, 1))
    assert all(b[1].size == 101 for b in full)
    it = dp.make_iterator(g, seed_override=3)
    for _ in range(7):
        it.get_next().release()
    rest = drain(dp.restore(g, it.save()), comps=(0, 1))
    assert len(rest) == len(full) - 7
    assert all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) for a, b in zip(rest, full[7:]))


def test_cfg4_filter_then_shuffle_then_padded(dp, orc):
    n = 5000
    reg = dp.Registry()
    reg.register_length_filter("short", 300)
    src = dp.Source.synthetic_tokens(n, 1024, 9, 9)
    g = dp.Dataset.token_sequences(reg, src).filter("short").shuffle(700, 5).padded_batch(64, padding_value=-1)
    batches = drain(dp.make_iterator(g, seed_override=3), comps=(0, 1))
    lens_all = orc.lengths(n, 1024, 9)
    toks, offs = orc.tokens(lens_all, 9)
    kept = orc.filter_len_le(lens_all, 300)
    order = kept[orc.shuffle_order(kept.size, 700, orc.shuffle_seed(3, 5))]
    k = 0
    for b in batches:
        for r in range(b[1].size):
            p = order[k]
            assert b[1][r] == lens_all[p]
            assert (b[0][r, :b[1][r]] == toks[offs[p]:offs[p + 1]]).all() and (b[0][r, b[1][r]:] == -1).all()
            k += 1
    assert k == kept.size


def _check_bucket_batches(batches, expect, lens_all, toks, offs, pad):
    assert len(batches) == len(expect)
    for b, pos in zip(batches, expect):
        assert b[1].size == pos.size and (b[1] == lens_all[pos]).all()
        assert b[0].shape == (pos.size, lens_all[pos].max())
        for r, p in enumerate(pos):
            assert (b[0][r, :b[1][r]] == toks[offs[p]:offs[p + 1]]).all() and (b[0][r, b[1][r]:] == pad).all()


@pytest.mark.parametrize("drop", [False, True])
def test_cfg4_bucket_by_length_equals_oracle(dp, orc, drop):
    """cfg4 "/ bucket-by-length": filter -> shuffle -> bucket_by_length (K8)
    equals the sequential group_by_window restatement batch for batch."""
    n = 20000
    bounds, sizes = [64, 128, 256, 400], [64, 32, 16, 8, 5]
    reg = dp.Registry()
    reg.register_length_filter("len<=512", 512)
    src = dp.Source.synthetic_tokens(n, 1024, 4, 4)
    g = (dp.Dataset.token_sequences(reg, src).filter("len<=512").shuffle(3000, 11)
         .bucket_by_length(bounds, sizes, padding_value=-7, drop_remainder=drop).prefetch(-1))
    batches = drain(dp.make_iterator(g, seed_override=2), comps=(0, 1))
    lens_all = orc.lengths(n, 1024, 4)
    toks, offs = orc.tokens(lens_all, 4)
    kept = orc.filter_len_le(lens_all, 512)
    order = kept[orc.shuffle_order(kept.size, 3000, orc.shuffle_seed(2, 11))]
    expect = orc.bucket_by_length(lens_all, order, bounds, sizes, drop)
    _check_bucket_batches(batches, expect, lens_all, toks, offs, -7)


def test_bucket_by_length_edge_cases_and_epochs(dp, orc):
    """One bucket (= padded_batch), a bucket that never fills, every element
    in one bucket, repeat above the stage (per-epoch reshuffle), checkpoint
    seek into the middle."""
    n = 3000
    lens_all = orc.lengths(n, 300, 6)
    toks, offs = orc.tokens(lens_all, 6)
    reg = dp.Registry()
    src = dp.Source.synthetic_tokens(n, 300, 6, 6)
    cases = [([], [100]), ([1000], [7, 9]), ([10, 20, 30, 290, 299], [1, 2, 3, 4, 500, 6]), ([150], [4096, 3])]
    for bounds, sizes in cases:
        g = dp.Dataset.token_sequences(reg, src).bucket_by_length(bounds, sizes)
        expect = orc.bucket_by_length(lens_all, None, bounds, sizes)
        _check_bucket_batches(drain(dp.make_iterator(g, seed_override=1), comps=(0, 1)), expect, lens_all, toks,
                              offs, 0)
    g = dp.Dataset.token_sequences(reg, src).shuffle(500).bucket_by_length([100, 200], [16, 8, 4]).repeat(3)
    got = drain(dp.make_iterator(g, seed_override=9), comps=(0, 1))
    expect = []
    for e in range(3):
        order = orc.shuffle_order(n, 500, orc.shuffle_seed(orc.mix_seeds(9, e), None))
        expect += orc.bucket_by_length(lens_all, order, [100, 200], [16, 8, 4])
    _check_bucket_batches(got, expect, lens_all, toks, offs, 0)
    it = dp.make_iterator(g, seed_override=9)
    for _ in range(len(got) // 2):
        it.get_next().release()
    rest = drain(dp.restore(g, it.save()), comps=(0, 1))
    _check_bucket_batches(rest, expect[len(got) // 2:], lens_all, toks, offs, 0)


# ------------------------------------------------------------------ cfg5 ----
def test_cfg5_interleave_shuffle_map_and_batch(dp, orc):
    c = [x for x in GOLDEN["interleave"] if "shuffle" in x][0]
    m, cycle, records = c["num_sources"], c["cycle"], c["records"]
    reg = image_registry(dp, 0, crop=(32, 32))
    reg.register_record_reader("reader", records)
    recs = dp.Source.synthetic_images(m * records, 48, 48)
    g = (dp.Dataset.range(reg, m).shard(*c["shard"]).interleave("reader", cycle, c["parallel"], records=recs)
         .shuffle(*c["shuffle"]).map("crop").map("norm").batch(64).prefetch(-1))
    g, _ = g.optimize()
    batches = drain(dp.make_iterator(g, seed_override=1), comps=(0, 1))
    ids = np.concatenate([b[0] for b in batches])
    assert ids.size == c["count"] and ids[:8].tolist() == c["first"] and fnv(orc, ids) == c["fnv"]
    pix = batches[1][1]
    for r in (0, 7):
        p = int(batches[1][0][r])
        assert np.array_equal(pix[r], orc.crop_flip_normalize(orc.images(p, 1, 48, 48)[0], p, 32, 32))


def test_cfg5_sharded_record_residency(dp, orc, tmp_path):
    """cfg5 with block residency: process g of k holds only the record files
    of the interleave inputs shard(k, g) keeps (synthetic or read from its own
    files); its output equals the same graph over fully resident records,
    the shards' ids partition the dataset, and a mismatched shard / reader is
    rejected."""
    m, rec, k, cycle = 11, 6, 3, 4
    reg = image_registry(dp, 0, crop=(32, 32))
    reg.register_record_reader("reader", rec)
    reg.register_decode_raw("decode", 48, 48)
    imgs = orc.images(0, m * rec, 48, 48)
    paths = [str(tmp_path / f"part-{x}.rec") for x in range(m)]
    for x, p in enumerate(paths):
        dp.write_record_file(p, [im.tobytes() for im in imgs[x * rec:(x + 1) * rec]])

    def run(recs, g, par, decode=False):
        d = dp.Dataset.range(reg, m).shard(k, g).interleave("reader", cycle, par, records=recs)
        if decode:
            d = d.map("decode")
        d, _ = d.shuffle(20, 42).map("crop").map("norm").batch(8).prefetch(-1).optimize()
        return drain(dp.make_iterator(d, seed_override=1), comps=(0, 1))

    full = dp.Source.synthetic_records_sharded(m, rec, 48, 48)
    seen = []
    for g in range(k):
        for par in (1, cycle):
            want = run(full, g, par)
            got = run(dp.Source.synthetic_records_sharded(m, rec, 48, 48, k, g), g, par)
            files = run(dp.Source.records_from_files(paths, num_shards=k, index=g), g, par, decode=True)
            held = np.concatenate([imgs[x * rec:(x + 1) * rec] for x in range(g, m, k)])
            view = run(dp.Source.images_from_host(held).as_shard(m * rec, k, g, rec), g, par)
            assert len(got) == len(want) == len(files) == len(view)
            for a, b, c, v in zip(got, want, files, view):
                assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
                assert np.array_equal(c[0], b[0]) and np.array_equal(c[1], b[1])
                assert np.array_equal(v[0], b[0]) and np.array_equal(v[1], b[1])
        ids = np.concatenate([b[0] for b in got])
        assert sorted(ids.tolist()) == sorted(x * rec + r for x in range(g, m, k) for r in range(rec))
        p = int(got[-1][0][-1])
        assert np.array_equal(got[-1][1][-1], orc.crop_flip_normalize(imgs[p], p, 32, 32))
        seen += ids.tolist()
    assert sorted(seen) == list(range(m * rec))
    # checkpoint / restore (seek) and DPG1 round trip over block-resident records
    mine = dp.Source.synthetic_records_sharded(m, rec, 48, 48, k, 1)
    d = dp.Dataset.range(reg, m).shard(k, 1).interleave("reader", cycle, cycle, records=mine)
    d = d.shuffle(20, 42).map("crop").map("norm").batch(4).repeat(2)
    whole = drain(dp.make_iterator(d, seed_override=3), comps=(0, 1))
    it = dp.make_iterator(d, seed_override=3)
    for _ in range(5):
        it.get_next().release()
    rest = drain(dp.restore(d, it.save()), comps=(0, 1))
    assert len(rest) == len(whole) - 5
    assert all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) for a, b in zip(rest, whole[5:]))
    again = dp.Dataset.deserialize(reg, d.serialize(), sources=[mine])
    assert np.array_equal(drain(dp.make_iterator(again, seed_override=3))[0][0], whole[0][0])
    bad = [dp.Dataset.range(reg, m).shard(k, 0).interleave("reader", cycle, 1, records=mine),
           dp.Dataset.range(reg, m).interleave("reader", cycle, 1, records=mine)]
    reg.register_record_reader("reader5", rec - 1)
    bad.append(dp.Dataset.range(reg, m).shard(k, 1).interleave("reader5", cycle, 1, records=mine))
    for d in bad:
        with pytest.raises(dp.DpError) as e:
            dp.make_iterator(d.map("crop").map("norm").batch(8))
        assert e.value.code == dp.ERR["InvalidAttr"]
    with pytest.raises(dp.DpError) as e:  # wrong size for shard 0's files
        dp.Source.images_from_host(imgs[:rec * 3]).as_shard(m * rec, k, 0, rec)
    assert e.value.code == dp.ERR["InvalidAttr"]
    with pytest.raises(dp.DpError) as e:  # an input past the resident records
        dp.make_iterator(dp.Dataset.range(reg, m + 1).interleave("reader", cycle, 1, records=full).map("crop")
                         .map("norm").batch(8))
    assert e.value.code == dp.ERR["MalformedInput"]
    dp.write_record_file(paths[4], [imgs[0].tobytes()])  # held by shard 1: unequal held files
    with pytest.raises(dp.DpError) as e:
        dp.Source.records_from_files(paths, num_shards=k, index=1)
    assert e.value.code == dp.ERR["MalformedInput"]
    dp.Source.records_from_files(paths, num_shards=k, index=0)  # shard 0 does not read it


def test_interleave_over_record_files_equals_cfg5(dp, orc, tmp_path):
    """Interleave over record files (from_file +
    Interleave): input element x opens file x; equals the same pipeline over
    the in-memory records, and a file with the wrong record count is
    MalformedInput."""
    c = [x for x in GOLDEN["interleave"] if "shuffle" in x][0]
    m, cycle, records = c["num_sources"], c["cycle"], c["records"]
    imgs = orc.images(0, m * records, 48, 48)
    paths = [str(tmp_path / f"part-{x}.rec") for x in range(m)]
    for x, p in enumerate(paths):
        dp.write_record_file(p, [im.tobytes() for im in imgs[x * records:(x + 1) * records]])
    reg = image_registry(dp, 0, crop=(32, 32))
    reg.register_record_reader("reader", records)
    reg.register_decode_raw("decode", 48, 48)
    out = []
    for recs, pre in ((dp.Source.records_from_files(paths), ("decode",)), (dp.Source.images_from_host(imgs), ())):
        g = dp.Dataset.range(reg, m).shard(*c["shard"]).interleave("reader", cycle, c["parallel"], records=recs)
        for f in pre:
            g = g.map(f)
        g, _ = g.shuffle(*c["shuffle"]).map("crop").map("norm").batch(64).prefetch(-1).optimize()
        out.append(drain(dp.make_iterator(g, seed_override=1), comps=(0, 1)))
    ids = np.concatenate([b[0] for b in out[0]])
    assert ids.size == c["count"] and ids[:8].tolist() == c["first"] and fnv(orc, ids) == c["fnv"]
    for a, b in zip(*out):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    dp.write_record_file(paths[-1], [imgs[0].tobytes()])  # one record short
    g = dp.Dataset.range(reg, m).interleave("reader", cycle, 1, records=dp.Source.records_from_files(paths))
    with pytest.raises(dp.DpError) as e:
        dp.make_iterator(g.map("decode").map("crop").map("norm").batch(8))
    assert e.value.code == dp.ERR["MalformedInput"]


def test_interleave_over_unequal_record_files(dp, orc, tmp_path):
    """Record files of different sizes (reader registered with 0 records =
    each file's own count): the host schedule + K6 interleave_var give the
    reference's order (sequential loop; parallel too when no file is empty),
    then shuffle + crop; an empty file under a parallel interleave is
    rejected (the reference's parallel order differs there)."""
    lens = [7, 3, 0, 9, 1, 5, 4, 6, 2, 8, 5]
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]])
    imgs = orc.images(0, int(sum(lens)), 40, 40)
    paths = [str(tmp_path / f"f{i}.rec") for i in range(len(lens))]
    for i, p in enumerate(paths):
        dp.write_record_file(p, [imgs[starts[i] + r].tobytes() for r in range(lens[i])])
    reg = image_registry(dp, 0, crop=(32, 32))
    reg.register_record_reader("files", 0)
    reg.register_decode_raw("decode", 40, 40)
    recs = dp.Source.records_from_files(paths)
    for cycle, par, shard in ((3, 1, None), (4, 1, (2, 1)), (2, 1, (3, 0))):
        g = dp.Dataset.range(reg, len(lens))
        if shard:
            g = g.shard(*shard)
        g = g.interleave("files", cycle, par, records=recs).map("decode").map("crop").map("norm").batch(6)
        got = drain(dp.make_iterator(g, seed_override=1), comps=(0, 1))
        inputs = np.arange(shard[1], len(lens), shard[0]) if shard else np.arange(len(lens))
        want = orc.interleave_var(inputs, cycle, lens)
        ids = np.concatenate([b[0] for b in got])
        assert ids.tolist() == want.tolist()
        p = int(ids[-1])
        assert np.array_equal(got[-1][1][-1], orc.crop_flip_normalize(imgs[p], p, 32, 32))
    # parallel is reproduced without empty files
    lens2 = [x + 1 for x in lens]
    starts2 = np.concatenate([[0], np.cumsum(lens2)[:-1]])
    imgs2 = orc.images(0, int(sum(lens2)), 40, 40)
    paths2 = [str(tmp_path / f"g{i}.rec") for i in range(len(lens2))]
    for i, p in enumerate(paths2):
        dp.write_record_file(p, [imgs2[starts2[i] + r].tobytes() for r in range(lens2[i])])
    g = (dp.Dataset.range(reg, len(lens2)).interleave("files", 4, 4, records=dp.Source.records_from_files(paths2))
         .shuffle(20, 3).map("decode").map("crop").map("norm").batch(8))
    ids = np.concatenate([b[0] for b in drain(dp.make_iterator(g, seed_override=2))])
    order = orc.interleave_var(np.arange(len(lens2)), 4, lens2)
    assert ids.tolist() == order[orc.shuffle_order(order.size, 20, orc.shuffle_seed(2, 3))].tolist()
    with pytest.raises(dp.DpError) as e:
        dp.make_iterator(dp.Dataset.range(reg, len(lens)).interleave("files", 4, 4, records=recs)
                         .map("decode").map("crop").map("norm").batch(8))
    assert e.value.code == dp.ERR["InvalidAttr"]


def test_sharded_residency_equals_shard_of_full_dataset(dp, orc):
    """Per-GPU residency: a process holding only shard i of k
    produces exactly shard(k, i) of the full dataset, ids and pixels."""
    n, buf = 2000, 300
    reg = image_registry(dp, 0, crop=(48, 48))
    for k in (2, 8):
        seen = []
        for i in range(k):
            src = dp.Source.synthetic_images_sharded(n, 64, 64, k, i)
            g, _ = dp.Dataset.tensor_slices(reg, src).shard(k, i).shuffle(buf, 42).map("crop").map("norm") \
                .batch(64).optimize()
            batches = drain(dp.make_iterator(g, seed_override=1), comps=(0, 1))
            ids = np.concatenate([b[0] for b in batches])
            pos = orc.shard_positions(n, k, i)
            want = pos[orc.shuffle_order(pos.size, buf, orc.shuffle_seed(1, 42))]
            assert (ids == want).all(), (k, i)
            p = int(batches[0][0][3])
            assert np.array_equal(batches[0][1][3], orc.crop_flip_normalize(orc.images(p, 1, 64, 64)[0], p, 48, 48))
            seen.append(ids)
        assert sorted(np.concatenate(seen).tolist()) == list(range(n))
    src = dp.Source.synthetic_images_sharded(n, 64, 64, 4, 1)
    bad = dp.Dataset.tensor_slices(reg, src).map("crop").map("norm").batch(8)
    with pytest.raises(Exception) as e:
        dp.make_iterator(bad)
    assert "apply shard(4, 1)" in str(e.value)


def _ids_all(dp, it, comp=0):
    out = []
    while (b := it.get_next()) is not None:
        out.append(b.numpy(comp).reshape(-1))
        b.release()
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def test_checkpoint_restore_equals_uninterrupted(dp):
    """Save at random cut points, Restore (O(1) seek, no replay) and continue:
    the concatenation equals the uninterrupted sequence
    (acceptance criterion #8, P/tests/acceptance/acceptance_main.cpp:361-398)."""
    rng = np.random.default_rng(8)
    reg = image_registry(dp, 0, crop=(32, 32))
    reg.register_affine("aff", 5, -2)
    reg.register_length_filter("short", 100)
    imgs = dp.Source.synthetic_images(700, 48, 48)
    toks = dp.Source.synthetic_tokens(900, 300, 3, 3)
    graphs = [  # spanning epochs, per-epoch repeat with a ragged last batch, big groups, padded batches
        dp.Dataset.tensor_slices(reg, imgs).shuffle(150, 9).repeat(3).map("crop").map("norm").batch(64),
        dp.Dataset.tensor_slices(reg, imgs).shuffle(150, 9).map("crop").map("norm").batch(64).repeat(3),
        dp.Dataset.range(reg, 100_000).shuffle(5000, 1).map("aff").batch(1000).repeat(2),
        dp.Dataset.token_sequences(reg, toks).filter("short").padded_batch(32).repeat(2),
    ]
    for g in graphs:
        g, _ = g.optimize()
        full = _ids_all(dp, dp.make_iterator(g, seed_override=4))
        total = dp.make_iterator(g, seed_override=4).skip(10 ** 9)
        for cut in sorted(set(rng.integers(0, total + 1, 5).tolist()) | {0, total}):
            it = dp.make_iterator(g, seed_override=4)
            head = []
            for _ in range(cut):
                b = it.get_next()
                head.append(b.numpy(0).reshape(-1))
                b.release()
            blob = it.save()
            assert blob[:4] == b"DPC1"
            rest = _ids_all(dp, dp.restore(g, blob))
            got = np.concatenate(head + [rest]) if head else rest
            assert np.array_equal(got, full), (str(g)[:60], cut, total)
        with pytest.raises(Exception):
            dp.restore(graphs[0] if g is not graphs[0] else graphs[1], blob)  # different pipeline


def test_edge_cases(dp, orc):
    reg = dp.Registry()
    reg.register_affine("inc", 1, 1)
    reg.register_length_filter("none", 0)
    reg.register_record_reader("zero", 0)

    def vals(g, **kw):
        return [b[0].tolist() for b in drain(dp.make_iterator(g, seed_override=1, **kw))]

    assert vals(dp.Dataset.range(reg, 0).map("inc").batch(4)) == []                       # empty source
    assert vals(dp.Dataset.range(reg, 5).map("inc").batch(10)) == [[1, 2, 3, 4, 5]]       # batch > dataset
    assert vals(dp.Dataset.range(reg, 5).map("inc").batch(10, drop_remainder=True)) == []
    assert vals(dp.Dataset.range(reg, 1).shuffle(100, 3).batch(4)) == [[0]]               # n = 1
    got = vals(dp.Dataset.range(reg, 50).shuffle(1000, 3).batch(64))[0]                     # buffer > n
    assert got == orc.shuffle_order(50, 1000, orc.shuffle_seed(1, 3)).tolist()
    assert vals(dp.Dataset.range(reg, 3).shard(8, 5).batch(2)) == []                        # shard past the end
    assert vals(dp.Dataset.range(reg, 3).shard(8, 2).batch(2)) == [[2]]
    assert vals(dp.Dataset.range(reg, 7).map("inc").batch(3).repeat(2)) == [[1, 2, 3], [4, 5, 6], [7]] * 2
    src = dp.Source.synthetic_tokens(100, 50, 1, 1)
    assert vals(dp.Dataset.token_sequences(reg, src).filter("none").padded_batch(8)) == []  # filter keeps none
    assert vals(dp.Dataset.range(reg, 4).interleave("zero", 2, 1).batch(2)) == []          # empty readers
    assert vals(dp.Dataset.token_sequences(reg, src).filter("none").bucket_by_length([10], [4, 4])) == []
    # EOF is sticky (runtime.cpp:147-156)
    it = dp.make_iterator(dp.Dataset.range(reg, 3).batch(2), seed_override=1)
    assert [it.get_next() is None for _ in range(5)] == [False, False, True, True, True]
    # infinite repeat keeps producing; sticky end never reached
    it = dp.make_iterator(dp.Dataset.range(reg, 3).batch(2).repeat(-1), seed_override=1)
    assert [it.get_next().numpy(0).tolist() for _ in range(5)] == [[0, 1], [2], [0, 1], [2], [0, 1]]


def test_unsupported_graph_fails_loudly(dp):
    reg = dp.Registry()
    src = dp.Source.synthetic_tokens(100, 50, 1, 1)
    g = dp.Dataset.token_sequences(reg, src).repeat(2).padded_batch(8)  # batches across epochs: not lowered
    with pytest.raises(Exception) as e:
        dp.make_iterator(g)
    assert "device lowering" in str(e.value)
