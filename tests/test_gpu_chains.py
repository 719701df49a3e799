"""The device UDF library's general image chains (K9) and multi-component
(image, label) elements, against known answers generated through the
compiled reference (tests/golden/chains.json, make_chain_golden.py): a
plain u8 batch with no map, crop-only u8, center crop, crop>>resize
(RandomResizedCrop at a fixed scale), resize>>center-crop (ResNet eval),
fp32 affine on images, pixel ops before a resize, two crops, and labels
through the K3 / K4 / K9 paths.  Bit-exact: ids, every output byte, labels,
batch sizes (the reference's map(f).map(g) composition and Batch,
P/src/optimizer.cpp:165-188, P/src/runtime.cpp:579-637)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "chains.json")))


@pytest.fixture(scope="module")
def dp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2101_12127_b200 import pipeline
    return pipeline


def register_steps(dp, reg, steps):
    names = []
    for i, st in enumerate(steps):
        name = f"s{i}_{st[0]}"
        if st[0] == "random_crop":
            reg.register_random_crop_flip(name, st[1], st[2], seed=st[3], flip=st[4])
        elif st[0] == "center_crop":
            reg.register_center_crop(name, st[1], st[2])
        elif st[0] == "resize":
            reg.register_resize_bilinear(name, st[1], st[2])
        elif st[0] == "normalize":
            reg.register_normalize(name, st[1], st[2])
        elif st[0] == "affine":
            reg.register_image_affine(name, st[1], st[2])
        names.append(name)
    return names


def labels_for(n):
    return (np.arange(n, dtype=np.int64) * 7919) % 1000 - 3


def build(dp, case, n=None, **kw):
    n = n or GOLD["n"]
    reg = dp.Registry()
    names = register_steps(dp, reg, case["steps"])
    src = dp.Source.synthetic_images(n, *case["in_hw"])
    if case["labels"]:
        src = src.with_labels(labels_for(n))
    g = dp.Dataset.tensor_slices(reg, src).shuffle(*GOLD["shuffle"])
    for nm in names:
        g = g.map(nm)
    return g, src


def drain_all(it, labels):
    ids, imgs, labs, sizes = [], [], [], []
    for b in it:
        ids.append(b.numpy(0))
        imgs.append(b.numpy(1))
        if labels:
            labs.append(b.numpy(2))
        sizes.append(ids[-1].size)
        b.release()
    return np.concatenate(ids), np.concatenate(imgs), (np.concatenate(labs) if labels else None), sizes


@pytest.mark.parametrize("name", [c["name"] for c in GOLD["cases"]])
def test_chain_equals_the_reference(dp, orc, name):
    case = [c for c in GOLD["cases"] if c["name"] == name][0]
    g, src = build(dp, case)
    g, _ = g.batch(GOLD["batch"]).prefetch(-1).optimize()
    it = dp.make_iterator(g, seed_override=GOLD["base_seed"])
    ids, imgs, labs, sizes = drain_all(it, case["labels"])
    assert sizes == case["batch_sizes"]
    assert imgs.shape[1:] == (case["out"][0], case["out"][1], 3) and imgs.dtype == np.dtype(case["out"][2])
    assert f"{orc.fnv_digest(ids):016x}" == case["ids"]
    assert f"{orc.order_digest(imgs.reshape(-1).view(np.uint32)):016x}" == case["images"], name
    if case["labels"]:
        assert f"{orc.fnv_digest(labs):016x}" == case["label_fnv"]
        assert np.array_equal(labs, labels_for(GOLD["n"])[ids])


def test_chain_kinds_lower_to_the_expected_kernels(dp):
    want = {"u8_batch": "K9 gather_copy", "crop_only": "K9 image_chain", "crop_resize_normalize": "K9 image_chain",
            "crop_flip_normalize_labels": "K3", "resize_normalize_labels": "K4", "center_crop_normalize_labels": "K3"}
    for name, kernel in want.items():
        case = [c for c in GOLD["cases"] if c["name"] == name][0]
        g, _ = build(dp, case)
        it = dp.make_iterator(g.batch(16), seed_override=1)
        assert kernel in it.describe(), (name, it.describe())


def test_chains_unbatched_host_output_and_restore(dp, orc):
    """Single elements (id, image, label) through a K9 chain; host_output
    batches equal device batches; a restored iterator continues exactly."""
    case = [c for c in GOLD["cases"] if c["name"] == "center_crop_normalize_labels"][0]
    g, src = build(dp, case, n=100)
    got = []
    for e in dp.make_iterator(g, seed_override=1):
        comps = e.components
        assert len(comps) == 3
        got.append((e.numpy(0), e.numpy(1), e.numpy(2)))
        e.release()
    gb, _ = g.batch(16).optimize()
    dev = drain_all(dp.make_iterator(gb, seed_override=1), True)
    host = []
    for b in dp.make_iterator(gb, seed_override=1, host_output=True):
        b.wait()
        host.append((b.host_view(0).copy(), b.host_view(1).copy(), b.host_view(2).copy()))
        b.release()
    assert np.array_equal(np.concatenate([h[0] for h in host]), dev[0])
    assert np.array_equal(np.concatenate([h[1] for h in host]).view(np.uint32), dev[1].view(np.uint32))
    assert np.array_equal(np.concatenate([h[2] for h in host]), dev[2])
    assert [int(x[0]) for x in got] == dev[0].tolist()
    assert [int(x[2]) for x in got] == dev[2].tolist()
    assert np.array_equal(np.stack([x[1] for x in got]).view(np.uint32), dev[1].view(np.uint32))
    it = dp.make_iterator(gb, seed_override=1)
    for _ in range(3):
        it.get_next().release()
    rest = drain_all(dp.restore(gb, it.save()), True)
    assert np.array_equal(rest[0], dev[0][48:]) and np.array_equal(rest[2], dev[2][48:])


def test_invalid_chains_fail_loudly(dp):
    reg = dp.Registry()
    reg.register_resize_bilinear("r1", 20, 20)
    reg.register_resize_bilinear("r2", 10, 10)
    reg.register_random_crop_flip("c", 8, 8, seed=1, flip=True)
    src = dp.Source.synthetic_images(10, 32, 32)
    g = dp.Dataset.tensor_slices(reg, src).map("r1").map("r2").batch(4)
    with pytest.raises(Exception, match="one resize"):
        dp.make_iterator(g)
    g = dp.Dataset.tensor_slices(reg, src).map("c").map("c").map("c").batch(4)
    with pytest.raises(Exception, match="crop"):
        dp.make_iterator(g)
    with pytest.raises(Exception):
        src.with_labels(np.arange(9))
