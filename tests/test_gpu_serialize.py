"""Cross-engine checkpoints and device-source serialization on the GPU.

* A DPC1 blob saved by the COMPILED REFERENCE after k GetNext calls
  (golden.json["checkpoint"], src/checkpoint.cpp Save) restores here and
  continues exactly where the uninterrupted sequence does; this engine's own
  Save of the same position carries the reference's fingerprint.
* from_file serializes to the reference's bytes (paths only).
* tensor_slices data is re-bound at Deserialize (descriptor-checked)."""
import json
import os

import numpy as np
import pytest

from tests.test_serialize import GOLDEN, CKPT, pipeline, registry

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2101_12127_b200 import pipeline
    return pipeline


def ids(it):
    out = []
    while (b := it.get_next()) is not None:
        out.append(b.numpy(0).reshape(-1).copy())
        b.release()
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def test_restore_from_reference_checkpoint(dp):
    reg = registry()
    for c in CKPT:
        g = pipeline(reg, c["which"])
        blob = bytes.fromhex(c["dpc1_hex"])
        full = ids(dp.make_iterator(g, seed_override=1))
        it = dp.make_iterator(g, seed_override=1)
        head = [it.get_next() for _ in range(c["k"])]
        done = sum(b.numpy(0).size for b in head)
        for b in head:
            b.release()
        ours = it.save()
        assert ours[6:38] == blob[6:38]                 # same fingerprint as the reference's Save
        assert ours[38:55] == blob[38:55]               # base seed, deterministic, root_delivered
        rest = ids(dp.restore(g, blob))
        assert np.array_equal(rest, full[done:])


def test_from_file_serializes_like_the_reference(dp, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    dp.write_record_file("part-0.rec", [b"a", b"bb"])
    dp.write_record_file("part-1.rec", [b"ccc"])
    reg = registry()
    g = dp.Dataset.from_file(reg, ["part-0.rec", "part-1.rec"]).batch(2)
    assert g.serialize().hex() == GOLDEN[5]["dpg1_hex"]
    assert g.fingerprint() == GOLDEN[5]["fingerprint"]
    assert dp.Dataset.deserialize(reg, g.serialize()).serialize() == g.serialize()


def test_tensor_slices_rebinds_its_source(dp):
    reg = dp.Registry()
    reg.register_random_crop_flip("crop", 32, 32, seed=7)
    reg.register_normalize("norm")
    src = dp.Source.synthetic_images(300, 48, 48)
    g, _ = dp.Dataset.tensor_slices(reg, src).shuffle(100, 3).map("crop").map("norm").batch(32).optimize()
    b = g.serialize()
    g2 = dp.Dataset.deserialize(reg, b, sources=[src])
    assert g2.serialize() == b and g2.fingerprint() == g.fingerprint()
    a = dp.make_iterator(g, seed_override=2)
    c = dp.make_iterator(g2, seed_override=2)
    while (x := a.get_next()) is not None:
        y = c.get_next()
        assert np.array_equal(x.numpy(0), y.numpy(0)) and np.array_equal(x.numpy(1), y.numpy(1))
        x.release()
        y.release()
    assert c.get_next() is None
    with pytest.raises(dp.DpError) as e:
        dp.Dataset.deserialize(reg, b)
    assert e.value.code == dp.ERR["ValidationFailed"]
    with pytest.raises(dp.DpError) as e:
        dp.Dataset.deserialize(reg, b, sources=[dp.Source.synthetic_images(301, 48, 48)])
    assert e.value.code == dp.ERR["ValidationFailed"]
