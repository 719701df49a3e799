"""Graph serialization and fingerprints (formats.md "Graph serialization" /
"Fingerprint"; reference src/serialize.cpp).  The DPG1 bytes and SHA-256
fingerprints of pipelines both engines express are compared with known
answers generated from the COMPILED REFERENCE (tests/golden/make_golden.py
-> golden.json["serialize"], oracle/ref_shim.cpp ref_serialize_pipeline).
Graph building does no device work for these sources, so this runs on CPU.
Mirrors P/tests/test_serialize.cpp (round trip, seed invariance, malformed
input, version mismatch, unknown UDF)."""
import json
import os

import pytest

from paper_2101_12127_b200 import pipeline as dp
from paper_2101_12127_b200._capi import DpError

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = {c["which"]: c for c in json.load(open(os.path.join(HERE, "golden", "golden.json")))["serialize"]}


def registry():
    reg = dp.Registry()
    reg.register_affine("affine(3,1)", 3, 1)
    reg.register_affine("affine(2,0)", 2, 0)
    reg.register_record_reader("reader(3)", 3)
    return reg


def pipeline(reg, which):
    """The same shapes as ref_serialize_pipeline (oracle/ref_shim.cpp)."""
    D = dp.Dataset
    if which in (0, 1):
        g = D.from_memory(reg, range(10)).map("affine(3,1)", 4).batch(4)
        return g.optimize()[0] if which == 1 else g
    if which == 2:
        return D.from_memory(reg, range(100)).shuffle(10, 42).repeat(3).batch(8).prefetch(-1).optimize()[0]
    if which == 3:
        g = D.from_memory(reg, range(64)).shard(4, 1).shuffle(50).map("affine(3,1)", -1).map("affine(2,0)", 2)
        return g.batch(16, drop_remainder=True).prefetch(2).optimize()[0]
    if which == 4:
        return D.from_memory(reg, range(8)).interleave("reader(3)", 2, 1).batch(5)
    raise ValueError(which)


@pytest.mark.parametrize("which", [0, 1, 2, 3, 4])
def test_bytes_and_fingerprint_equal_the_reference(which):
    g = pipeline(registry(), which)
    assert g.serialize().hex() == GOLDEN[which]["dpg1_hex"]
    assert g.fingerprint() == GOLDEN[which]["fingerprint"]


@pytest.mark.parametrize("which", [0, 1, 2, 3, 4])
def test_round_trip(which):
    reg = registry()
    b = pipeline(reg, which).serialize()
    g2 = dp.Dataset.deserialize(reg, b)
    assert g2.serialize() == b
    assert str(g2) == str(pipeline(reg, which))


def test_fingerprint_is_seed_invariant_and_structure_sensitive():
    reg = registry()
    D = dp.Dataset
    a = D.from_memory(reg, range(100)).shuffle(10, 42).batch(8)
    b = D.from_memory(reg, range(100)).shuffle(10, 7).batch(8)
    c = D.from_memory(reg, range(100)).shuffle(11, 42).batch(8)
    d = D.from_memory(reg, range(101)).shuffle(10, 42).batch(8)
    assert a.serialize() != b.serialize()
    assert a.fingerprint() == b.fingerprint()
    assert len({a.fingerprint(), c.fingerprint(), d.fingerprint()}) == 3


def test_device_kinds_round_trip():
    """Range / padded_batch are this engine's kinds (ids 32-35): they
    serialize and round-trip; a device-source descriptor needs its source."""
    reg = registry()
    g = dp.Dataset.range(reg, 1000).map("affine(3,1)").batch(64).optimize()[0]
    b = g.serialize()
    assert dp.Dataset.deserialize(reg, b).serialize() == b


def test_malformed_and_version_errors():
    reg = registry()
    b = pipeline(reg, 0).serialize()
    cases = [(b"XXXX" + b[4:], "MalformedInput"), (b[:-3], "MalformedInput"), (b + b"\0", "MalformedInput"),
             (b[:4] + b"\x02\x00" + b[6:], "VersionMismatch"),
             (b[:6] + (5).to_bytes(4, "little") + b[10:], "MalformedInput"),  # node count mismatch
             (b[:10] + b"\x63" + b[11:], "MalformedInput")]                    # unknown kind
    for data, code in cases:
        with pytest.raises(DpError) as e:
            dp.Dataset.deserialize(reg, data)
        assert e.value.code == dp.ERR[code], (data[:12], str(e.value))
    # a reference kind off the device path (flat_map = 4) fails validation
    with pytest.raises(DpError) as e:
        dp.Dataset.deserialize(reg, b[:10] + b"\x04" + b[11:])
    assert e.value.code == dp.ERR["ValidationFailed"]


def test_unknown_udf_on_deserialize():
    """Graphs reference UDFs by name only (formats.md): the deserialized graph
    reports UnknownUdf at MakeIterator, as a freshly built one does
    (runtime.cpp:2117-2156), before any device work."""
    b = pipeline(registry(), 0).serialize()
    reg = dp.Registry()  # affine(3,1) not registered
    g = dp.Dataset.deserialize(reg, b)
    with pytest.raises(DpError) as e:
        dp.make_iterator(g, seed_override=1)
    assert e.value.code == dp.ERR["UnknownUdf"]


CKPT = json.load(open(os.path.join(HERE, "golden", "golden.json")))["checkpoint"]


def test_reference_checkpoint_passes_validation_here():
    """A DPC1 blob SAVED BY THE REFERENCE (golden) passes this engine's magic /
    version / fingerprint checks for the same graph -- without a GPU the
    Restore then stops at the device step (no CPU fallback) -- while a
    different graph is FingerprintMismatch and a damaged blob CorruptBlob."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU (tests/test_gpu_serialize.py restores for real)")
    reg = registry()
    for c in CKPT:
        blob = bytes.fromhex(c["dpc1_hex"])
        with pytest.raises(DpError) as e:
            dp.restore(pipeline(reg, c["which"]), blob)
        assert e.value.code == dp.ERR["Cuda"], str(e.value)
        other = pipeline(reg, 4 if c["which"] != 4 else 0)
        with pytest.raises(DpError) as e:
            dp.restore(other, blob)
        assert e.value.code == dp.ERR["FingerprintMismatch"]
        with pytest.raises(DpError) as e:
            dp.restore(pipeline(reg, c["which"]), blob[:-3])
        assert e.value.code == dp.ERR["CorruptBlob"]
