"""CPU-side checks of the C ABI and the host graph layer (no GPU needed).

* libdpcuda.so loads and exports every dp_* symbol include/*.h declares;
* graph construction / validation / Optimize mirror the reference's
  operator API and rewrite contract (P/tests/test_graph.cpp,
  P/tests/test_optimizer.cpp: map_batch fusion yields map_and_batch, a fused
  predicate blocks it, rule disabling, composed-UDF names);
* MakeIterator validates UDFs before touching the device (UnknownUdf,
  runtime.cpp:2117-2156) and fails loudly without a GPU (no CPU fallback).
"""
import ctypes

import pytest

from paper_2101_12127_b200 import _capi, pipeline as dp
from paper_2101_12127_b200._capi import DpError


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    names = _capi.declared_symbols()
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert b"sm_100a" in lib.dp_build_info()


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not any(a in out for a in ("sm_80", "sm_90", "sm_89"))


def test_device_count_without_gpu_is_not_an_error():
    c = ctypes.c_int(-1)
    assert _capi.lib().dp_device_count(ctypes.byref(c)) == 0 and c.value >= 0


def reg_cfg1():
    reg = dp.Registry()
    reg.register_affine("affine(3,1)", 3, 1)
    return reg


def test_map_batch_fusion_yields_map_and_batch():
    reg = reg_cfg1()
    g = dp.Dataset.range(reg, 1_000_000).map("affine(3,1)").batch(1024)
    assert g.root_kind == "batch"
    opt, report = g.optimize()
    assert opt.root_kind == "map_and_batch"
    assert "map_batch_fusion at /batch@0" in report
    # spec of the fused node: an int64 batch tensor of unknown length
    assert "map_and_batch" in str(opt) and "tensor<int64[?]>" in str(opt)


def test_disabled_rule_keeps_unfused_graph():
    reg = reg_cfg1()
    g = dp.Dataset.range(reg, 10).map("affine(3,1)").batch(4)
    opt, report = g.optimize(disabled_rules=("map_batch_fusion",))
    assert opt.root_kind == "batch" and "no rewrites applied" in report
    with pytest.raises(DpError) as e:
        g.optimize(disabled_rules=("no_such_rule",))
    assert e.value.code == dp.ERR["InvalidAttr"]


def test_map_map_fusion_composes_names_then_fuses_batch():
    reg = reg_cfg1()
    reg.register_affine("times2", 2, 0)
    g = dp.Dataset.range(reg, 10).map("affine(3,1)", 2).map("times2", -1).batch(4)
    opt, report = g.optimize()
    assert report.index("map_map_fusion") < report.index("map_batch_fusion")
    assert opt.root_kind == "map_and_batch"
    s = str(opt)
    assert "udf=(affine(3,1))>>(times2)" in s and "num_parallel_calls=-1" in s  # AUTOTUNE absorbing
    assert reg.contains("(affine(3,1))>>(times2)")


def test_map_on_wrong_element_type_is_type_mismatch():
    reg = dp.Registry()
    reg.register_random_crop_flip("crop", 224, 224, seed=7)
    with pytest.raises(DpError) as e:
        dp.Dataset.range(reg, 10).map("crop")
    assert e.value.code == dp.ERR["TypeMismatch"]


def test_shuffle_repeat_fusion_and_fused_predicate_blocks_map_batch():
    reg = reg_cfg1()
    reg.register_length_filter("short", 512)
    g = dp.Dataset.range(reg, 100).shuffle(10, seed=42).repeat(3)
    opt, report = g.optimize()
    assert "shuffle_repeat_fusion" in report and "fused_with_repeat=1" in str(opt)
    # map + filter fuse into one map carrying the predicate; batch then does
    # NOT fuse with it (optimizer.cpp:258-264)
    g2 = dp.Dataset.range(reg, 100).map("affine(3,1)").filter("short").batch(8)
    opt2, report2 = g2.optimize()
    assert "map_filter_fusion" in report2 and "map_batch_fusion" not in report2
    assert opt2.root_kind == "batch"


def test_attr_validation_errors():
    reg = reg_cfg1()
    base = dp.Dataset.range(reg, 10)
    for build in (lambda: base.batch(0), lambda: base.shard(2, 2), lambda: base.shard(0, 0),
                  lambda: base.shuffle(0), lambda: base.prefetch(0), lambda: base.repeat(0),
                  lambda: base.map("affine(3,1)", 0), lambda: dp.Dataset.range(reg, -1)):
        with pytest.raises(DpError) as e:
            build()
        assert e.value.code == dp.ERR["InvalidAttr"]
    # AUTOTUNE is legal for parallelism and prefetch
    base.map("affine(3,1)", -1).batch(4).prefetch(-1)


def test_duplicate_udf_name():
    reg = reg_cfg1()
    with pytest.raises(DpError) as e:
        reg.register_affine("affine(3,1)", 1, 1)
    assert e.value.code == dp.ERR["DuplicateName"]


def test_unknown_udf_fails_at_make_iterator_before_device():
    reg = dp.Registry()
    g = dp.Dataset.range(reg, 3).map("nope").batch(2)
    with pytest.raises(DpError) as e:
        dp.make_iterator(g, seed_override=1)
    assert e.value.code == dp.ERR["UnknownUdf"]


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    reg = reg_cfg1()
    g = dp.Dataset.range(reg, 3).map("affine(3,1)").batch(2)
    with pytest.raises(DpError) as e:
        dp.make_iterator(g, seed_override=1)
    assert e.value.code == dp.ERR["Cuda"] and "no CPU fallback" in str(e.value)


def test_checkpoint_restore_validation_before_device():
    """Restore checks magic / version / length / fingerprint first
    (P/tests/test_checkpoint.cpp:104-139: corrupt, truncated, versioned)."""
    import struct
    reg = reg_cfg1()
    g = dp.Dataset.range(reg, 100).map("affine(3,1)").batch(10)

    def blob(magic=b"DPC1", version=1, fp=b"\0" * 32, entries=b"", extra=b""):
        return magic + struct.pack("<H", version) + fp + struct.pack("<QBQI", 1, 1, 3, 0) + entries + extra

    for bad, code in ((b"", "CorruptBlob"), (b"XXXX\x01\x00", "CorruptBlob"), (blob(version=2), "VersionMismatch"),
                      (blob()[:20], "CorruptBlob"), (blob(extra=b"\0"), "CorruptBlob"),
                      (blob(), "FingerprintMismatch")):
        with pytest.raises(DpError) as e:
            dp.restore(g, bad)
        assert code in str(e.value), (bad, str(e.value))
    codes = {"CorruptBlob": 12, "VersionMismatch": 11, "FingerprintMismatch": 10}
    with pytest.raises(DpError) as e:
        dp.restore(g, blob(version=7))
    assert e.value.code == codes["VersionMismatch"]


def test_kernel_entry_rejects_bad_args_without_launching():
    lib = _capi.lib()
    assert lib.dp_k_range_affine_batch(0, -1, 1, 0, None, None) == dp.ERR["InvalidAttr"]
    assert lib.dp_k_shuffle_plan(10, 0, 1, None, None, None, None) == dp.ERR["InvalidAttr"]
    assert lib.dp_k_shard_index(10, 0, 0, None, None, None) == dp.ERR["InvalidAttr"]
    assert b"num_shards" in lib.dp_last_error()
    assert lib.dp_k_shard_interleave_count(64, 8, 3, 16) == 8 * 16


def test_write_record_file_format(tmp_path):
    """WriteRecordFile (runtime.hpp:102-107, formats.md:67-74): [u32 LE len][payload]."""
    p = tmp_path / "r.rec"
    dp.write_record_file(str(p), [b"ab", b"", b"xyz"])
    assert p.read_bytes() == b"\x02\x00\x00\x00ab" + b"\x00\x00\x00\x00" + b"\x03\x00\x00\x00xyz"


def test_from_file_errors_raised_before_device(tmp_path):
    """FromFileIterator (runtime.cpp:416-474): a missing file is MissingFile, a
    truncated length or payload MalformedInput -- raised while reading, before
    any device memory is touched (so they hold without a GPU)."""
    reg = dp.Registry()
    with pytest.raises(DpError) as e:
        dp.Dataset.from_file(reg, [str(tmp_path / "absent.rec")])
    assert e.value.code == dp.ERR["MissingFile"]
    good = tmp_path / "good.rec"
    dp.write_record_file(str(good), [b"hello"])
    for name, blob in (("len.rec", b"\x05\x00"), ("payload.rec", b"\x05\x00\x00\x00hel")):
        bad = tmp_path / name
        bad.write_bytes(blob)
        with pytest.raises(DpError) as e:
            dp.Dataset.from_file(reg, [str(good), str(bad)])
        assert e.value.code == dp.ERR["MalformedInput"]
        assert "truncated record" in str(e.value)
    with pytest.raises(DpError) as e:
        dp.Dataset.from_file(reg, [])
    assert e.value.code == dp.ERR["InvalidAttr"]


def test_bucket_by_length_attr_validation():
    """bucket_by_length attrs are checked when the node is built (before any
    device work): increasing boundaries, one batch size per bucket, <= 32
    buckets; a non-sequence input is TypeMismatch."""
    reg = dp.Registry()
    base = dp.Dataset.range(reg, 10)
    for bounds, sizes in (([5, 3], [1, 1, 1]), ([5], [1, 0]), (list(range(1, 33)), [1] * 33), ([-1], [1, 1])):
        with pytest.raises(DpError) as e:
            base.bucket_by_length(bounds, sizes)
        assert e.value.code == dp.ERR["InvalidAttr"], (bounds, sizes)
    with pytest.raises(ValueError):
        base.bucket_by_length([5], [1])
    with pytest.raises(DpError) as e:
        base.bucket_by_length([5], [1, 2])
    assert e.value.code == dp.ERR["TypeMismatch"]


def test_value_filter_optimizes_like_the_reference():
    """from_memory -> map(affine) -> filter(keep_even/odd) [-> shuffle] ->
    batch: Optimize rewrites it to the same node chain as the compiled
    reference (golden value_filters: map_filter_fusion, then no map_batch
    fusion because of the fused predicate)."""
    import json, os
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))["value_filters"]
    for c in golden:
        reg = dp.Registry()
        reg.register_standard_predicates()
        f = reg.register_affine(f"affine({c['a']},{c['b']})", c["a"], c["b"])
        g = dp.Dataset.from_memory(reg, range(c["n"])).map(f).filter("keep_odd" if c["odd"] else "keep_even")
        if c["shuffle"]:
            g = g.shuffle(c["shuffle"], 42)
        g = g.batch(64)
        if c["optimize"]:
            g = g.optimize()[0]
        chain = "<-".join(line.split()[0] for line in str(g).splitlines())
        assert chain == c["graph"], (chain, c)


def test_value_filter_validation():
    reg = dp.Registry()
    with pytest.raises(DpError) as e:
        reg.register_value_filter("bad", [("mod_eq", 0, 0)])
    assert e.value.code == dp.ERR["InvalidAttr"]
    with pytest.raises(DpError) as e:
        reg.register_value_filter("many", [("lt", 5)] * 9)
    assert e.value.code == dp.ERR["InvalidAttr"]


def test_pipeline_spec_parses_like_the_builders():
    """ParsePipelineSpec (the reference's stanza grammar over the device UDF
    library) builds the same graph as the ops:: builders, with the trailers."""
    reg = dp.Registry()
    g, info = dp.Dataset.from_spec(reg, """
        # cfg1 as text
        source range count=1000000
        map affine a=3 b=1 parallel=AUTO
        filter keep=even
        shuffle buffer=100 seed=42
        batch size=1024 drop_remainder=true
        prefetch buffer=AUTO
        options seed=7 deterministic=false
        epochs 3
        disable rule=map_batch_fusion
    """)
    reg2 = dp.Registry()
    reg2.register_affine("affine(3,1)", 3, 1)
    reg2.register_standard_predicates()
    want = (dp.Dataset.range(reg2, 1000000).map("affine(3,1)", -1).filter("keep_even").shuffle(100, 42)
            .batch(1024, drop_remainder=True).prefetch(-1))
    assert str(g) == str(want) and g.fingerprint() == want.fingerprint()
    assert info == {"epochs": 3, "seed": 7, "deterministic": False, "disabled_rules": ["map_batch_fusion"]}


def test_pipeline_spec_errors_carry_line_and_column():
    reg = dp.Registry()
    cases = [("map affine a=1", "line 1, col 1: 'map' before a source stanza"),
             ("source range count=5\nfrob x=1", "line 2, col 1: unknown stanza 'frob'"),
             ("source range count=5\nbatch size=x", "line 2, col 7: 'size' must be an integer"),
             ("source range count=5\nbatch size=4 speed=9", "line 2, col 14: batch: unknown argument 'speed'"),
             ("source range count=5\nsource range count=6", "line 2, col 1: multiple source stanzas"),
             ("source range count=5\nbatch size=0", "line 2, col 1: "),
             ("epochs 3", "no source stanza")]
    for text, msg in cases:
        with pytest.raises(DpError) as e:
            dp.Dataset.from_spec(reg, text)
        assert e.value.code == dp.ERR["ParseError"], (text, str(e.value))
        assert msg in str(e.value), (text, str(e.value))


def test_image_chain_kernel_choice_without_gpu():
    """dp_image_chain_kernel: resize chains (periodic column maps, or any
    other with runtime taps) run on K10 (k_roll.cu), the rest on K9; pure
    host logic."""
    mean, std = (123.675, 116.28, 103.53), (58.395, 57.12, 57.375)

    def kern(steps, h, w):
        c = _capi.ImageChain.from_steps(steps, h, w)
        k = ctypes.c_int()
        _capi.check(_capi.lib().dp_image_chain_kernel(ctypes.byref(c), ctypes.byref(k)))
        return k.value

    assert kern([("random_crop", 160, 160, 7, True), ("resize", 224, 224), ("normalize", mean, std)], 256, 256) == 10
    assert kern([("resize", 256, 256), ("center_crop", 224, 224), ("normalize", mean, std)], 320, 320) == 10
    assert kern([("resize", 224, 224), ("normalize", mean, std)], 320, 320) == 10
    assert kern([("random_crop", 28, 28, 3, True), ("resize", 24, 24)], 48, 48) == 10  # 7:6: runtime taps
    assert kern([("normalize", mean, std), ("resize", 24, 24)], 48, 48) == 9           # pixel op before the resize
    assert kern([("random_crop", 24, 24, 3, True), ("normalize", mean, std)], 48, 48) == 9  # no resize
    assert kern([("random_crop", 24, 24, 3, True)], 48, 48) == 9


def test_bench_e2e_consumer_builds_against_the_c_abi():
    """tools/e2e_consumer.c (bench.py's token e2e loop) is plain C over
    include/dpcuda_pipeline.h and links against libdpcuda.so."""
    import __graft_entry__
    import os
    __graft_entry__._build_e2e_consumer()
    path = os.path.join(os.path.dirname(_capi.LIB_PATH), "..", "..", "tools", "bin", "libdpe2e.so")
    lib = ctypes.CDLL(os.path.abspath(path))
    assert hasattr(lib, "dpe2e_consume_host_batches")
