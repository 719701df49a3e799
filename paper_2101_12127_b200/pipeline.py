"""Python binding of the Dataset / Iterator operator API (include/dpcuda_pipeline.h).

Mirrors the reference's C++ operator API (/root/reference/proj/include/
datapipe/{graph,udf,optimizer,runtime}.hpp): ``Registry`` is UdfRegistry,
``Dataset`` wraps DatasetGraph and its methods are the ops:: builders,
``optimize`` is Optimize, ``make_iterator`` is MakeIterator and
``Iterator.get_next`` is PipelineIterator::GetNext (None at the sticky end).
Errors raise ``DpError`` whose ``code`` is datapipe::ErrorCode + 1.

Every call goes through libdpcuda.so; there is no Python or CPU compute path.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._capi import DpError, lib

c_i64, c_u64, c_int, c_vp, c_size = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t
PP = ctypes.POINTER(c_vp)

ERR = {  # dp_status values (include/dpcuda.h)
    "ParseError": 18, "InvalidArity": 1, "InvalidAttr": 2, "TypeMismatch": 3, "MalformedInput": 4, "ValidationFailed": 5,
    "DuplicateName": 6, "UnknownUdf": 7, "MissingFile": 8, "FingerprintMismatch": 10, "VersionMismatch": 11,
    "CorruptBlob": 12, "RewriteDiverged": 14, "Internal": 19, "Cuda": 100, "OutOfMemory": 101,
    "EndOfSequence": 102,
}
DTYPES = {0: np.uint8, 1: np.int32, 2: np.int64, 3: np.float32}
MEAN = (123.675, 116.28, 103.53)
STD = (58.395, 57.12, 57.375)


class dp_tensor(ctypes.Structure):
    _fields_ = [("dtype", c_int), ("ndim", c_int), ("shape", c_i64 * 6), ("data", c_vp), ("on_host", c_int)]


class dp_batch(ctypes.Structure):
    _fields_ = [("handle", c_vp), ("num_components", c_int), ("components", dp_tensor * 4), ("ready_event", c_vp),
                ("index", c_i64)]


class dp_iterator_options(ctypes.Structure):
    _fields_ = [("deterministic", c_int), ("has_seed_override", c_int), ("seed_override", c_u64), ("device", c_int),
                ("consumer_stream", c_vp), ("host_output", c_int), ("slot_memory_budget", c_u64),
                ("max_launch_bytes", c_u64), ("launch_batches", c_i64),
                ("first_launch_batches", c_i64)]


class dp_iterator_stats(ctypes.Structure):
    _fields_ = [("live_plans", c_i64), ("slots", c_i64), ("slot_bytes", c_i64), ("prefetch_depth", c_i64),
                ("group_batches", c_i64), ("max_depth", c_i64), ("producer_groups_per_s", ctypes.c_double),
                ("consumer_groups_per_s", ctypes.c_double), ("p_empty", ctypes.c_double)]


class dp_node_metrics(ctypes.Structure):
    _fields_ = [("path", ctypes.c_char * 192), ("label", ctypes.c_char * 96), ("self_time_ns", c_i64),
                ("elements_produced", c_i64)]


_SIGS = {
    "dp_registry_create": [PP], "dp_registry_destroy": [c_vp],
    "dp_registry_register_affine": [c_vp, ctypes.c_char_p, c_i64, c_i64],
    "dp_registry_register_random_crop_flip": [c_vp, ctypes.c_char_p, c_i64, c_i64, c_u64, c_int],
    "dp_registry_register_resize_bilinear": [c_vp, ctypes.c_char_p, c_i64, c_i64],
    "dp_registry_register_normalize": [c_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_float),
                                       ctypes.POINTER(ctypes.c_float)],
    "dp_registry_register_length_filter": [c_vp, ctypes.c_char_p, c_i64],
    "dp_registry_register_cast": [c_vp, ctypes.c_char_p],
    "dp_registry_register_record_reader": [c_vp, ctypes.c_char_p, c_i64],
    "dp_registry_register_value_filter": [c_vp, ctypes.c_char_p, c_vp, c_int],
    "dp_registry_register_standard_predicates": [c_vp],
    "dp_registry_register_decode_raw": [c_vp, ctypes.c_char_p, c_i64, c_i64],
    "dp_registry_contains": [c_vp, ctypes.c_char_p],
    "dp_source_synthetic_images": [c_i64, c_i64, c_i64, c_u64, c_int, PP],
    "dp_source_images_from_host": [c_vp, c_i64, c_i64, c_i64, c_int, PP],
    "dp_source_synthetic_images_sharded": [c_i64, c_i64, c_i64, c_u64, c_i64, c_i64, c_int, PP],
    "dp_source_images_pinned_host": [c_vp, c_i64, c_i64, c_i64, c_int, PP],
    "dp_source_synthetic_tokens": [c_i64, ctypes.c_uint32, c_u64, c_u64, c_int, PP],
    "dp_source_tokens_from_host": [c_vp, c_i64, c_vp, c_int, PP],
    "dp_source_tokens_pinned_host": [c_vp, c_i64, c_vp, c_int, PP],
    "dp_source_records_from_files": [ctypes.POINTER(ctypes.c_char_p), c_i64, c_int, PP],
    "dp_source_records_from_files_sharded": [ctypes.POINTER(ctypes.c_char_p), c_i64, c_i64, c_i64, c_int, PP],
    "dp_source_as_shard": [c_vp, c_i64, c_i64, c_i64, c_i64, PP],
    "dp_source_with_labels": [c_vp, c_vp, c_i64, PP],
    "dp_registry_register_center_crop": [c_vp, ctypes.c_char_p, c_i64, c_i64],
    "dp_registry_register_image_affine": [c_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_float),
                                          ctypes.POINTER(ctypes.c_float)],
    "dp_source_synthetic_records_sharded": [c_i64, c_i64, c_i64, c_i64, c_u64, c_i64, c_i64, c_int, PP],
    "dp_source_release": [c_vp],
    "dp_graph_range": [c_vp, c_i64, PP],
    "dp_graph_from_memory_i64": [c_vp, c_vp, c_i64, c_int, PP],
    "dp_graph_tensor_slices": [c_vp, c_vp, PP],
    "dp_graph_from_file": [c_vp, ctypes.POINTER(ctypes.c_char_p), c_i64, c_int, PP],
    "dp_write_record_file": [ctypes.c_char_p, c_vp, c_vp, c_i64],
    "dp_graph_token_sequences": [c_vp, c_vp, PP],
    "dp_graph_map": [c_vp, ctypes.c_char_p, c_i64, c_vp, PP],
    "dp_graph_filter": [c_vp, ctypes.c_char_p, c_vp, PP],
    "dp_graph_interleave": [c_vp, ctypes.c_char_p, c_i64, c_i64, c_vp, c_vp, PP],
    "dp_graph_batch": [c_vp, c_i64, c_int, c_vp, PP],
    "dp_graph_padded_batch": [c_vp, c_i64, c_i64, c_int, c_vp, PP],
    "dp_graph_bucket_by_length": [c_vp, c_vp, c_i64, c_vp, c_i64, c_int, c_vp, PP],
    "dp_graph_prefetch": [c_vp, c_i64, c_vp, PP],
    "dp_graph_repeat": [c_vp, c_i64, c_vp, PP],
    "dp_graph_shuffle": [c_vp, c_i64, c_int, c_u64, c_vp, PP],
    "dp_graph_shard": [c_vp, c_i64, c_i64, c_vp, PP],
    "dp_graph_optimize": [c_vp, c_vp, ctypes.c_char_p, PP, ctypes.c_char_p, c_size],
    "dp_graph_root_kind": [c_vp, ctypes.c_char_p, c_size],
    "dp_graph_to_string": [c_vp, ctypes.c_char_p, c_size],
    "dp_graph_serialize": [c_vp, c_vp, c_size, ctypes.POINTER(c_size)],
    "dp_graph_deserialize": [c_vp, c_vp, c_size, c_vp, c_i64, c_int, PP],
    "dp_graph_fingerprint": [c_vp, c_vp],
    "dp_graph_from_spec": [c_vp, ctypes.c_char_p, c_int, PP, ctypes.POINTER(c_int), ctypes.POINTER(c_int),
                           ctypes.POINTER(c_u64), ctypes.POINTER(c_int), ctypes.c_char_p, c_size],
    "dp_graph_release": [c_vp],
    "dp_iterator_options_default": [ctypes.POINTER(dp_iterator_options)],
    "dp_iterator_create": [c_vp, c_vp, ctypes.POINTER(dp_iterator_options), PP],
    "dp_iterator_get_next": [c_vp, ctypes.POINTER(dp_batch)],
    "dp_batch_release": [ctypes.POINTER(dp_batch)],
    "dp_batch_wait": [ctypes.POINTER(dp_batch)],
    "dp_iterator_skip": [c_vp, c_i64, ctypes.POINTER(c_i64)],
    "dp_iterator_save": [c_vp, c_vp, c_size, ctypes.POINTER(c_size)],
    "dp_iterator_restore": [c_vp, c_vp, ctypes.c_char_p, c_size, ctypes.POINTER(dp_iterator_options), PP],
    "dp_tensor_copy_to_host": [ctypes.POINTER(dp_batch), c_int, c_vp, c_size],
    "dp_iterator_stream": [c_vp], "dp_iterator_kernel_launches": [c_vp], "dp_iterator_prefetch_depth": [c_vp],
    "dp_iterator_batch_stage_timing": [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)],
    "dp_iterator_batches_launched": [c_vp], "dp_iterator_get_stats": [c_vp, ctypes.POINTER(dp_iterator_stats)],
    "dp_iterator_metrics": [c_vp, ctypes.POINTER(dp_node_metrics), c_int, ctypes.POINTER(c_int)],
    "dp_iterator_root_delivered": [c_vp], "dp_iterator_base_seed": [c_vp],
    "dp_iterator_describe": [c_vp, ctypes.c_char_p, c_size], "dp_iterator_destroy": [c_vp],
}
_RES = {"dp_registry_destroy": None, "dp_source_release": None, "dp_graph_release": None,
        "dp_iterator_options_default": None, "dp_iterator_destroy": None, "dp_iterator_stream": c_vp,
        "dp_iterator_kernel_launches": c_i64, "dp_iterator_prefetch_depth": c_i64,
        "dp_iterator_root_delivered": c_i64, "dp_iterator_base_seed": c_u64, "dp_iterator_batches_launched": c_i64}

_bound = None


def L():
    global _bound
    if _bound is None:
        l = lib()
        for name, args in _SIGS.items():
            f = getattr(l, name)
            f.argtypes = args
            f.restype = _RES.get(name, c_int)
        _bound = l
    return _bound


def _check(st):
    if st != 0:
        raise DpError(st, lib().dp_last_error().decode())


def _release(obj, fn):
    h = getattr(obj, "h", None)
    obj.h = None
    if h and _bound is not None:
        try:
            getattr(_bound, fn)(h)
        except Exception:  # interpreter shutdown
            pass


def _b(s: str) -> bytes:
    return s.encode()


class Registry:
    """UdfRegistry (udf.hpp:41-87) holding device UDF descriptors."""

    def __init__(self):
        h = c_vp()
        _check(L().dp_registry_create(ctypes.byref(h)))
        self.h = h

    def __del__(self, _rel=_release):
        _rel(self, "dp_registry_destroy")

    def register_affine(self, name, a, b):
        _check(L().dp_registry_register_affine(self.h, _b(name), a, b))
        return name

    def register_random_crop_flip(self, name, crop_h=224, crop_w=224, seed=7, flip=True):
        _check(L().dp_registry_register_random_crop_flip(self.h, _b(name), crop_h, crop_w, seed, int(flip)))
        return name

    def register_resize_bilinear(self, name, out_h=224, out_w=224):
        _check(L().dp_registry_register_resize_bilinear(self.h, _b(name), out_h, out_w))
        return name

    def register_cast(self, name):
        """u8 image -> fp32 values, exact (normalize with mean 0, std 1)."""
        _check(L().dp_registry_register_cast(self.h, _b(name)))
        return name

    def register_center_crop(self, name, crop_h, crop_w):
        _check(L().dp_registry_register_center_crop(self.h, _b(name), crop_h, crop_w))
        return name

    def register_image_affine(self, name, scale, shift):
        """x * scale[c] + shift[c] per channel -> fp32."""
        _check(L().dp_registry_register_image_affine(self.h, _b(name), (ctypes.c_float * 3)(*map(float, scale)),
                                                     (ctypes.c_float * 3)(*map(float, shift))))
        return name

    def register_normalize(self, name, mean=MEAN, std=STD):
        m = (ctypes.c_float * 3)(*mean)
        s = (ctypes.c_float * 3)(*std)
        _check(L().dp_registry_register_normalize(self.h, _b(name), m, s))
        return name

    def register_length_filter(self, name, max_len):
        _check(L().dp_registry_register_length_filter(self.h, _b(name), max_len))
        return name

    PRED = {"le": 0, "ge": 1, "lt": 2, "mod_eq": 3, "mod_ne": 4}

    def register_value_filter(self, name, terms):
        """Predicate on int64 element values: [("mod_eq", 2, 0), ("lt", 100), ...], all must hold."""
        class Term(ctypes.Structure):
            _fields_ = [("op", c_int), ("a", c_i64), ("b", c_i64)]
        arr = (Term * max(1, len(terms)))(*[Term(self.PRED[t[0]], t[1], t[2] if len(t) > 2 else 0) for t in terms])
        _check(L().dp_registry_register_value_filter(self.h, _b(name), ctypes.cast(arr, c_vp), len(terms)))
        return name

    def register_standard_predicates(self):
        """keep_even / keep_odd / keep_all, as the reference's pipeline_spec registers them."""
        _check(L().dp_registry_register_standard_predicates(self.h))

    def register_record_reader(self, name, records):
        _check(L().dp_registry_register_record_reader(self.h, _b(name), records))
        return name

    def register_decode_raw(self, name, h, w):
        _check(L().dp_registry_register_decode_raw(self.h, _b(name), h, w))
        return name

    def contains(self, name):
        return bool(L().dp_registry_contains(self.h, _b(name)))


class Source:
    """Device-resident (or pinned-host) element data for the source kinds."""

    def __init__(self, h, keepalive=None):
        self.h = h
        self._keep = keepalive

    def __del__(self, _rel=_release):
        _rel(self, "dp_source_release")

    @staticmethod
    def records_from_files(paths, device=0, num_shards=1, index=0):
        """Record files read into device memory: the records of an interleave
        over files.  num_shards > 1 reads only the files f % num_shards ==
        index (graphs apply .shard(num_shards, index) to the interleave's
        inputs)."""
        arr = (ctypes.c_char_p * max(1, len(paths)))(*[os.fsencode(p) for p in paths])
        out = c_vp()
        _check(L().dp_source_records_from_files_sharded(arr, len(paths), num_shards, index, device,
                                                        ctypes.byref(out)))
        return Source(out)

    def as_shard(self, global_count, num_shards, index, block=1):
        """A view of this source holding shard `index` of `num_shards` of a
        `global_count`-element dataset, in blocks of `block` positions."""
        out = c_vp()
        _check(L().dp_source_as_shard(self.h, global_count, num_shards, index, block, ctypes.byref(out)))
        return Source(out, self)

    @staticmethod
    def synthetic_records_sharded(num_files, records_per_file, h, w, num_shards=1, index=0, seed=0x5EED, device=0):
        """Interleave records: `num_files` inputs of `records_per_file` images
        (record r of file x = image id x * R + r); holds only the files
        x % num_shards == index."""
        out = c_vp()
        _check(L().dp_source_synthetic_records_sharded(num_files, records_per_file, h, w, seed, num_shards, index,
                                                       device, ctypes.byref(out)))
        return Source(out)

    @staticmethod
    def synthetic_images(count, h, w, seed=0x5EED, device=0):
        out = c_vp()
        _check(L().dp_source_synthetic_images(count, h, w, seed, device, ctypes.byref(out)))
        return Source(out)

    @staticmethod
    def synthetic_images_sharded(global_count, h, w, num_shards, index, seed=0x5EED, device=0):
        """Holds only shard `index` of `num_shards` (one process per GPU);
        graphs over it must start with .shard(num_shards, index)."""
        out = c_vp()
        _check(L().dp_source_synthetic_images_sharded(global_count, h, w, seed, num_shards, index, device,
                                                      ctypes.byref(out)))
        return Source(out)

    def with_labels(self, labels):
        """This image source with an int64 label per row: elements (id, image, label)."""
        labels = np.ascontiguousarray(labels, np.int64)
        out = c_vp()
        _check(L().dp_source_with_labels(self.h, labels.ctypes.data if labels.size else None, labels.size,
                                         ctypes.byref(out)))
        return Source(out, keepalive=self)

    @staticmethod
    def images_from_host(arr: np.ndarray, device=0):
        arr = np.ascontiguousarray(arr, np.uint8)
        out = c_vp()
        _check(L().dp_source_images_from_host(arr.ctypes.data, arr.shape[0], arr.shape[1], arr.shape[2], device,
                                              ctypes.byref(out)))
        return Source(out)

    @staticmethod
    def images_pinned_host(arr: np.ndarray, device=0):
        """`arr` must stay alive; it is page-locked in place and read over PCIe."""
        assert arr.dtype == np.uint8 and arr.flags["C_CONTIGUOUS"]
        out = c_vp()
        _check(L().dp_source_images_pinned_host(arr.ctypes.data, arr.shape[0], arr.shape[1], arr.shape[2], device,
                                                ctypes.byref(out)))
        return Source(out, keepalive=arr)

    @staticmethod
    def synthetic_tokens(count, max_len=1024, len_seed=4, tok_seed=4, device=0):
        out = c_vp()
        _check(L().dp_source_synthetic_tokens(count, max_len, len_seed, tok_seed, device, ctypes.byref(out)))
        return Source(out)

    @staticmethod
    def tokens_from_host(lengths, tokens, device=0, pinned=False):
        """Token sequences (lengths + concatenated tokens) copied to the device,
        or (pinned=True) into pinned host memory the kernels read over PCIe."""
        lengths = np.ascontiguousarray(lengths, np.int32)
        tokens = np.ascontiguousarray(tokens, np.int32)
        if tokens.size != int(lengths.astype(np.int64).sum()):
            raise DpError(2, f"token sequences: {tokens.size} tokens but the lengths sum to "
                          f"{int(lengths.astype(np.int64).sum())}")
        out = c_vp()
        fn = L().dp_source_tokens_pinned_host if pinned else L().dp_source_tokens_from_host
        _check(fn(lengths.ctypes.data, lengths.size, tokens.ctypes.data if tokens.size else None, device,
                  ctypes.byref(out)))
        return Source(out)


class Dataset:
    """DatasetGraph + the ops:: builders (graph.hpp:134-165)."""

    def __init__(self, h, reg: Registry, keep=()):
        self.h = h
        self.reg = reg
        self._keep = keep  # sources referenced by the graph stay alive with it

    def __del__(self, _rel=_release):
        _rel(self, "dp_graph_release")

    def _emit(self, fn, *args, keep=()):
        out = c_vp()
        _check(fn(*args, ctypes.byref(out)))
        return Dataset(out, self.reg, tuple(self._keep) + tuple(keep))

    # sources
    @staticmethod
    def range(reg, n):
        out = c_vp()
        _check(L().dp_graph_range(reg.h, n, ctypes.byref(out)))
        return Dataset(out, reg)

    @staticmethod
    def from_memory(reg, values, device=0):
        v = np.ascontiguousarray(values, np.int64)
        out = c_vp()
        _check(L().dp_graph_from_memory_i64(reg.h, v.ctypes.data if v.size else None, v.size, device,
                                            ctypes.byref(out)))
        return Dataset(out, reg)

    @staticmethod
    def tensor_slices(reg, src: Source):
        out = c_vp()
        _check(L().dp_graph_tensor_slices(reg.h, src.h, ctypes.byref(out)))
        return Dataset(out, reg, (src,))

    @staticmethod
    def from_file(reg, paths, device=0):
        """ops::FromFile (graph.hpp:137): length-prefixed record files read in order."""
        if isinstance(paths, (str, bytes, os.PathLike)):
            paths = [paths]
        arr = (ctypes.c_char_p * max(1, len(paths)))(*[os.fsencode(p) for p in paths])
        out = c_vp()
        _check(L().dp_graph_from_file(reg.h, arr, len(paths), device, ctypes.byref(out)))
        return Dataset(out, reg)

    @staticmethod
    def token_sequences(reg, src: Source):
        out = c_vp()
        _check(L().dp_graph_token_sequences(reg.h, src.h, ctypes.byref(out)))
        return Dataset(out, reg, (src,))

    # transformations
    def map(self, udf, num_parallel_calls=1):
        return self._emit(L().dp_graph_map, self.h, _b(udf), num_parallel_calls, self.reg.h)

    def filter(self, udf):
        return self._emit(L().dp_graph_filter, self.h, _b(udf), self.reg.h)

    def interleave(self, udf, cycle_length, num_parallel_calls=1, records: Source = None):
        return self._emit(L().dp_graph_interleave, self.h, _b(udf), cycle_length, num_parallel_calls,
                          records.h if records else None, self.reg.h, keep=(records,) if records else ())

    def batch(self, batch_size, drop_remainder=False):
        return self._emit(L().dp_graph_batch, self.h, batch_size, int(drop_remainder), self.reg.h)

    def padded_batch(self, batch_size, padding_value=0, drop_remainder=False):
        return self._emit(L().dp_graph_padded_batch, self.h, batch_size, padding_value, int(drop_remainder),
                          self.reg.h)

    def bucket_by_length(self, boundaries, batch_sizes, padding_value=0, drop_remainder=False):
        """tf.data bucket_by_sequence_length over token sequences (K8)."""
        b = np.ascontiguousarray(boundaries, np.int64)
        s = np.ascontiguousarray(batch_sizes, np.int64)
        if s.size != b.size + 1:
            raise ValueError("batch_sizes needs len(boundaries) + 1 entries")
        return self._emit(L().dp_graph_bucket_by_length, self.h, b.ctypes.data if b.size else None, b.size,
                          s.ctypes.data, padding_value, int(drop_remainder), self.reg.h)

    def prefetch(self, buffer_size):
        return self._emit(L().dp_graph_prefetch, self.h, buffer_size, self.reg.h)

    def repeat(self, count):
        return self._emit(L().dp_graph_repeat, self.h, count, self.reg.h)

    def shuffle(self, buffer_size, seed=None):
        return self._emit(L().dp_graph_shuffle, self.h, buffer_size, 0 if seed is None else 1, seed or 0,
                          self.reg.h)

    def shard(self, num_shards, index):
        return self._emit(L().dp_graph_shard, self.h, num_shards, index, self.reg.h)

    def optimize(self, disabled_rules=()):
        """Optimize(graph, RuleSet::Default() minus disabled) -> (Dataset, report)."""
        out = c_vp()
        rep = ctypes.create_string_buffer(8192)
        _check(L().dp_graph_optimize(self.h, self.reg.h, _b(",".join(disabled_rules)), ctypes.byref(out), rep,
                                     len(rep)))
        return Dataset(out, self.reg, self._keep), rep.value.decode()

    def serialize(self) -> bytes:
        """Serialize (DPG1, formats.md): the reference's bytes for graphs both engines express."""
        n = c_size()
        _check(L().dp_graph_serialize(self.h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(max(1, n.value))
        _check(L().dp_graph_serialize(self.h, buf, n.value, ctypes.byref(n)))
        return buf.raw[: n.value]

    @staticmethod
    def deserialize(reg, data: bytes, sources=(), device=0):
        arr = (c_vp * max(1, len(sources)))(*[s.h for s in sources])
        out = c_vp()
        buf = ctypes.create_string_buffer(bytes(data), len(data))
        _check(L().dp_graph_deserialize(reg.h, buf, len(data), arr, len(sources), device, ctypes.byref(out)))
        return Dataset(out, reg, tuple(sources))

    @staticmethod
    def from_spec(reg, text, device=0):
        """ParsePipelineSpec: (Dataset, {"epochs", "seed", "deterministic", "disabled_rules"})."""
        out = c_vp()
        ep, hs, det = c_int(), c_int(), c_int()
        seed = c_u64()
        buf = ctypes.create_string_buffer(4096)
        _check(L().dp_graph_from_spec(reg.h, _b(text), device, ctypes.byref(out), ctypes.byref(ep), ctypes.byref(hs),
                                      ctypes.byref(seed), ctypes.byref(det), buf, len(buf)))
        rules = [r for r in buf.value.decode().split(",") if r]
        return Dataset(out, reg), {"epochs": ep.value, "seed": seed.value if hs.value else None,
                                   "deterministic": bool(det.value), "disabled_rules": rules}

    def fingerprint(self) -> str:
        """GraphFingerprint: SHA-256 of the seed-zeroed serialization (hex)."""
        buf = ctypes.create_string_buffer(65)
        _check(L().dp_graph_fingerprint(self.h, buf))
        return buf.value.decode()

    @property
    def root_kind(self):
        buf = ctypes.create_string_buffer(64)
        _check(L().dp_graph_root_kind(self.h, buf, len(buf)))
        return buf.value.decode()

    def __str__(self):
        buf = ctypes.create_string_buffer(1 << 16)
        _check(L().dp_graph_to_string(self.h, buf, len(buf)))
        return buf.value.decode()


class Batch:
    """One element returned by GetNext: device (or pinned host) tensors."""

    def __init__(self, b: dp_batch, it):
        self.b = b
        self._it = it

    @property
    def components(self):
        out = []
        for c in range(self.b.num_components):
            t = self.b.components[c]
            out.append((DTYPES[t.dtype], tuple(t.shape[k] for k in range(t.ndim)), t.data, bool(t.on_host)))
        return out

    def numpy(self, c):
        dt, shape, _, _ = self.components[c]
        arr = np.empty(shape, dt)
        _check(L().dp_tensor_copy_to_host(ctypes.byref(self.b), c, arr.ctypes.data, arr.nbytes))
        return arr

    def torch(self, c):
        """Zero-copy torch view of a device component (valid until release;
        ready on the iterator's consumer_stream)."""
        import torch
        dt, shape, ptr, on_host = self.components[c]
        assert not on_host, "torch() views device components"

        class _View:
            __cuda_array_interface__ = {"shape": shape, "typestr": np.dtype(dt).str, "data": (ptr, False),
                                        "version": 2, "strides": None}
        return torch.as_tensor(_View(), device="cuda")

    def wait(self):
        """Host-blocking wait until the batch is written (and copied, with host_output)."""
        _check(L().dp_batch_wait(ctypes.byref(self.b)))
        return self

    def host_view(self, c):
        """Zero-copy numpy view of a host_output component (valid until release)."""
        dt, shape, ptr, on_host = self.components[c]
        assert on_host, "host_view needs make_iterator(..., host_output=True)"
        n = int(np.prod(shape)) * np.dtype(dt).itemsize
        buf = (ctypes.c_char * n).from_address(ptr)
        return np.frombuffer(buf, dtype=dt).reshape(shape)

    def release(self):
        if self.b.handle:
            L().dp_batch_release(ctypes.byref(self.b))

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class Iterator:
    """PipelineIterator (runtime.hpp:52-90)."""

    def __init__(self, h, ds):
        self.h = h
        self._ds = ds

    def __del__(self, _rel=_release):
        _rel(self, "dp_iterator_destroy")

    def get_next(self):
        b = dp_batch()
        st = L().dp_iterator_get_next(self.h, ctypes.byref(b))
        if st == ERR["EndOfSequence"]:
            return None
        _check(st)
        return Batch(b, self)

    def save(self) -> bytes:
        """Checkpoint blob (DPC1 layout)."""
        n = c_size()
        L().dp_iterator_save(self.h, None, 0, ctypes.byref(n))
        buf = ctypes.create_string_buffer(n.value)
        _check(L().dp_iterator_save(self.h, buf, n.value, ctypes.byref(n)))
        return buf.raw[:n.value]

    def skip(self, n):
        """GetNext n times in C++ dropping the batches; returns how many were delivered."""
        k = c_i64()
        _check(L().dp_iterator_skip(self.h, n, ctypes.byref(k)))
        return k.value

    def __iter__(self):
        while True:
            b = self.get_next()
            if b is None:
                return
            yield b

    @property
    def stream(self):
        return L().dp_iterator_stream(self.h)

    @property
    def kernel_launches(self):
        return L().dp_iterator_kernel_launches(self.h)

    def batch_stage_timing(self):
        """(total device ns, launches) of the fused batch-stage kernels so far."""
        ns, n = c_i64(), c_i64()
        _check(L().dp_iterator_batch_stage_timing(self.h, ctypes.byref(ns), ctypes.byref(n)))
        return ns.value, n.value

    @property
    def batches_launched(self):
        return L().dp_iterator_batches_launched(self.h)

    @property
    def prefetch_depth(self):
        return L().dp_iterator_prefetch_depth(self.h)

    def stats(self) -> dict:
        """dp_iterator_get_stats: live epoch plans, slots, slot bytes, depth, batches per launch."""
        st = dp_iterator_stats()
        _check(L().dp_iterator_get_stats(self.h, ctypes.byref(st)))
        return {f: (getattr(st, f) if t is ctypes.c_double else int(getattr(st, f)))
                for f, t in dp_iterator_stats._fields_}

    def metrics(self) -> list:
        """Metrics() (runtime.hpp:76): [(path, label, self_time_ns, elements_produced)] root first."""
        rows = (dp_node_metrics * 32)()
        n = c_int()
        _check(L().dp_iterator_metrics(self.h, rows, 32, ctypes.byref(n)))
        return [(r.path.decode(), r.label.decode(), int(r.self_time_ns), int(r.elements_produced))
                for r in rows[:min(n.value, 32)]]

    @property
    def root_delivered(self):
        return L().dp_iterator_root_delivered(self.h)

    @property
    def base_seed(self):
        return L().dp_iterator_base_seed(self.h)

    def describe(self):
        buf = ctypes.create_string_buffer(4096)
        _check(L().dp_iterator_describe(self.h, buf, len(buf)))
        return buf.value.decode()


def restore(ds: Dataset, blob: bytes, device=0, consumer_stream=None, host_output=False, launch_batches=0,
            first_launch_batches=0):
    """Restore(graph, registry, blob) (checkpoint.hpp:44-49): seeks, never replays."""
    o = dp_iterator_options()
    L().dp_iterator_options_default(ctypes.byref(o))
    o.device = device
    o.consumer_stream = consumer_stream
    o.host_output = int(host_output)
    o.launch_batches = launch_batches
    o.first_launch_batches = first_launch_batches
    out = c_vp()
    _check(L().dp_iterator_restore(ds.h, ds.reg.h, blob, len(blob), ctypes.byref(o), ctypes.byref(out)))
    return Iterator(out, ds)


def make_iterator(ds: Dataset, seed_override=None, device=0, consumer_stream=None, host_output=False,
                  slot_memory_budget=0, deterministic=True, max_launch_bytes=0, launch_batches=0,
                  first_launch_batches=0):
    """MakeIterator(graph, registry, IteratorOptions) (runtime.hpp:98-100)."""
    o = dp_iterator_options()
    L().dp_iterator_options_default(ctypes.byref(o))
    o.deterministic = int(deterministic)
    if seed_override is not None:
        o.has_seed_override = 1
        o.seed_override = seed_override
    o.device = device
    o.consumer_stream = consumer_stream
    o.host_output = int(host_output)
    o.slot_memory_budget = slot_memory_budget
    o.max_launch_bytes = max_launch_bytes
    o.launch_batches = launch_batches
    o.first_launch_batches = first_launch_batches
    out = c_vp()
    _check(L().dp_iterator_create(ds.h, ds.reg.h, ctypes.byref(o), ctypes.byref(out)))
    return Iterator(out, ds)


def write_record_file(path, payloads):
    """WriteRecordFile (runtime.hpp:102-107): [u32 LE length][payload] per record."""
    bufs = [bytes(p) for p in payloads]
    offs = np.zeros(len(bufs) + 1, np.int64)
    offs[1:] = np.cumsum([len(b) for b in bufs]) if bufs else []
    data = np.frombuffer(b"".join(bufs) or b"\0", np.uint8)
    _check(L().dp_write_record_file(os.fsencode(path), data.ctypes.data, offs.ctypes.data, len(bufs)))
