"""ctypes binding of the C ABI in include/dpcuda.h / include/dpcuda_pipeline.h.

This is the binding a Python caller of the reference's operator API would add
(INTEGRATION.md shows the same stub).  The shared library is built in-tree by
``__graft_entry__.build()`` into ``paper_2101_12127_b200/lib/libdpcuda.so``;
there is no fallback: if it is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DP_LIB_PATH") or os.path.join(_HERE, "lib", "libdpcuda.so")
INCLUDE_DIR = os.path.join(os.path.dirname(_HERE), "include")

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
c_size = ctypes.c_size_t
c_fp = ctypes.POINTER(ctypes.c_float)

# name -> (restype, argtypes)
_SIGS = {
    "dp_last_error": (ctypes.c_char_p, []),
    "dp_build_info": (ctypes.c_char_p, []),
    "dp_device_count": (c_int, [ctypes.POINTER(c_int)]),
    "dp_k_range_affine_batch": (c_int, [c_i64, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "dp_k_shuffle_plan_scratch_bytes": (c_size, [c_u64, c_u64]),
    "dp_k_shuffle_plan": (c_int, [c_u64, c_u64, c_u64, c_vp, c_vp, c_vp, c_vp]),
    "dp_k_crop_flip_normalize_batch": (c_int, [c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_i64, c_u64, c_int, c_int,
                                               c_int, c_fp, c_fp, c_vp, c_vp, c_vp]),
    "dp_k_resize_normalize_batch": (c_int, [c_vp, c_i64, c_int, c_int, c_vp, c_i64, c_i64, c_int, c_int, c_fp, c_fp,
                                            c_vp, c_vp, c_vp]),
    "dp_k_filter_scratch_bytes": (c_size, [c_i64]),
    "dp_k_filter_len_le": (c_int, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dp_k_batch_max_len": (c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "dp_k_padded_batch": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "dp_k_shard_interleave_count": (c_i64, [c_i64, c_i64, c_i64, c_i64]),
    "dp_k_shard_interleave_index": (c_int, [c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "dp_k_shard_index": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "dp_k_order_digest": (c_int, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "dp_k_word_digest": (c_int, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "dp_k_synth_images": (c_int, [c_vp, c_u64, c_u64, c_u64, c_u64, c_vp]),
    "dp_k_synth_tokens": (c_int, [c_vp, c_vp, c_i64, c_u64, c_vp]),
    "dp_k_image_chain_batch": (c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "dp_image_chain_kernel": (c_int, [c_vp, ctypes.POINTER(c_int)]),
    "dp_fast_div_proven": (c_int, [c_fp, c_fp, ctypes.POINTER(c_int)]),
}


class DpError(RuntimeError):
    """A non-zero dp_status; ``code`` mirrors datapipe::ErrorCode + 1."""

    def __init__(self, code: int, message: str):
        super().__init__(f"dp_status {code}: {message}")
        self.code = code


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise DpError(status, lib().dp_last_error().decode())


def declared_symbols() -> list[str]:
    """Every dp_* function declared in include/*.h."""
    names = []
    for fn in sorted(os.listdir(INCLUDE_DIR)):
        if fn.endswith(".h"):
            with open(os.path.join(INCLUDE_DIR, fn)) as f:
                text = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
            names += re.findall(r"\b(dp_\w+)\s*\(", text)
    return sorted(set(names))


class ImageChain(ctypes.Structure):
    """dp_image_chain (include/dpcuda.h): [crop A][pixel ops][resize][crop B][pixel ops]."""
    _fields_ = [("in_h", c_int), ("in_w", c_int),
                ("pre_mode", c_int), ("pre_h", c_int), ("pre_w", c_int), ("pre_flip", c_int), ("pre_seed", c_u64),
                ("resize", c_int), ("rs_h", c_int), ("rs_w", c_int),
                ("post_mode", c_int), ("post_h", c_int), ("post_w", c_int), ("post_flip", c_int),
                ("post_seed", c_u64),
                ("num_pre_ops", c_int), ("num_post_ops", c_int), ("op_kind", c_int * 4),
                ("op_a", (ctypes.c_float * 3) * 4), ("op_b", (ctypes.c_float * 3) * 4), ("out_f32", c_int)]

    @classmethod
    def from_steps(cls, steps, in_h, in_w):
        """The descriptor of a chain given as oracle steps (tests/oracle_lib.steps_array's tuples), the
        way the engine lowers map chains (csrc/engine/lowering.cpp LowerImageChain)."""
        c = cls()
        c.in_h, c.in_w = in_h, in_w
        nops = 0
        for st in steps:
            kind = st[0]
            if kind in ("random_crop", "center_crop"):
                mode = 1 if kind == "random_crop" else 2
                if not c.resize and not c.pre_mode:
                    c.pre_mode, c.pre_h, c.pre_w = mode, st[1], st[2]
                    if mode == 1:
                        c.pre_seed, c.pre_flip = st[3], int(st[4])
                else:
                    c.post_mode, c.post_h, c.post_w = mode, st[1], st[2]
                    if mode == 1:
                        c.post_seed, c.post_flip = st[3], int(st[4])
            elif kind == "resize":
                c.resize, c.rs_h, c.rs_w = 1, st[1], st[2]
            else:
                a, b = ((0, 0, 0), (1, 1, 1)) if kind == "cast" else (st[1], st[2])
                c.op_kind[nops] = 1 if kind == "affine" else 0
                c.op_a[nops][:] = [float(x) for x in a]
                c.op_b[nops][:] = [float(x) for x in b]
                if c.resize:
                    c.num_post_ops += 1
                else:
                    c.num_pre_ops += 1
                nops += 1
        c.out_f32 = 1 if (c.resize or nops) else 0
        return c


def floats3(vals) -> ctypes.Array:
    return (ctypes.c_float * 3)(*[float(v) for v in vals])
