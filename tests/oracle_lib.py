"""numpy/ctypes front end of the TEST-ONLY checkers in oracle/.

Oracle     -- oracle/liboracle.so, the plain-C restatement (oracle/restate.c)
Reference  -- oracle/_ref/libdpref.so, the compiled reference library driven
              through its own operator API by oracle/ref_shim.cpp

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libdpref.so")

i64, u64, u32, i32, c_int = ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int
vp = ctypes.c_void_p

MEAN = (123.675, 116.28, 103.53)
STD = (58.395, 57.12, 57.375)
PIX_SEED = 0x5EED
UDF_SEED = 7


class orc_map_step(ctypes.Structure):
    _fields_ = [("op", c_int), ("h", c_int), ("w", c_int), ("flip", c_int), ("seed", u64),
                ("a", ctypes.c_float * 3), ("b", ctypes.c_float * 3)]


STEP = {"random_crop": 1, "center_crop": 2, "resize": 3, "normalize": 4, "affine": 5, "cast": 6}


def steps_array(steps):
    """[("random_crop", h, w, seed, flip) | ("center_crop", h, w) | ("resize", h, w) |
    ("normalize", mean3, std3) | ("affine", scale3, shift3) | ("cast",)] -> orc_map_step[]"""
    arr = (orc_map_step * max(len(steps), 1))()
    for i, st in enumerate(steps):
        o = arr[i]
        o.op = STEP[st[0]]
        if st[0] in ("random_crop", "center_crop", "resize"):
            o.h, o.w = st[1], st[2]
        if st[0] == "random_crop":
            o.seed, o.flip = st[3], int(st[4])
        if st[0] in ("normalize", "affine"):
            o.a[:] = [float(x) for x in st[1]]
            o.b[:] = [float(x) for x in st[2]]
    return arr


def P(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(vp)


class Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-C", ORACLE_DIR, "restate"], check=True, capture_output=True)
        L = ctypes.CDLL(ORACLE_SO)
        sig = {
            "orc_splitmix64_next": (u64, [ctypes.POINTER(u64)]),
            "orc_mix_seeds": (u64, [u64, u64]),
            "orc_shuffle_seed": (u64, [u64, c_int, u64]),
            "orc_shuffle_order": (None, [u64, u64, u64, vp]),
            "orc_digest_init": (u64, []),
            "orc_digest_i64": (u64, [u64, vp, ctypes.c_size_t]),
            "orc_digest_u32": (u64, [u64, vp, ctypes.c_size_t]),
            "orc_synth_images": (None, [u64, u64, u64, u64, vp]),
            "orc_synth_lengths": (None, [u64, u32, u64, vp]),
            "orc_synth_token": (i32, [u64, u64, u64]),
            "orc_philox4x32_10": (None, [vp, vp, vp]),
            "orc_crop_params": (None, [u64, i64, c_int, c_int, c_int, c_int, vp, vp, vp]),
            "orc_crop_flip_normalize": (None, [vp, c_int, c_int, i64, u64, c_int, c_int, c_int, vp]),
            "orc_resize_normalize": (None, [vp, c_int, c_int, c_int, c_int, vp]),
            "orc_filter_len_le": (u64, [vp, u64, i32, vp]),
            "orc_bucket_by_length": (i64, [vp, vp, i64, vp, c_int, vp, c_int, vp, vp]),
            "orc_shard_positions": (u64, [u64, u64, u64, vp]),
            "orc_interleave_order": (u64, [u64, vp, u64, u64, vp]),
            "orc_chain_output": (c_int, [vp, c_int, c_int, c_int, vp, vp, vp]),
            "orc_apply_chain": (c_int, [vp, c_int, c_int, i64, vp, c_int, vp]),
            "orc_epoch_image_digest": (u64, [vp, c_int, u64, vp, i64, c_int, c_int, c_int, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        self.L = L

    # ---- PRNG / shuffle ----
    def mix_seeds(self, a, b):
        return self.L.orc_mix_seeds(a, b)

    def shuffle_seed(self, epoch_salt, attr_seed=None):
        return self.L.orc_shuffle_seed(epoch_salt, 0 if attr_seed is None else 1, attr_seed or 0)

    def shuffle_order(self, n, buffer, engine_seed) -> np.ndarray:
        out = np.zeros(max(n, 1), np.uint32)
        self.L.orc_shuffle_order(n, buffer, engine_seed, P(out))
        return out[:n].astype(np.int64)

    # ---- digest ----
    def fnv_digest(self, values) -> int:
        v = np.ascontiguousarray(values, dtype=np.int64)
        return self.L.orc_digest_i64(self.L.orc_digest_init(), P(v), v.size)

    @staticmethod
    def order_digest(values, first=0) -> int:
        """K7's position-keyed digest: sum_i SplitMix64Next(v_i ^ (i*golden))."""
        v = np.ascontiguousarray(values).astype(np.uint64)
        with np.errstate(over="ignore"):
            i = np.arange(first, first + v.size, dtype=np.uint64)
            s = v ^ (i * np.uint64(0x9E3779B97F4A7C15))
            z = s + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            return int(z.sum(dtype=np.uint64))

    # ---- synthetic inputs ----
    def images(self, first_id, count, h, w, seed=PIX_SEED) -> np.ndarray:
        out = np.zeros((count, h, w, 3), np.uint8)
        self.L.orc_synth_images(seed, first_id, count, h * w * 3, P(out))
        return out

    def lengths(self, n, max_len=1024, seed=4) -> np.ndarray:
        out = np.zeros(n, np.int32)
        self.L.orc_synth_lengths(seed, max_len, n, P(out))
        return out

    def tokens(self, lengths, seed=4):
        offs = np.zeros(len(lengths) + 1, np.int64)
        offs[1:] = np.cumsum(lengths)
        # vectorised restatement of orc_synth_token (checked against it in tests)
        i = np.repeat(np.arange(len(lengths), dtype=np.uint64), lengths)
        j = (np.arange(offs[-1], dtype=np.int64) - np.repeat(offs[:-1], lengths)).astype(np.uint64)
        with np.errstate(over="ignore"):
            s = np.uint64(seed) ^ ((i << np.uint64(20)) | j)
            z = s + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        return (z & np.uint64(0x7FFFFFFF)).astype(np.int32), offs

    def token(self, seed, i, j):
        return self.L.orc_synth_token(seed, i, j)

    # ---- map UDFs ----
    def crop_params(self, seed, ident, in_h, in_w, ch, cw):
        oy, ox, fl = c_int(), c_int(), c_int()
        self.L.orc_crop_params(seed, ident, in_h, in_w, ch, cw, ctypes.byref(oy), ctypes.byref(ox), ctypes.byref(fl))
        return oy.value, ox.value, fl.value

    def crop_flip_normalize(self, img, ident, crop_h=224, crop_w=224, seed=UDF_SEED, do_flip=True):
        img = np.ascontiguousarray(img, np.uint8)
        out = np.zeros((crop_h, crop_w, 3), np.float32)
        self.L.orc_crop_flip_normalize(P(img), img.shape[0], img.shape[1], ident, seed, crop_h, crop_w,
                                       1 if do_flip else 0, P(out))
        return out

    def resize(self, img, out_h, out_w):
        img = np.ascontiguousarray(img, np.uint8)
        out = np.zeros((out_h, out_w, 3), np.float32)
        self.L.orc_resize(P(img), img.shape[0], img.shape[1], out_h, out_w, P(out))
        return out

    def resize_normalize(self, img, out_h=224, out_w=224):
        img = np.ascontiguousarray(img, np.uint8)
        out = np.zeros((out_h, out_w, 3), np.float32)
        self.L.orc_resize_normalize(P(img), img.shape[0], img.shape[1], out_h, out_w, P(out))
        return out

    def chain_output(self, steps, in_h, in_w):
        """(out_h, out_w, np dtype) of an image map chain (oracle/chain.c)."""
        h, w, f = c_int(), c_int(), c_int()
        arr = steps_array(steps)
        if self.L.orc_chain_output(arr, len(steps), in_h, in_w, ctypes.byref(h), ctypes.byref(w), ctypes.byref(f)):
            raise ValueError("invalid chain")
        return h.value, w.value, (np.float32 if f.value else np.uint8)

    def chain(self, img, ident, steps):
        """One element (id, img) through the image map chain, as MapFns in order."""
        img = np.ascontiguousarray(img, np.uint8)
        oh, ow, dt = self.chain_output(steps, img.shape[0], img.shape[1])
        out = np.zeros((oh, ow, 3), dt)
        if self.L.orc_apply_chain(P(img), img.shape[0], img.shape[1], ident, steps_array(steps), len(steps), P(out)):
            raise ValueError("chain failed")
        return out

    def epoch_image_digest(self, steps, ids, in_h, in_w, threads=None, seed=PIX_SEED):
        """K7 word digest of every output image of `ids` through the chain
        (position = running u32 word index across the epoch)."""
        ids = np.ascontiguousarray(ids, np.int64)
        err = c_int()
        d = self.L.orc_epoch_image_digest(steps_array(steps), len(steps), seed, P(ids), ids.size, in_h, in_w,
                                          threads or os.cpu_count() or 1, ctypes.byref(err))
        if err.value:
            raise ValueError("chain failed")
        return d

    # ---- filter / shard / interleave ----
    def filter_len_le(self, lengths, max_keep):
        lengths = np.ascontiguousarray(lengths, np.int32)
        kept = np.zeros(max(lengths.size, 1), np.uint32)
        m = self.L.orc_filter_len_le(P(lengths), lengths.size, max_keep, P(kept))
        return kept[:m].astype(np.int64)

    def bucket_by_length(self, lengths, order, boundaries, batch_sizes, drop=False):
        """-> list of position arrays, one per emitted batch (restate.c orc_bucket_by_length)."""
        lengths = np.ascontiguousarray(lengths, np.int32)
        order = None if order is None else np.ascontiguousarray(order, np.int64)
        n = lengths.size if order is None else order.size
        b = np.ascontiguousarray(boundaries, np.int32)
        s = np.ascontiguousarray(batch_sizes, np.int64)
        pos = np.zeros(max(n, 1), np.int64)
        rows = np.zeros(max(n + s.size, 1), np.int64)
        nb = self.L.orc_bucket_by_length(P(lengths), None if order is None else P(order), n,
                                         P(b) if b.size else None, b.size, P(s), int(drop), P(pos), P(rows))
        out, at = [], 0
        for r in rows[:nb]:
            out.append(pos[at:at + r])
            at += r
        return out

    def shard_positions(self, n, k, g):
        out = np.zeros(max(n, 1), np.uint64)
        m = self.L.orc_shard_positions(n, k, g, P(out))
        return out[:m].astype(np.int64)

    def interleave_var(self, inputs, cycle, lengths):
        """Interleave over readers of unequal lengths (restate.c orc_interleave_var)."""
        inputs = np.ascontiguousarray(inputs, np.uint64)
        lengths = np.ascontiguousarray(lengths, np.uint64)
        starts = np.zeros(lengths.size, np.uint64)
        starts[1:] = np.cumsum(lengths)[:-1]
        out = np.zeros(max(int(lengths.sum()), 1), np.uint64)
        self.L.orc_interleave_var.restype = ctypes.c_uint64
        self.L.orc_interleave_var.argtypes = [ctypes.c_uint64, vp, ctypes.c_uint64, vp, vp, vp]
        m = self.L.orc_interleave_var(inputs.size, P(inputs), cycle, P(lengths), P(starts), P(out))
        return out[:m].astype(np.int64)

    def interleave_order(self, inputs, cycle, records):
        inputs = np.ascontiguousarray(inputs, np.uint64)
        out = np.zeros(max(inputs.size * records, 1), np.uint64)
        m = self.L.orc_interleave_order(inputs.size, P(inputs), cycle, records, P(out))
        return out[:m].astype(np.int64)


class Reference:
    """The compiled reference runtime (oracle/_ref/libdpref.so)."""

    @staticmethod
    def load():
        if not os.path.exists(REF_SO):
            if os.path.isdir("/root/reference/proj/src"):
                subprocess.run(["make", "-C", ORACLE_DIR, "ref", "-j8"], check=True, capture_output=True)
            else:
                return None
        return Reference(ctypes.CDLL(REF_SO))

    def __init__(self, L):
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_range_map_batch.argtypes = [i64, i64, i64, i64, c_int, i64, c_int, u64, vp, vp, vp, ctypes.c_char_p]
        L.ref_shuffle_ids.argtypes = [i64, i64, i64, i64, c_int, u64, u64, i64, c_int, vp, vp]
        L.ref_image_pipeline.argtypes = [c_int, c_int, c_int, c_int, c_int, u64, u64, i64, i64, i64, i64, c_int, u64,
                                         i64, c_int, i64, i64, u64, vp, vp, vp, vp]
        L.ref_filter_batch_tokens.argtypes = [i64, u64, u32, u64, i32, i64, c_int, vp, vp, vp, vp, vp, vp]
        L.ref_image_chain_pipeline.argtypes = [vp, c_int, c_int, c_int, u64, i64, vp, i64, u64, i64, c_int, u64, vp,
                                               vp, vp, vp, vp]
        L.ref_interleave_ids.argtypes = [i64, i64, i64, i64, i64, i64, i64, u64, u64, vp, vp]
        L.ref_time_image_pipeline.argtypes = [c_int, c_int, c_int, c_int, c_int, u64, u64, i64, i64, u64, i64, i64,
                                              i64, u64, c_int, vp, vp]
        L.ref_time_range_map_batch.argtypes = [i64, i64, i64, c_int, vp]
        L.ref_time_filter_batch_tokens.argtypes = [i64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                                   ctypes.c_int32, i64, c_int, vp]
        self.L = L

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.L.ref_last_error().decode())

    def range_map_batch(self, n, a=3, b=1, batch=1024, drop_remainder=False, parallel=1, optimize=True, base_seed=1):
        vals = np.zeros(max(n, 1), np.int64)
        sizes = np.zeros(max(n, 1), np.int64)
        nb = np.zeros(1, np.int64)
        kind = ctypes.create_string_buffer(32)
        self._check(self.L.ref_range_map_batch(n, a, b, batch, int(drop_remainder), parallel, int(optimize),
                                               base_seed, P(vals), P(sizes), P(nb), kind))
        sizes = sizes[: nb[0]]
        return vals[: int(sizes.sum())], sizes, kind.value.decode()

    def shuffle_ids(self, n, buffer, seed=42, base_seed=1, shard=None, epochs=1, optimize=False, has_seed=True):
        out = np.zeros(max(n * epochs, 1), np.int64)
        cnt = np.zeros(1, np.int64)
        k, g = shard if shard else (0, 0)
        self._check(self.L.ref_shuffle_ids(n, k, g, buffer, int(has_seed), seed or 0, base_seed, epochs,
                                           int(optimize), P(out), P(cnt)))
        return out[: cnt[0]]

    def image_pipeline(self, mode, n, in_hw, out_hw, shuffle_buffer=0, shuffle_seed=42, batch=256,
                       drop_remainder=False, parallel=4, prefetch=2, base_seed=1, shard=None, udf_seed=UDF_SEED,
                       pix_seed=PIX_SEED):
        """mode 0 = crop+flip+normalize, 1 = resize+normalize, 2 = crop+normalize."""
        k, g = shard if shard else (0, 0)
        m = n if not shard else (n - g + k - 1) // k
        ids = np.zeros(max(m, 1), np.int64)
        pix = np.zeros((max(m, 1), out_hw[0], out_hw[1], 3), np.float32)
        sizes = np.zeros(max(m, 1), np.int64)
        nb = np.zeros(1, np.int64)
        self._check(self.L.ref_image_pipeline(mode, in_hw[0], in_hw[1], out_hw[0], out_hw[1], udf_seed, pix_seed, n,
                                              k, g, shuffle_buffer, 1, shuffle_seed, batch, int(drop_remainder),
                                              parallel, prefetch, base_seed, P(ids), P(pix), P(sizes), P(nb)))
        sizes = sizes[: nb[0]]
        t = int(sizes.sum())
        return ids[:t], pix[:t], sizes

    def image_chain_pipeline(self, steps, n, in_hw, labels=None, shuffle_buffer=0, shuffle_seed=42, batch=32,
                             drop_remainder=False, base_seed=1, pix_seed=PIX_SEED):
        """from_memory(synthetic images [, labels]) -> [shuffle] -> one map per
        chain step -> batch, optimized, through the reference runtime.
        -> (ids, images [n, h, w, 3] u8/f32, labels or None, batch sizes)"""
        orc = Oracle()
        oh, ow, dt = orc.chain_output(steps, *in_hw)
        ids = np.zeros(max(n, 1), np.int64)
        imgs = np.zeros((max(n, 1), oh, ow, 3), dt)
        lab_out = np.zeros(max(n, 1), np.int64)
        sizes = np.zeros(max(n, 1) + 1, np.int64)
        nb = i64()
        lab = None if labels is None else np.ascontiguousarray(labels, np.int64)
        self._check(self.L.ref_image_chain_pipeline(steps_array(steps), len(steps), in_hw[0], in_hw[1], pix_seed, n,
                                                    None if lab is None else P(lab), shuffle_buffer, shuffle_seed,
                                                    batch, int(drop_remainder), base_seed, P(ids), P(imgs),
                                                    P(lab_out), P(sizes), ctypes.byref(nb)))
        sizes = sizes[:nb.value]
        k = int(sizes.sum())
        return ids[:k], imgs[:k], (None if lab is None else lab_out[:k]), sizes

    def filter_batch_tokens(self, n, max_keep=512, batch=128, len_seed=4, max_len=1024, tok_seed=4,
                            drop_remainder=False):
        lens = Oracle().lengths(n, max_len, len_seed)
        rows_cap = n
        tok_cap = int(lens.sum())
        row_len = np.zeros(max(rows_cap, 1), np.int64)
        toks = np.zeros(max(tok_cap, 1), np.int64)
        sizes = np.zeros(max(rows_cap, 1), np.int64)
        nb, nr, nt = (np.zeros(1, np.int64) for _ in range(3))
        self._check(self.L.ref_filter_batch_tokens(n, len_seed, max_len, tok_seed, max_keep, batch,
                                                   int(drop_remainder), P(row_len), P(toks), P(sizes), P(nb), P(nr),
                                                   P(nt)))
        return row_len[: nr[0]], toks[: nt[0]], sizes[: nb[0]]

    def interleave_ids(self, num_sources, cycle, records, parallel=1, shard=None, shuffle_buffer=0, shuffle_seed=42,
                       base_seed=1):
        k, g = shard if shard else (0, 0)
        out = np.zeros(max(num_sources * records, 1), np.int64)
        cnt = np.zeros(1, np.int64)
        self._check(self.L.ref_interleave_ids(num_sources, k, g, cycle, parallel, records, shuffle_buffer,
                                              shuffle_seed, base_seed, P(out), P(cnt)))
        return out[: cnt[0]]

    def filter_values(self, n, a, b, odd, shuffle_buffer=0, optimize=True):
        out = np.zeros(max(n, 1), np.int64)
        cnt = np.zeros(1, np.int64)
        txt = ctypes.create_string_buffer(4096)
        self.L.ref_filter_values.argtypes = [i64, i64, i64, c_int, i64, c_int, vp, vp, vp, ctypes.c_size_t]
        self._check(self.L.ref_filter_values(n, a, b, int(odd), shuffle_buffer, int(optimize), P(out), P(cnt),
                                             ctypes.cast(txt, vp), len(txt)))
        return out[: cnt[0]], txt.value.decode()

    def interleave_var_ids(self, lengths, cycle, parallel=1, shard=None, base_seed=1):
        lengths = np.ascontiguousarray(lengths, np.int64)
        k, g = shard if shard else (0, 0)
        out = np.zeros(max(int(lengths.sum()), 1), np.int64)
        cnt = np.zeros(1, np.int64)
        self.L.ref_interleave_var_ids.argtypes = [i64, vp, i64, i64, i64, i64, ctypes.c_uint64, vp, vp]
        self._check(self.L.ref_interleave_var_ids(lengths.size, P(lengths), k, g, cycle, parallel, base_seed,
                                                  P(out), P(cnt)))
        return out[: cnt[0]]

    def time_image_pipeline(self, mode, n, in_hw, out_hw, parallel, epochs=3, shuffle_buffer=10000, batch=256,
                            prefetch=2):
        eps = np.zeros(epochs, np.float64)
        cnt = np.zeros(1, np.int64)
        self._check(self.L.ref_time_image_pipeline(mode, in_hw[0], in_hw[1], out_hw[0], out_hw[1], UDF_SEED,
                                                   PIX_SEED, n, shuffle_buffer, 42, batch, parallel, prefetch, 1,
                                                   epochs, P(eps), P(cnt)))
        return eps, int(cnt[0])

    def serialize_pipeline(self, which):
        """(DPG1 bytes, fingerprint hex) of known pipeline `which` (ref_shim.cpp)."""
        buf = ctypes.create_string_buffer(1 << 16)
        n = ctypes.c_size_t()
        hexs = ctypes.create_string_buffer(65)
        self.L.ref_serialize_pipeline.argtypes = [c_int, vp, ctypes.c_size_t, vp, vp]
        self._check(self.L.ref_serialize_pipeline(which, ctypes.cast(buf, vp), len(buf), ctypes.byref(n),
                                                  ctypes.cast(hexs, vp)))
        return buf.raw[: n.value], hexs.value.decode()

    def checkpoint_after(self, which, k):
        """DPC1 blob of known pipeline `which` after k GetNext calls (ref_shim.cpp)."""
        buf = ctypes.create_string_buffer(1 << 16)
        n = ctypes.c_size_t()
        self.L.ref_checkpoint_after.argtypes = [c_int, i64, vp, ctypes.c_size_t, vp]
        self._check(self.L.ref_checkpoint_after(which, k, ctypes.cast(buf, vp), len(buf), ctypes.byref(n)))
        return buf.raw[: n.value]

    def time_filter_batch_tokens(self, n, len_seed, max_len, tok_seed, max_keep, batch, epochs=3):
        eps = np.zeros(epochs, np.float64)
        self._check(self.L.ref_time_filter_batch_tokens(n, len_seed, max_len, tok_seed, max_keep, batch, epochs,
                                                        P(eps)))
        return eps

    def time_range_map_batch(self, n, batch, parallel, epochs=3):
        eps = np.zeros(epochs, np.float64)
        self._check(self.L.ref_time_range_map_batch(n, batch, parallel, epochs, P(eps)))
        return eps
