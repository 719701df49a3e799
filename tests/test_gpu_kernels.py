"""GPU parity of every sm_100a kernel family, called through the C ABI
(include/dpcuda.h), against the CPU oracle (oracle/restate.c) and the golden
vectors generated from the compiled reference (tests/golden/golden.json).

Bar: bit exact for all integer / index work and for crop + flip + normalize
(whose fp32 inputs are uint8, so the exact-division sequence is proven
exhaustively in test_oracle.py); resize + normalize within 1 ulp of fp32
(north star), and we also report how many values are not bit identical.
"""
import ctypes
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "golden.json")))
MEAN = (123.675, 116.28, 103.53)
STD = (58.395, 57.12, 57.375)


@pytest.fixture(scope="module")
def K():
    from paper_2101_12127_b200 import _capi
    return _capi


def vp(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def fnv(orc, v):
    return f"{orc.fnv_digest(np.asarray(v, dtype=np.int64)):016x}"


def ulp_diff(a, b):
    ai = a.view(np.int32).astype(np.int64)
    bi = b.view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(ai & 0x7FFFFFFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFFFFFF), bi)
    return np.abs(ai - bi)


def gpu_shuffle(K, n, buffer, engine_seed, in_map=None):
    import torch
    out = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    sb = K.lib().dp_k_shuffle_plan_scratch_bytes(n, buffer)
    scratch = torch.empty(max(sb, 1), dtype=torch.uint8, device="cuda") if sb else None
    K.check(K.lib().dp_k_shuffle_plan(n, buffer, engine_seed, vp(in_map), vp(out), vp(scratch), stream()))
    torch.cuda.synchronize()
    return out[:n]


# ------------------------------------------------------------------ K1 ----
def test_k1_range_affine_cfg1(K, orc, dev):
    import torch
    n, b = 1_000_000, 1024
    out = torch.empty(n, dtype=torch.int64, device=dev)
    sizes = []
    for first in range(0, n, b):
        rows = min(b, n - first)
        K.check(K.lib().dp_k_range_affine_batch(first, rows, 3, 1, vp(out[first:]), stream()))
        sizes.append(rows)
    vals = out.cpu().numpy()
    want = GOLDEN["cfg1_range_map_batch_1024"]["1000000"]
    assert len(sizes) == want["num_batches"] == 977 and sizes[-1] == want["last_batch"] == 576
    assert int(vals.sum()) == want["sum"] == 1_499_999_500_000
    assert fnv(orc, vals) == want["fnv"] == "8bc444c576bd14a5"


def test_k1_odd_and_unaligned(K, dev):
    import torch
    buf = torch.zeros(1001, dtype=torch.int64, device=dev)
    K.check(K.lib().dp_k_range_affine_batch(-5, 999, -7, 11, vp(buf[1:]), stream()))
    got = buf.cpu().numpy()
    assert got[0] == 0 and (got[1:1000] == (np.arange(-5, 994) * -7 + 11)).all() and got[1000] == 0


# ------------------------------------------------------------------ K2 ----
def test_k2_shuffle_golden(K, orc, dev):
    for c in GOLDEN["shuffle"]:
        got = gpu_shuffle(K, c["n"], c["buffer"], orc.shuffle_seed(c["base_seed"], c["seed"])).cpu().numpy()
        assert got[:8].tolist() == c["first"], c
        assert fnv(orc, got) == c["fnv"], c


def test_k2_shuffle_random_vs_oracle(K, orc, dev):
    rng = np.random.default_rng(5)
    for _ in range(60):
        n = int(rng.integers(1, 200_000))
        b = int(rng.choice([1, 2, 31, 32, 33, 1000, 10000, int(rng.integers(1, n + 10))]))
        seed = int(rng.integers(0, 2**64, dtype=np.uint64))
        want = orc.shuffle_order(n, b, seed)
        got = gpu_shuffle(K, n, b, seed).cpu().numpy()
        assert (got == want).all(), (n, b, seed)


def test_k2_shuffle_global_scratch_and_in_map(K, orc, dev):
    import torch
    n, b, seed = 150_000, 120_000, 99  # 480 KB reservoir -> global scratch path
    assert K.lib().dp_k_shuffle_plan_scratch_bytes(n, b) > 0
    in_map = torch.arange(n, dtype=torch.int64, device=dev) * 5 + 3
    got = gpu_shuffle(K, n, b, seed, in_map=in_map).cpu().numpy()
    assert (got == orc.shuffle_order(n, b, seed) * 5 + 3).all()


def test_k2_rejects_bad_buffer(K, dev):
    import torch
    out = torch.empty(4, dtype=torch.int64, device=dev)
    rc = K.lib().dp_k_shuffle_plan(4, 0, 1, None, vp(out), None, stream())
    assert rc == 2 and b"buffer_size" in K.lib().dp_last_error()  # DP_ERR_INVALID_ATTR


# --------------------------------------------------------------- K3/K4 ----
def device_images(K, dev, n, h, w, first=0):
    import torch
    imgs = torch.empty((n, h, w, 3), dtype=torch.uint8, device=dev)
    K.check(K.lib().dp_k_synth_images(vp(imgs), first, n, h * w * 3, 0x5EED, stream()))
    return imgs


def run_crop(K, imgs, order, first, rows, crop=(224, 224), do_flip=1, seed=7):
    import torch
    ids = torch.empty(rows, dtype=torch.int64, device=imgs.device)
    out = torch.empty((rows, crop[0], crop[1], 3), dtype=torch.float32, device=imgs.device)
    K.check(K.lib().dp_k_crop_flip_normalize_batch(
        vp(imgs), imgs.shape[0], imgs.shape[1], imgs.shape[2], vp(order), first, rows, seed, crop[0], crop[1],
        do_flip, K.floats3(MEAN), K.floats3(STD), vp(ids), vp(out), stream()))
    torch.cuda.synchronize()
    return ids.cpu().numpy(), out.cpu().numpy()


def run_resize(K, imgs, order, first, rows, out_hw=(224, 224)):
    import torch
    ids = torch.empty(rows, dtype=torch.int64, device=imgs.device)
    out = torch.empty((rows, out_hw[0], out_hw[1], 3), dtype=torch.float32, device=imgs.device)
    K.check(K.lib().dp_k_resize_normalize_batch(
        vp(imgs), imgs.shape[0], imgs.shape[1], imgs.shape[2], vp(order), first, rows, out_hw[0], out_hw[1],
        K.floats3(MEAN), K.floats3(STD), vp(ids), vp(out), stream()))
    torch.cuda.synchronize()
    return ids.cpu().numpy(), out.cpu().numpy()


def test_synth_images_match_oracle(K, orc, dev):
    imgs = device_images(K, dev, 3, 256, 256, first=1000).cpu().numpy()
    assert (imgs == orc.images(1000, 3, 256, 256)).all()


def test_k3_crop_flip_normalize_bit_exact(K, orc, dev):
    import torch
    imgs = device_images(K, dev, 300, 256, 256)
    order = gpu_shuffle(K, 300, 100, orc.shuffle_seed(1, 42))
    ids, out = run_crop(K, imgs, order, 40, 64)
    host = imgs.cpu().numpy()
    want_ids = order.cpu().numpy()[40:104]
    assert (ids == want_ids).all()
    flips = 0
    for k, p in enumerate(want_ids):
        want = orc.crop_flip_normalize(host[p], int(p))
        assert np.array_equal(out[k].view(np.uint32), want.view(np.uint32)), k
        flips += orc.crop_params(7, int(p), 256, 256, 224, 224)[2]
    assert 0 < flips < 64  # both flip branches exercised


def test_k3_unaligned_generic_path(K, orc, dev):
    imgs = device_images(K, dev, 20, 250, 251)  # row bytes 753: not 16B aligned
    ids, out = run_crop(K, imgs, None, 3, 9, crop=(200, 222))
    host = imgs.cpu().numpy()
    for k in range(9):
        want = orc.crop_flip_normalize(host[3 + k], 3 + k, 200, 222)
        assert np.array_equal(out[k].view(np.uint32), want.view(np.uint32))


def test_k3_crop_only(K, orc, dev):
    imgs = device_images(K, dev, 8, 256, 256)
    ids, out = run_crop(K, imgs, None, 0, 8, do_flip=0)
    host = imgs.cpu().numpy()
    for k in range(8):
        assert np.array_equal(out[k], orc.crop_flip_normalize(host[k], k, do_flip=False))


@pytest.mark.parametrize("roll", ["1", "0"])
def test_k4_resize_normalize_within_1ulp(K, orc, dev, monkeypatch, roll):
    """320 -> 224 runs on K10 (periodic column map, k_roll.cu) by default and
    on K4's periodic-tap consumer with K10 disabled; both bit-exact."""
    monkeypatch.setenv("DP_DEV_ROLL", roll)
    imgs = device_images(K, dev, 40, 320, 320)
    order = gpu_shuffle(K, 40, 16, orc.shuffle_seed(1, 42))
    ids, out = run_resize(K, imgs, order, 5, 30)
    host = imgs.cpu().numpy()
    worst, nonzero = 0, 0
    for k, p in enumerate(order.cpu().numpy()[5:35]):
        want = orc.resize_normalize(host[p])
        d = ulp_diff(out[k], want)
        worst = max(worst, int(d.max()))
        nonzero += int((d > 0).sum())
    assert worst <= 1
    assert nonzero == 0, f"{nonzero} values differ by 1 ulp"  # design goal: 0 ulp


def test_k4_periodic_and_general_paths_agree(K, dev, monkeypatch):
    """320 -> 224 runs the periodic-tap consumer (ResizePOp<7, 10>); the
    general ResizeOp (DP_DEV_RESIZE_PERIODIC=0) must give the same bits."""
    imgs = device_images(K, dev, 24, 320, 320)
    order = gpu_shuffle(K, 24, 8, 99)
    _, k10 = run_resize(K, imgs, order, 0, 24)
    monkeypatch.setenv("DP_DEV_ROLL", "0")
    _, a = run_resize(K, imgs, order, 0, 24)
    monkeypatch.setenv("DP_DEV_RESIZE_PERIODIC", "0")
    _, b = run_resize(K, imgs, order, 0, 24)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert np.array_equal(a.view(np.uint32), k10.view(np.uint32))


@pytest.mark.parametrize("roll", ["1", "0"])
def test_k4_other_shapes(K, orc, dev, monkeypatch, roll):
    monkeypatch.setenv("DP_DEV_ROLL", roll)
    # (256, 256) and (160, 160) -> periodic column taps (ResizePOp 7/8, 7/10
    # with 16 groups per row), the rest the general ResizeOp / generic kernel
    for (ih, iw, oh, ow) in ((100, 160, 224, 224), (480, 360, 224, 224), (33, 57, 17, 23), (256, 256, 224, 224),
                             (160, 160, 112, 112), (200, 320, 96, 224)):
        imgs = device_images(K, dev, 3, ih, iw)
        ids, out = run_resize(K, imgs, None, 0, 3, (oh, ow))
        host = imgs.cpu().numpy()
        for k in range(3):
            assert ulp_diff(out[k], orc.resize_normalize(host[k], oh, ow)).max() <= 1


def test_golden_image_pipelines_through_kernels(K, orc, dev):
    import torch
    for c in GOLDEN["image_pipelines"]:
        n, (ih, iw), (oh, ow) = c["n"], c["in_hw"], c["out_hw"]
        imgs = device_images(K, dev, n, ih, iw)
        if c["shard"]:
            k, g = c["shard"]
            m = (n - g + k - 1) // k
            order = torch.empty(m, dtype=torch.int64, device=dev)
            K.check(K.lib().dp_k_shard_index(n, k, g, None, vp(order), stream()))
        else:
            m, order = n, torch.arange(n, dtype=torch.int64, device=dev)
        if c["shuffle_buffer"]:
            order = gpu_shuffle(K, m, c["shuffle_buffer"], orc.shuffle_seed(c["base_seed"], c["shuffle_seed"]),
                                in_map=order)
        all_ids, all_pix, sizes = [], [], []
        for first in range(0, m, c["batch"]):
            rows = min(c["batch"], m - first)
            if c["mode"] == 1:
                ids, pix = run_resize(K, imgs, order, first, rows, (oh, ow))
            else:
                ids, pix = run_crop(K, imgs, order, first, rows, (oh, ow), do_flip=1 if c["mode"] == 0 else 0)
            all_ids.append(ids)
            all_pix.append(pix)
            sizes.append(rows)
        assert sizes == c["batch_sizes"]
        assert fnv(orc, np.concatenate(all_ids)) == c["fnv_ids"]
        pix = np.concatenate(all_pix)
        assert fnv(orc, pix.view(np.uint32).astype(np.int64)) == c["fnv_pixels"], c


# ------------------------------------------------------------------ K5 ----
def test_k5_filter_padded_batch(K, orc, dev):
    import torch
    c = GOLDEN["cfg4_filter_batch"]
    lens = orc.lengths(c["n"], c["max_len"], c["len_seed"])
    toks, offs = orc.tokens(lens, c["tok_seed"])
    d_len = torch.from_numpy(lens).to(dev)
    d_off = torch.from_numpy(offs).to(dev)
    d_tok = torch.empty(int(offs[-1]), dtype=torch.int32, device=dev)
    K.check(K.lib().dp_k_synth_tokens(vp(d_tok), vp(d_off), lens.size, c["tok_seed"], stream()))
    assert (d_tok.cpu().numpy() == toks).all()
    kept = torch.empty(lens.size, dtype=torch.int64, device=dev)
    nk = torch.zeros(1, dtype=torch.int64, device=dev)
    scratch = torch.empty(K.lib().dp_k_filter_scratch_bytes(lens.size), dtype=torch.uint8, device=dev)
    K.check(K.lib().dp_k_filter_len_le(vp(d_len), lens.size, c["max_keep"], None, vp(kept), vp(nk), vp(scratch),
                                       stream()))
    m = int(nk.item())
    want_kept = orc.filter_len_le(lens, c["max_keep"])
    assert m == want_kept.size == c["rows"]
    assert (kept[:m].cpu().numpy() == want_kept).all()
    b = c["batch"]
    nb = (m + b - 1) // b
    lmax = torch.empty(nb, dtype=torch.int32, device=dev)
    K.check(K.lib().dp_k_batch_max_len(vp(d_len), vp(kept), m, b, vp(lmax), stream()))
    lmax = lmax.cpu().numpy()
    flat_rows, flat_toks, sizes = [], [], []
    for j in range(nb):
        rows = min(b, m - j * b)
        rl = lens[want_kept[j * b:j * b + rows]]
        assert lmax[j] == rl.max()
        out = torch.full((rows, int(lmax[j])), -7, dtype=torch.int32, device=dev)
        olen = torch.empty(rows, dtype=torch.int32, device=dev)
        K.check(K.lib().dp_k_padded_batch(vp(d_tok), vp(d_off), vp(d_len), vp(kept), j * b, rows, int(lmax[j]), 0,
                                          vp(out), vp(olen), stream()))
        out, olen = out.cpu().numpy(), olen.cpu().numpy()
        assert (olen == rl).all()
        for r in range(rows):
            p = want_kept[j * b + r]
            assert (out[r, :rl[r]] == toks[offs[p]:offs[p + 1]]).all()
            assert (out[r, rl[r]:] == 0).all()
            flat_toks.append(out[r, :rl[r]])
        flat_rows.append(olen)
        sizes.append(rows)
    assert fnv(orc, np.concatenate(flat_rows)) == c["fnv_row_lengths"]
    assert fnv(orc, np.concatenate(flat_toks)) == c["fnv_tokens"]
    assert fnv(orc, sizes) == c["fnv_batch_sizes"]


def test_k5_filter_edge_cases(K, orc, dev):
    import torch
    for n, keep in ((0, 5), (1, 0), (1, 5), (4095, 512), (4096, 512), (4097, 512), (100_000, 0), (100_000, 2000)):
        lens = orc.lengths(max(n, 1), 1024, 11)[:n]
        d_len = torch.from_numpy(np.ascontiguousarray(lens)).to(dev) if n else torch.empty(0, dtype=torch.int32,
                                                                                          device=dev)
        kept = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        nk = torch.full((1,), -1, dtype=torch.int64, device=dev)
        scratch = torch.empty(K.lib().dp_k_filter_scratch_bytes(n), dtype=torch.uint8, device=dev)
        K.check(K.lib().dp_k_filter_len_le(vp(d_len), n, keep, None, vp(kept), vp(nk), vp(scratch), stream()))
        want = orc.filter_len_le(lens, keep) if n else np.zeros(0, np.int64)
        m = int(nk.item())
        assert m == want.size and (kept[:m].cpu().numpy() == want).all(), (n, keep)


# ------------------------------------------------------------------ K6 ----
def test_k6_shard_interleave_golden(K, orc, dev):
    import torch
    for c in GOLDEN["interleave"]:
        k, g = c["shard"] if c["shard"][0] else (1, 0)
        cnt = K.lib().dp_k_shard_interleave_count(c["num_sources"], k, g, c["records"])
        assert cnt == c["count"] or "shuffle" in c
        out = torch.empty(max(cnt, 1), dtype=torch.int64, device=dev)
        K.check(K.lib().dp_k_shard_interleave_index(c["num_sources"], k, g, c["cycle"], c["records"], vp(out),
                                                    stream()))
        if "shuffle" in c:
            buf, seed = c["shuffle"]
            out = gpu_shuffle(K, cnt, buf, orc.shuffle_seed(1, seed), in_map=out[:cnt])
        got = out[:cnt].cpu().numpy()
        assert got[:8].tolist() == c["first"] and fnv(orc, got) == c["fnv"], c


def test_k6_shard_index(K, orc, dev):
    import torch
    for n, k, g in ((10, 3, 0), (10, 3, 2), (7, 8, 6), (1_000_003, 8, 5)):
        m = (n - g + k - 1) // k
        out = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        K.check(K.lib().dp_k_shard_index(n, k, g, None, vp(out), stream()))
        assert (out[:m].cpu().numpy() == orc.shard_positions(n, k, g)).all()


# ------------------------------------------------------------------ K7 ----
def test_k7_order_digest(K, orc, dev):
    import torch
    v = np.random.default_rng(3).integers(-2**62, 2**62, 1_000_003, dtype=np.int64)
    d = torch.zeros(1, dtype=torch.int64, device=dev)
    t = torch.from_numpy(v).to(dev)
    K.check(K.lib().dp_k_order_digest(vp(t[:500_000]), 500_000, 0, vp(d), stream()))
    K.check(K.lib().dp_k_order_digest(vp(t[500_000:]), v.size - 500_000, 500_000, vp(d), stream()))
    got = int(d.cpu().numpy().view(np.uint64)[0])
    assert got == orc.order_digest(v)
    # order sensitive
    assert orc.order_digest(v[::-1]) != got
