"""K10 (csrc/k_roll.cu): bilinear-resize image chains over a periodic column
map, horizontal blends rolled in registers.  Called through the C ABI
(dp_k_image_chain_batch, include/dpcuda.h) and compared bit for bit with the
oracle's sequential map chain (oracle/chain.c: each MapFn on the whole image,
every fp32 op rounded once -- the reference's map(f).map(g) composition,
P/src/optimizer.cpp:165-188) for every output value, and with K9 (the same
chain with K10 disabled).

Cases cover each periodic ratio (10:7, 8:7, 5:7, 5:4), crop A random with
and without flip / center, crop B center / random with flip (one and two
column stripes), each pixel op (none, proven two-FMA normalize, affine,
IEEE normalize for constants the device proof rejects), sharded element ids,
batches not a multiple of anything, and BASELINE-size RandomResizedCrop /
ResNet eval images."""
import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MEAN = (123.675, 116.28, 103.53)
STD = (58.395, 57.12, 57.375)
ADV_STD = (1.99999988, 0.99999994, 3.0)  # with mean 0: two-FMA division is NOT exact (k_prove.cu)


@pytest.fixture(scope="module")
def K():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2101_12127_b200 import _capi
    return _capi


def run_chain(K, steps, imgs_dev, order_dev, rows, id_base=0, id_stride=1, first=0, roll=True):
    import torch
    n, h, w, _ = imgs_dev.shape
    c = K.ImageChain.from_steps(steps, h, w)
    oh, ow, f32 = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    K.check(K.lib().dp_image_chain_output(ctypes.byref(c), ctypes.byref(oh), ctypes.byref(ow), ctypes.byref(f32)))
    out = torch.full((rows, oh.value, ow.value, 3), float("nan"), dtype=torch.float32, device="cuda")
    ids = torch.full((rows,), -1, dtype=torch.int64, device="cuda")
    old = os.environ.get("DP_DEV_ROLL")
    os.environ["DP_DEV_ROLL"] = "1" if roll else "0"
    try:
        K.check(K.lib().dp_k_image_chain_batch(
            ctypes.c_void_p(imgs_dev.data_ptr()), n, ctypes.c_void_p(order_dev.data_ptr()), first, rows, id_base,
            id_stride, 1, ctypes.byref(c), ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    finally:
        if old is None:
            del os.environ["DP_DEV_ROLL"]
        else:
            os.environ["DP_DEV_ROLL"] = old
    torch.cuda.synchronize()
    return ids.cpu().numpy(), out.cpu().numpy()


def kernel_of(K, steps, h, w):
    c = K.ImageChain.from_steps(steps, h, w)
    k = ctypes.c_int()
    K.check(K.lib().dp_image_chain_kernel(ctypes.byref(c), ctypes.byref(k)))
    return k.value


CASES = {
    # name: (in_hw, steps, n, rows)
    "rrc_5to7_flip": ((64, 64), [("random_crop", 40, 40, 3, True), ("resize", 56, 56), ("normalize", MEAN, STD)],
                      40, 37),
    "rrc_5to7_noflip": ((64, 48), [("random_crop", 40, 20, 5, False), ("resize", 56, 28), ("normalize", MEAN, STD)],
                        24, 24),
    "k4_10to7": ((80, 80), [("resize", 56, 56), ("normalize", MEAN, STD)], 24, 21),
    "k4_8to7": ((64, 64), [("resize", 56, 56), ("normalize", MEAN, STD)], 24, 21),
    "eval_5to4_center": ((80, 80), [("resize", 64, 64), ("center_crop", 56, 56), ("normalize", MEAN, STD)], 24, 19),
    "post_random_crop_flip_affine": ((80, 80), [("resize", 64, 64), ("random_crop", 48, 44, 11, True),
                                                ("affine", (1 / 255, 2 / 255, 0.5), (-0.5, 0.25, 3.0))], 32, 32),
    "center_pre_crop_resize_only": ((64, 64), [("center_crop", 40, 40), ("resize", 56, 56)], 16, 16),
    "ieee_normalize": ((64, 64), [("random_crop", 40, 40, 9, True), ("resize", 56, 56),
                                  ("normalize", (0.0, 0.0, 0.0), ADV_STD)], 24, 23),
    "cast": ((80, 80), [("resize", 56, 56), ("normalize", (0, 0, 0), (1, 1, 1))], 16, 16),
    "rrc_full_size": ((256, 256), [("random_crop", 160, 160, 7, True), ("resize", 224, 224),
                                   ("normalize", MEAN, STD)], 40, 33),
    "eval_full_size": ((320, 320), [("resize", 256, 256), ("center_crop", 224, 224), ("normalize", MEAN, STD)],
                       24, 17),
    "two_stripes_random_post_crop": ((320, 320), [("resize", 256, 256), ("random_crop", 224, 224, 5, True),
                                                  ("normalize", MEAN, STD)], 16, 12),
    "k4_full_size": ((320, 320), [("resize", 224, 224), ("normalize", MEAN, STD)], 24, 20),
    # the other instantiated ratios: 9:7, 12:7, 6:7, 4:7, 3:2, 2:1
    "ratio_9to7": ((144, 144), [("resize", 112, 112), ("normalize", MEAN, STD)], 12, 11),
    "ratio_12to7": ((48, 48), [("resize", 28, 28), ("normalize", MEAN, STD)], 16, 16),
    "ratio_6to7_post_crop": ((96, 96), [("resize", 112, 112), ("random_crop", 96, 92, 2, True),
                                        ("normalize", MEAN, STD)], 12, 12),
    "ratio_4to7_pre_crop": ((64, 64), [("random_crop", 48, 48, 6, True), ("resize", 84, 84),
                                       ("normalize", MEAN, STD)], 12, 12),
    "ratio_3to2_center": ((96, 96), [("resize", 64, 64), ("center_crop", 48, 48), ("normalize", MEAN, STD)], 12, 12),
    "ratio_2to1_affine": ((128, 128), [("resize", 64, 64), ("affine", (0.5, 0.25, 2.0), (1.0, -1.0, 0.0))], 12, 12),
    # any other ratio: the general column map (runtime taps per pixel)
    "general_7to6_crop_flip": ((48, 48), [("random_crop", 28, 28, 3, True), ("resize", 24, 24),
                                          ("normalize", MEAN, STD)], 16, 16),
    "general_25to16": ((112, 112), [("resize", 72, 72), ("normalize", MEAN, STD)], 8, 8),
    "general_16to25_up": ((64, 64), [("resize", 100, 100), ("normalize", MEAN, STD)], 8, 8),
    "general_rrc_11to14_up": ((256, 256), [("random_crop", 176, 176, 5, True), ("resize", 224, 224),
                                           ("normalize", MEAN, STD)], 12, 12),
    "general_8to5_affine": ((96, 96), [("resize", 60, 60), ("affine", (0.5, 0.25, 2.0), (1.0, -1.0, 0.0))], 8, 8),
    "general_post_crop_flip": ((80, 80), [("resize", 72, 72), ("random_crop", 64, 60, 4, True),
                                          ("normalize", MEAN, STD)], 8, 8),
    "general_ieee": ((80, 48), [("random_crop", 66, 44, 1, False), ("resize", 50, 36),
                                ("normalize", (0.0, 0.0, 0.0), ADV_STD)], 8, 8),
    "general_wide_two_stripes": ((128, 512), [("resize", 96, 300), ("normalize", MEAN, STD)], 4, 4),
    # two pixel ops after the resize (general form): cast then affine, affine then normalize (IEEE), proven
    # normalize then affine, IEEE normalize then IEEE normalize
    "two_ops_cast_affine": ((80, 80), [("resize", 56, 56), ("normalize", (0, 0, 0), (1, 1, 1)),
                                       ("affine", (1 / 255, 1 / 255, 1 / 255), (0.0, -0.5, 0.25))], 8, 8),
    "two_ops_affine_normalize": ((64, 64), [("random_crop", 40, 40, 3, True), ("resize", 56, 56),
                                            ("affine", (1 / 255, 2 / 255, 0.5), (-0.5, 0.25, 3.0)),
                                            ("normalize", (0.5, 0.5, 0.5), (0.25, 0.5, 2.0))], 8, 8),
    "two_ops_normalize_affine": ((96, 96), [("resize", 60, 60), ("normalize", MEAN, STD),
                                            ("affine", (2.0, 0.5, -1.0), (0.1, 0.2, 0.3))], 8, 8),
    "two_ops_ieee_ieee": ((80, 48), [("resize", 50, 36), ("normalize", (0.0, 0.0, 0.0), ADV_STD),
                                     ("normalize", (0.5, 1.0, -2.0), (3.0, 0.75, 1.5))], 8, 8),
}


@pytest.mark.parametrize("name", list(CASES))
def test_k10_chain_bit_exact_vs_oracle(K, orc, name):
    import torch
    (h, w), steps, n, rows = CASES[name]
    assert kernel_of(K, steps, h, w) == 10, name
    imgs = orc.images(0, n, h, w)
    rng = np.random.default_rng(len(name))
    order = rng.integers(0, n, size=rows + 5).astype(np.int64)
    dimgs = torch.from_numpy(imgs).cuda()
    dorder = torch.from_numpy(order).cuda()
    ids, out = run_chain(K, steps, dimgs, dorder, rows, first=5)
    assert np.array_equal(ids, order[5:5 + rows])
    for j in range(rows):
        want = orc.chain(imgs[order[5 + j]], int(order[5 + j]), steps)
        got = out[j]
        if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
            bad = np.argwhere(got.view(np.uint32) != want.view(np.uint32))
            raise AssertionError(f"{name}: row {j} differs at {bad[:5].tolist()} ({bad.shape[0]} values): "
                                 f"{got[tuple(bad[0])]} vs {want[tuple(bad[0])]}")
    # K9 computes the same values
    _, out9 = run_chain(K, steps, dimgs, dorder, rows, first=5, roll=False)
    assert np.array_equal(out9.view(np.uint32), out.view(np.uint32))


def test_k10_sharded_ids_key_the_crops(K, orc):
    """Sharded residency: resident row r is element id base + r * stride, the
    Philox counter of both crops (id_base / id_stride as K3's _ex)."""
    import torch
    steps = [("random_crop", 40, 40, 3, True), ("resize", 56, 56), ("random_crop", 48, 48, 4, True),
             ("normalize", MEAN, STD)]
    n, base, stride = 12, 1, 3
    gids = base + stride * np.arange(n)
    imgs = np.stack([orc.images(int(g), 1, 64, 64)[0] for g in gids])
    order = np.arange(n, dtype=np.int64)[::-1].copy()
    ids, out = run_chain(K, steps, torch.from_numpy(imgs).cuda(), torch.from_numpy(order).cuda(), n, base, stride)
    assert np.array_equal(ids, gids[order])
    for j in range(n):
        want = orc.chain(imgs[order[j]], int(gids[order[j]]), steps)
        assert np.array_equal(out[j].view(np.uint32), want.view(np.uint32)), j


def test_k10_eligibility(K):
    # resize chains run on K10 (periodic maps or runtime taps); pre-resize pixel ops, two post ops and
    # output rows that are not whole float4 stay on K9
    assert kernel_of(K, [("random_crop", 160, 160, 7, True), ("resize", 224, 224), ("normalize", MEAN, STD)],
                     256, 256) == 10
    assert kernel_of(K, [("resize", 256, 256), ("center_crop", 224, 224), ("normalize", MEAN, STD)], 320, 320) == 10
    assert kernel_of(K, [("random_crop", 28, 28, 3, True), ("resize", 24, 24), ("normalize", MEAN, STD)],
                     48, 48) == 10  # general column map
    assert kernel_of(K, [("random_crop", 28, 28, 3, True), ("resize", 24, 26)], 48, 48) == 9  # 26 * 3 % 4 != 0
    assert kernel_of(K, [("resize", 100, 100), ("normalize", MEAN, STD)], 64, 64) == 10  # a non-periodic upscale
    assert kernel_of(K, [("normalize", MEAN, STD), ("resize", 56, 56)], 80, 80) == 9
    assert kernel_of(K, [("resize", 56, 56), ("affine", (1, 1, 1), (0, 0, 0)), ("normalize", MEAN, STD)],
                     80, 80) == 10  # two pixel ops: the general form
    assert kernel_of(K, [("resize", 56, 56), ("affine", (1, 1, 1), (0, 0, 0)), ("normalize", MEAN, STD),
                         ("affine", (1, 1, 1), (0, 0, 0))], 80, 80) == 9  # three


def test_fast_division_proof_on_device(K):
    """The device proof accepts the ImageNet constants and rejects a std whose
    two-FMA quotient is not IEEE-exact; K3 with such constants still matches
    the oracle (it runs the chain through K9's IEEE division)."""
    p = ctypes.c_int(-1)
    K.check(K.lib().dp_fast_div_proven(K.floats3(MEAN), K.floats3(STD), ctypes.byref(p)))
    assert p.value == 1
    K.check(K.lib().dp_fast_div_proven(K.floats3((0.0, 0.0, 0.0)), K.floats3(ADV_STD), ctypes.byref(p)))
    assert p.value == 0
    K.check(K.lib().dp_fast_div_proven(K.floats3((127.5, 127.5, 127.5)), K.floats3((127.5, 64, 1)),
                                       ctypes.byref(p)))
    assert p.value == 1


@pytest.mark.parametrize("which", ["k3", "k4"])
def test_unproven_constants_use_ieee_division(K, orc, which):
    """K3 / K4 entry points with normalize constants whose two-FMA division
    is not exact: every value still equals the oracle's IEEE division."""
    import torch
    mean = (0.0, 0.0, 0.0)
    n, rows = 12, 10
    imgs = orc.images(0, n, 32, 32)
    order = np.arange(n, dtype=np.int64)[::-1].copy()
    out = torch.empty((rows, 24, 24, 3), dtype=torch.float32, device="cuda")
    ids = torch.empty((rows,), dtype=torch.int64, device="cuda")
    dimgs, dorder = torch.from_numpy(imgs).cuda(), torch.from_numpy(order).cuda()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if which == "k3":
        steps = [("random_crop", 24, 24, 9, True), ("normalize", mean, ADV_STD)]
        K.check(K.lib().dp_k_crop_flip_normalize_batch(
            ctypes.c_void_p(dimgs.data_ptr()), n, 32, 32, ctypes.c_void_p(dorder.data_ptr()), 0, rows, 9, 24, 24, 1,
            K.floats3(mean), K.floats3(ADV_STD), ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(out.data_ptr()), s))
    else:
        steps = [("resize", 24, 24), ("normalize", mean, ADV_STD)]
        K.check(K.lib().dp_k_resize_normalize_batch(
            ctypes.c_void_p(dimgs.data_ptr()), n, 32, 32, ctypes.c_void_p(dorder.data_ptr()), 0, rows, 24, 24,
            K.floats3(mean), K.floats3(ADV_STD), ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(out.data_ptr()), s))
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for j in range(rows):
        want = orc.chain(imgs[order[j]], int(order[j]), steps)
        assert np.array_equal(got[j].view(np.uint32), want.view(np.uint32)), j


def test_k10_random_chains_bit_exact(K, orc):
    """40 seeded random resize chains (image sizes, crop A / B modes and
    flips, output sizes of any ratio -- periodic or not, up or down --,
    the pixel op and its constants), each on K10 when eligible, compared
    value for value with the oracle's sequential chain."""
    import torch
    rng = np.random.default_rng(2024)
    ran = 0
    for case in range(40):
        in_w = int(rng.choice([16, 32, 48, 64, 80, 96]))
        in_h = int(rng.integers(8, 97))
        steps = []
        win_h, win_w = in_h, in_w
        if rng.random() < 0.6:
            win_h, win_w = int(rng.integers(4, in_h + 1)), int(rng.integers(4, in_w + 1))
            if rng.random() < 0.7:
                steps.append(("random_crop", win_h, win_w, int(rng.integers(0, 100)), bool(rng.random() < 0.5)))
            else:
                steps.append(("center_crop", win_h, win_w))
        mid_h, mid_w = int(rng.integers(4, 2 * win_h + 4)), 4 * int(rng.integers(1, (2 * win_w + 8) // 4 + 1))
        steps.append(("resize", mid_h, mid_w))
        out_h, out_w = mid_h, mid_w
        if rng.random() < 0.4:
            out_h, out_w = int(rng.integers(1, mid_h + 1)), 4 * int(rng.integers(1, mid_w // 4 + 1))
            if rng.random() < 0.5:
                steps.append(("random_crop", out_h, out_w, int(rng.integers(0, 100)), bool(rng.random() < 0.5)))
            else:
                steps.append(("center_crop", out_h, out_w))
        op = rng.integers(0, 4)
        if op == 1:
            steps.append(("normalize", MEAN, STD))
        elif op == 2:
            steps.append(("affine", tuple(rng.normal(size=3)), tuple(rng.normal(size=3))))
        elif op == 3:
            steps.append(("normalize", tuple(rng.uniform(0, 255, 3)), tuple(rng.uniform(0.5, 100, 3))))
        if kernel_of(K, steps, in_h, in_w) != 10:
            continue
        ran += 1
        n, rows = 6, 5
        imgs = orc.images(case * 100, n, in_h, in_w)
        order = rng.integers(0, n, size=rows).astype(np.int64)
        ids, out = run_chain(K, steps, torch.from_numpy(imgs).cuda(), torch.from_numpy(order).cuda(), rows)
        for j in range(rows):
            want = orc.chain(imgs[order[j]], int(order[j]), steps)
            assert np.array_equal(out[j].view(np.uint32), want.view(np.uint32)), (case, steps, j)
    assert ran >= 25, ran
