"""K10 general column map vs K9 / K4 on non-periodic ratios (dev timing)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2101_12127_b200 import _capi as K  # noqa: E402

MEAN, STD = (123.675, 116.28, 103.53), (58.395, 57.12, 57.375)


INPUTS = {}


def run(steps, hw, n=2048, rows=4096, reps=5, entry="chain"):
    if hw not in INPUTS:
        INPUTS[hw] = (torch.randint(0, 256, (n, hw[0], hw[1], 3), dtype=torch.uint8, device="cuda"),
                      torch.randint(0, n, (rows,), dtype=torch.int64, device="cuda"))
    imgs, order = INPUTS[hw]
    c = K.ImageChain.from_steps(steps, *hw)
    oh, ow, f = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    K.check(K.lib().dp_image_chain_output(ctypes.byref(c), ctypes.byref(oh), ctypes.byref(ow), ctypes.byref(f)))
    out = torch.empty((rows, oh.value, ow.value, 3), dtype=torch.float32, device="cuda")
    ids = torch.empty(rows, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()

    def launch():
        if entry == "k4":
            K.check(K.lib().dp_k_resize_normalize_batch(
                ctypes.c_void_p(imgs.data_ptr()), n, hw[0], hw[1], ctypes.c_void_p(order.data_ptr()), 0, rows,
                oh.value, ow.value, K.floats3(MEAN), K.floats3(STD), ctypes.c_void_p(ids.data_ptr()),
                ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream)))
            return
        K.check(K.lib().dp_k_image_chain_batch(ctypes.c_void_p(imgs.data_ptr()), n, ctypes.c_void_p(order.data_ptr()),
                                               0, rows, 0, 1, 1, ctypes.byref(c), ctypes.c_void_p(ids.data_ptr()),
                                               ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream)))
    launch()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    win_bytes = rows * out[0].numel() * 4
    return best, rows / best * 1e3, out


CASES = [
    ("rrc 176->224 (11:14, up)", (256, 256), [("random_crop", 176, 176, 7, True), ("resize", 224, 224),
                                               ("normalize", MEAN, STD)], "chain"),
    ("crop 240 -> 176 (15:11, down)", (256, 256), [("random_crop", 240, 240, 7, True), ("resize", 176, 176),
                                                    ("normalize", MEAN, STD)], "chain"),
    ("resize 300->224 (K4 entry)", (300, 304), [("resize", 224, 224), ("normalize", MEAN, STD)], "k4"),
    ("resize 180->224 (K4 entry, up)", (180, 192), [("resize", 224, 224), ("normalize", MEAN, STD)], "k4"),
]
for name, hw, steps, entry in CASES:
    res = {}
    for mode, env in (("K10 general", "1"), ("fallback", "0")):
        os.environ["DP_DEV_ROLL_GENERAL"] = env
        os.environ["DP_DEV_K4_GENERAL"] = env
        ms, ips, out = run(steps, hw, entry=entry)
        res[mode] = out.clone()
        print(f"{name:32s} {mode:12s}: {ms:.3f} ms per 4096 images, {ips / 1e6:.2f} M img/s", flush=True)
    print("   bit-identical:", torch.equal(res["K10 general"].view(torch.int32), res["fallback"].view(torch.int32)))
