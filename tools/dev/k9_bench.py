"""K9 non-resize chains (crop-only u8, crop + pixel ops): dev timing, fraction of 6.46 TB/s."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2101_12127_b200 import _capi as K  # noqa: E402

MEAN, STD = (123.675, 116.28, 103.53), (58.395, 57.12, 57.375)
n, rows = 2048, 4096
imgs = torch.randint(0, 256, (n, 256, 256, 3), dtype=torch.uint8, device="cuda")
order = torch.randint(0, n, (rows,), dtype=torch.int64, device="cuda")
for name, steps in [("center crop 224 (u8)", [("center_crop", 224, 224)]),
                    ("random crop 224 + flip (u8)", [("random_crop", 224, 224, 7, True)]),
                    ("crop 224 + affine (fp32)", [("random_crop", 224, 224, 7, True),
                                                  ("affine", (1 / 255,) * 3, (0, 0, 0))]),
                    ("crop 224 + affine + normalize", [("random_crop", 224, 224, 7, True),
                                                       ("affine", (1 / 255,) * 3, (0, 0, 0)),
                                                       ("normalize", (0.5,) * 3, (0.25,) * 3)])]:
    c = K.ImageChain.from_steps(steps, 256, 256)
    oh, ow, f = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    K.check(K.lib().dp_image_chain_output(ctypes.byref(c), ctypes.byref(oh), ctypes.byref(ow), ctypes.byref(f)))
    el = 4 if f.value else 1
    out = torch.empty(rows * oh.value * ow.value * 3 * el, dtype=torch.uint8, device="cuda")
    ids = torch.empty(rows, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()

    def launch():
        K.check(K.lib().dp_k_image_chain_batch(ctypes.c_void_p(imgs.data_ptr()), n, ctypes.c_void_p(order.data_ptr()),
                                               0, rows, 0, 1, 1, ctypes.byref(c), ctypes.c_void_p(ids.data_ptr()),
                                               ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(s.cuda_stream)))
    launch()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    alg = rows * (oh.value * ow.value * 3 * (1 + el))
    print(f"{name:32s} {best:.3f} ms  {rows / best / 1e3:.2f} M img/s  {alg / best / 1e6:.0f} GB/s  "
          f"frac {alg / best / 1e6 / 6457:.2f}", flush=True)
