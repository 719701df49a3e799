"""Runs one kernel family a few times on cfg-sized inputs (for ncu captures)."""
import ctypes, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2101_12127_b200 import _capi as K
MEAN = (123.675, 116.28, 103.53); STD = (58.395, 57.12, 57.375)
vp = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
which = sys.argv[1] if len(sys.argv) > 1 else "k3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda:0"); S = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream); L = K.lib()
m3, s3 = K.floats3(MEAN), K.floats3(STD)
N = 8192
hw = 256 if which in ("k3", "plan") else 320
imgs = torch.empty((N, hw, hw, 3), dtype=torch.uint8, device=dev)
K.check(L.dp_k_synth_images(vp(imgs), 0, N, hw * hw * 3, 0x5EED, S))
order = torch.randperm(N, device=dev)
outs = [torch.empty((256, 224, 224, 3), dtype=torch.float32, device=dev) for _ in range(4)]
ids = torch.empty(256, dtype=torch.int64, device=dev)
for i in range(iters):
    b = i % (N // 256)
    if which == "k3":
        K.check(L.dp_k_crop_flip_normalize_batch(vp(imgs), N, 256, 256, vp(order), b * 256, 256, 7, 224, 224, 1, m3, s3, vp(ids), vp(outs[i % 4]), S))
    elif which == "k4":
        K.check(L.dp_k_resize_normalize_batch(vp(imgs), N, 320, 320, vp(order), b * 256, 256, 224, 224, m3, s3, vp(ids), vp(outs[i % 4]), S))
    elif which == "plan":
        o = torch.empty(65536, dtype=torch.int64, device=dev)
        K.check(L.dp_k_shuffle_plan(65536, 10000, 12345, None, vp(o), None, S))
torch.cuda.synchronize()
print("ok", which)
