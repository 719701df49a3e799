"""Tuning sweep for the K3/K4 fast path (stages x band rows), CUDA events.
    python tools/dev/ksweep.py k3|k4|k4p STAGES,.. BANDS,..   (k4p: periodic-tap K4)"""
import ctypes, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2101_12127_b200 import _capi as K
MEAN = (123.675, 116.28, 103.53); STD = (58.395, 57.12, 57.375)
vp = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
dev = torch.device("cuda:0"); s = torch.cuda.current_stream(); S = ctypes.c_void_p(s.cuda_stream); L = K.lib()
m3, s3 = K.floats3(MEAN), K.floats3(STD)
which = sys.argv[1]
hw, per_img = (256, 752640) if which == "k3" else (320, 909312)
N = 32768
imgs = torch.empty((N, hw, hw, 3), dtype=torch.uint8, device=dev)
K.check(L.dp_k_synth_images(vp(imgs), 0, N, hw * hw * 3, 0x5EED, S))
order = torch.randperm(N, device=dev)
D = 4
outs = [torch.empty((256, 224, 224, 3), dtype=torch.float32, device=dev) for _ in range(D)]
ids = [torch.empty(256, dtype=torch.int64, device=dev) for _ in range(D)]
def run(i):
    b = i % (N // 256)
    if which == "k3":
        K.check(L.dp_k_crop_flip_normalize_batch(vp(imgs), N, 256, 256, vp(order), b * 256, 256, 7, 224, 224, 1, m3, s3, vp(ids[i % D]), vp(outs[i % D]), S))
    else:
        K.check(L.dp_k_resize_normalize_batch(vp(imgs), N, 320, 320, vp(order), b * 256, 256, 224, 224, m3, s3, vp(ids[i % D]), vp(outs[i % D]), S))
res = []
for stages in sys.argv[2].split(","):
    for band in sys.argv[3].split(","):
        os.environ["DP_DEV_STAGES"] = stages
        os.environ[{"k3": "DP_DEV_CROP_BAND", "k4": "DP_DEV_RESIZE_BAND", "k4p": "DP_DEV_RESIZE_PBAND"}[which]] = band
        os.environ["DP_DEV_RESIZE_PERIODIC"] = "1" if which == "k4p" else "0"
        for i in range(5): run(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for i in range(128): run(i)
        e1.record(s); e1.synchronize()
        ms = e0.elapsed_time(e1) / 128
        r = {"k": which, "stages": int(stages), "band": int(band), "ms": round(ms, 5), "GBps": round(256 * per_img / ms / 1e6, 1)}
        print(json.dumps(r), flush=True)
