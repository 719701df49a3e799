"""Kernel micro-timings (CUDA events on the launch stream) -- development aid."""
import ctypes, json, sys, time
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))))
from paper_2101_12127_b200 import _capi as K

MEAN = (123.675, 116.28, 103.53); STD = (58.395, 57.12, 57.375)
vp = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
dev = torch.device("cuda:0")
s = torch.cuda.current_stream(); S = ctypes.c_void_p(s.cuda_stream)
L = K.lib()
res = {}

def timeit(fn, iters, warm=3):
    for _ in range(warm): fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s)
    for i in range(iters): fn(i)
    e1.record(s); e1.synchronize()
    return e0.elapsed_time(e1) / iters

# cfg2: K3
N = 65536
imgs = torch.empty((N, 256, 256, 3), dtype=torch.uint8, device=dev)
K.check(L.dp_k_synth_images(vp(imgs), 0, N, 196608, 0x5EED, S))
order = torch.empty(N, dtype=torch.int64, device=dev)
from tests.oracle_lib import Oracle
orc = Oracle()
seed = orc.shuffle_seed(1, 42)
t = timeit(lambda i: K.check(L.dp_k_shuffle_plan(N, 10000, seed, None, vp(order), None, S)), 5, 1)
res["shuffle_plan_65536_ms"] = t
o1m = torch.empty(1 << 20, dtype=torch.int64, device=dev)
res["shuffle_plan_1M_ms"] = timeit(lambda i: K.check(L.dp_k_shuffle_plan(1000000, 10000, seed, None, vp(o1m), None, S)), 3, 1)
D = 4
outs = [torch.empty((256, 224, 224, 3), dtype=torch.float32, device=dev) for _ in range(D)]
ids = [torch.empty(256, dtype=torch.int64, device=dev) for _ in range(D)]
m3, s3 = K.floats3(MEAN), K.floats3(STD)
def k3(i):
    b = i % 256
    K.check(L.dp_k_crop_flip_normalize_batch(vp(imgs), N, 256, 256, vp(order), b * 256, 256, 7, 224, 224, 1, m3, s3, vp(ids[i % D]), vp(outs[i % D]), S))
t = timeit(k3, 256)
res["k3_ms_per_batch"] = t
res["k3_img_s"] = 256 / (t / 1e3)
res["k3_GBps"] = 256 * 752640 / (t / 1e3) / 1e9
print(json.dumps(res), flush=True)
del imgs
torch.cuda.empty_cache()
# cfg3: K4
N4 = 32768
imgs4 = torch.empty((N4, 320, 320, 3), dtype=torch.uint8, device=dev)
K.check(L.dp_k_synth_images(vp(imgs4), 0, N4, 307200, 0x5EED, S))
def k4(i):
    b = i % 128
    K.check(L.dp_k_resize_normalize_batch(vp(imgs4), N4, 320, 320, None, b * 256, 256, 224, 224, m3, s3, vp(ids[i % D]), vp(outs[i % D]), S))
t = timeit(k4, 128)
res["k4_ms_per_batch"] = t
res["k4_img_s"] = 256 / (t / 1e3)
res["k4_GBps"] = 256 * 909312 / (t / 1e3) / 1e9
del imgs4
torch.cuda.empty_cache()
# K1 at 2^28
n1 = 1 << 28
o = torch.empty(n1, dtype=torch.int64, device=dev)
t = timeit(lambda i: K.check(L.dp_k_range_affine_batch(0, n1, 3, 1, vp(o), S)), 10)
res["k1_2^28_ms"] = t; res["k1_GBps"] = n1 * 8 / (t / 1e3) / 1e9
print(json.dumps(res, indent=1))
