import sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2101_12127_b200 import pipeline as dp
src = dp.Source.synthetic_images(65536, 256, 256)
for mb, depth in [(800, 2), (1200, 2), (1600, 2), (2400, 2), (3200, 2), (1600, 3)]:
    os.environ["DP_DEV_GROUP_MB"] = str(mb)
    reg = dp.Registry(); reg.register_random_crop_flip("crop"); reg.register_normalize("norm")
    g, _ = dp.Dataset.tensor_slices(reg, src).shuffle(10000, 42).map("crop").map("norm").batch(256).repeat(-1).prefetch(depth).optimize()
    it = dp.make_iterator(g, seed_override=1)
    s = torch.cuda.ExternalStream(it.stream)
    for _ in range(16): it.get_next().release()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 512; ns0, k0 = it.batch_stage_timing()
    e0.record(s)
    for _ in range(n): it.get_next().release()
    e1.record(s); e1.synchronize()
    ns1, k1 = it.batch_stage_timing()
    ms = e0.elapsed_time(e1)
    print(f"group_mb {mb} depth {depth}: {1e3*ms/n:.2f} us/step  {n*256/ms*1e3/1e6:.3f} M img/s  kernel/batch {(ns1-ns0)/1e3/n:.2f} us  launches {k1-k0}", flush=True)
    del it
