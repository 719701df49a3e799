import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2101_12127_b200 import pipeline as dp
src = dp.Source.synthetic_images(65536, 256, 256)
for depth in (2, 4, 8):
    reg = dp.Registry(); reg.register_random_crop_flip("crop"); reg.register_normalize("norm")
    g, _ = dp.Dataset.tensor_slices(reg, src).shuffle(10000, 42).map("crop").map("norm").batch(256).repeat(-1).prefetch(depth).optimize()
    it = dp.make_iterator(g, seed_override=1)
    for _ in range(16): it.get_next().release()
    torch.cuda.synchronize()
    tg = tr = 0.0; n = 256
    t0 = time.perf_counter()
    for _ in range(n):
        a = time.perf_counter(); b = it.get_next(); c = time.perf_counter(); b.release(); d = time.perf_counter()
        tg += c - a; tr += d - c
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"depth {depth} (actual {it.prefetch_depth}): get_next {1e6*tg/n:.1f} us, release {1e6*tr/n:.1f} us, wall {1e6*(t2-t0)/n:.1f} us/step", flush=True)
    del it
