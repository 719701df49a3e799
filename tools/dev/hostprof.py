"""Host-side cost of GetNext through the Python/ctypes binding vs device time."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2101_12127_b200 import pipeline as dp
import bench
cfg = bench.CFG["cfg2"]
src = dp.Source.synthetic_images(65536, 256, 256)
g, _ = bench.build_graph(dp, cfg, src)
it = dp.make_iterator(g, seed_override=1)
for _ in range(16): it.get_next().release()
torch.cuda.synchronize()
t0 = time.perf_counter(); n = 512
for _ in range(n): it.get_next().release()
t1 = time.perf_counter()
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host issue {1e6*(t1-t0)/n:.1f} us/step, wall incl. drain {1e6*(t2-t0)/n:.1f} us/step, depth {it.prefetch_depth}")
ns, k = it.batch_stage_timing(); print("kernel avg us", ns / k / 1e3)
# raw C-ABI cost without python Batch wrapper
import ctypes
b = dp.dp_batch(); Lb = dp.L()
t0 = time.perf_counter()
for _ in range(n):
    Lb.dp_iterator_get_next(it.h, ctypes.byref(b)); Lb.dp_batch_release(ctypes.byref(b))
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"raw ctypes: host {1e6*(t1-t0)/n:.1f} us/step, wall {1e6*(t2-t0)/n:.1f} us/step")
