"""Token e2e loop alone (bench run_e2e_tokens) for profiling."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2101_12127_b200 import pipeline as dp  # noqa: E402

cfg = dict(bench.CFG[sys.argv[1] if len(sys.argv) > 1 else "cfg4b"])
n_host = 200_000
rng = np.random.default_rng(1)
lens = rng.integers(1, 1025, n_host).astype(np.int32)
toks = rng.integers(0, 2 ** 31 - 1, int(lens.sum()), dtype=np.int64).astype(np.int32)
src = dp.Source.tokens_from_host(lens, toks, device=0, pinned=True)
g, _ = bench.build_other_graph(dp, cfg, 0, 0, 1, src=src)
it = dp.make_iterator(g, seed_override=1, host_output=True)
print(it.stats())
per = int(__import__("re").search(r"elements, (\d+) batches", it.describe()).group(1))
for _ in range(per):
    it.get_next().wait().release()
t0 = time.perf_counter()
ts = []
for k in range(2 * per):
    t = time.perf_counter()
    it.get_next().wait().release()
    ts.append(time.perf_counter() - t)
el = time.perf_counter() - t0
ts = np.array(ts)
slow = np.nonzero(ts > 0.02)[0]
print("slow batches", [(int(k), round(float(ts[k]) * 1e3, 1)) for k in slow][:10])
print(f"{2 * per} batches in {el * 1e3:.1f} ms; per batch median {np.median(ts) * 1e6:.1f} us, max {ts.max() * 1e3:.2f} ms, "
      f"top5 {np.sort(ts)[-5:] * 1e3}", it.stats())
