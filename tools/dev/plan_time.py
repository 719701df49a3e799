"""dev: per-epoch plan build time of a token config (helper thread) vs the
host's GetNext time per epoch (DP_DEBUG_TIMING line at iterator teardown)."""
import os
import re
import sys
import time

os.environ["DP_DEBUG_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2101_12127_b200 import pipeline as dp  # noqa: E402

for name in sys.argv[1:] or ["cfg4", "cfg4r", "cfg4b"]:
    cfg = dict(bench.CFG[name])
    g, _ = bench.build_other_graph(dp, cfg, 0, 0, 1)
    it = dp.make_iterator(g, seed_override=1)
    per = int(re.search(r"elements, (\d+) batches", it.describe()).group(1))
    it.skip(2 * per)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it.skip(10 * per)
    torch.cuda.synchronize()
    print(name, "us per epoch", round((time.perf_counter() - t0) / 10 * 1e6, 1), flush=True)
    del it
    sys.stderr.flush()

# per-node self time (CUDA events) over the epochs above: which plan op dominates
for name in sys.argv[1:] or ["cfg4b"]:
    cfg = dict(bench.CFG[name])
    g, _ = bench.build_other_graph(dp, cfg, 0, 0, 1)
    it = dp.make_iterator(g, seed_override=1)
    per = int(re.search(r"elements, (\d+) batches", it.describe()).group(1))
    it.skip(12 * per)
    torch.cuda.synchronize()
    for row in it.metrics():
        print(name, row[1], "self us per epoch", round(row[2] / 12 / 1e3, 1))
    del it
