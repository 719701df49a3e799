"""One epoch of a token config (for ncu on K5 / K8)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2101_12127_b200 import pipeline as dp  # noqa: E402

cfg = dict(bench.CFG[sys.argv[1] if len(sys.argv) > 1 else "cfg4r"])
g, _ = bench.build_other_graph(dp, cfg, 0, 0, 1)
it = dp.make_iterator(g, seed_override=1)
per = int(__import__("re").search(r"elements, (\d+) batches", it.describe()).group(1))
it.skip(2 * per)
torch.cuda.synchronize()
