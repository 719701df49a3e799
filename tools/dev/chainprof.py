"""Runs a few launch groups of a bench chain config (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2101_12127_b200 import pipeline as dp  # noqa: E402

cfg = dict(bench.CFG[sys.argv[1] if len(sys.argv) > 1 else "cfg2rrc"])
cfg["n"] = 16384
src = dp.Source.synthetic_images(cfg["n"], *cfg["in_hw"])
g, _ = bench.build_graph(dp, cfg, src)
it = dp.make_iterator(g, seed_override=1, launch_batches=4)
it.skip(24)
torch.cuda.synchronize()
ns, k = it.batch_stage_timing()
print("us per batch", ns / 1e3 / (k * 4))
