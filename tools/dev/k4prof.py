"""A few cfg3 launch groups (for ncu on the K4 variants)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2101_12127_b200 import pipeline as dp  # noqa: E402

cfg = dict(bench.CFG["cfg3"])
cfg["n"] = 16384
src = dp.Source.synthetic_images(cfg["n"], *cfg["in_hw"])
g, _ = bench.build_graph(dp, cfg, src)
it = dp.make_iterator(g, seed_override=1, launch_batches=16)
it.skip(48)
torch.cuda.synchronize()
