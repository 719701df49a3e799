"""bench.run_e2e_tokens alone (profiling the token e2e leg)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2101_12127_b200 import pipeline as dp  # noqa: E402

cfg = dict(bench.CFG[sys.argv[1]])
args = argparse.Namespace(steps=64, warmup=8)
print(json.dumps(bench.run_e2e_tokens(dp, cfg, 0, args, 1, torch.device("cuda", 0))))
