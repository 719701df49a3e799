"""dev: the batch-stage CUDA-event time of a token config's epoch launch
with the stream idle at launch (as in bench.py's window) vs queued behind a
~2 ms sleep kernel (launch latency hidden)."""
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2101_12127_b200 import pipeline as dp  # noqa: E402

for name in sys.argv[1:] or ["cfg4r", "cfg4b", "cfg4"]:
    cfg = dict(bench.CFG[name])
    g, _ = bench.build_other_graph(dp, cfg, 0, 0, 1)
    it = dp.make_iterator(g, seed_override=1)
    per = int(re.search(r"elements, (\d+) batches", it.describe()).group(1))
    st = torch.cuda.ExternalStream(it.stream)
    it.skip(3 * per)
    torch.cuda.synchronize()
    for mode in ("idle", "gated", "idle", "gated"):
        ns0, k0 = it.batch_stage_timing()
        for _ in range(5):
            torch.cuda.synchronize()
            if mode == "gated":
                with torch.cuda.stream(st):
                    torch.cuda._sleep(4_000_000)
            it.skip(per)
        torch.cuda.synchronize()
        ns1, k1 = it.batch_stage_timing()
        print(name, mode, "us/launch", round((ns1 - ns0) / max(k1 - k0, 1) / 1e3, 1), "launches", k1 - k0, flush=True)
    del it
