"""Per-launch fixed cost of the fused batch stage: cfg2 / cfg3 with exactly
g batches per launch (IteratorOptions::launch_batches), 320 timed batches.
Reports the stream-window time per batch and the kernel time per batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
from paper_2101_12127_b200 import pipeline as dp  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "crop"
groups = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,5,8,10,16,20").split(",")]
hw = 256 if mode == "crop" else 320
src = dp.Source.synthetic_images(65536, hw, hw)
for gsz in groups:
    reg = dp.Registry()
    if mode == "crop":
        reg.register_random_crop_flip("f", 224, 224, seed=7, flip=True)
    else:
        reg.register_resize_bilinear("f", 224, 224)
    reg.register_normalize("norm")
    g, _ = (dp.Dataset.tensor_slices(reg, src).shuffle(10000, 42).map("f").map("norm").batch(256).repeat(-1)
            .prefetch(-1).optimize())
    it = dp.make_iterator(g, seed_override=1, launch_batches=gsz)
    s = torch.cuda.ExternalStream(it.stream)
    n = 320 // gsz * gsz
    it.skip(2 * gsz)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ns0, k0 = it.batch_stage_timing()
    e0.record(s)
    it.skip(n)
    e1.record(s)
    e1.synchronize()
    ns1, k1 = it.batch_stage_timing()
    ms = e0.elapsed_time(e1)
    print(f"{mode} group {gsz:3d}: window {1e3 * ms / n:7.2f} us/batch ({n * 256 / ms / 1e3:.3f} M img/s)  "
          f"kernel {(ns1 - ns0) / 1e3 / max((k1 - k0) * gsz, 1):7.2f} us/batch  launches {k1 - k0}", flush=True)
    del it
