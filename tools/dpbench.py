"""dpbench for device pipelines: the reference's CLI loop (src/bench.cpp:
192-249 -- one warm-up epoch discarded, then the median of the measured
epochs, each a fresh iterator drained to EOF) over a pipeline description
file in the reference's stanza grammar with the device UDF library
(engine/pipeline_spec.cpp lists the stanzas).

    python tools/dpbench.py pipeline.txt [--device 0]
"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def rows_of(batch):
    shape = batch.components[0][1]
    if not shape:
        return 1  # unbatched element
    if len(batch.components) > 1 and batch.components[0][0].__name__ == "int32" and len(shape) == 1:
        return batch.components[1][1][0] - 1  # ragged: row splits
    return shape[0]


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("spec")
    ap.add_argument("--device", type=int, default=0)
    args = ap.parse_args()
    from paper_2101_12127_b200 import pipeline as dp
    reg = dp.Registry()
    with open(args.spec) as f:
        g, info = dp.Dataset.from_spec(reg, f.read(), device=args.device)
    g, report = g.optimize(info["disabled_rules"])
    print(f"optimized: {report.strip() or '(no rewrite)'}")
    times, elements = [], 0
    for epoch in range(info["epochs"] + 1):  # the first epoch is the warm-up
        it = dp.make_iterator(g, seed_override=info["seed"], device=args.device, deterministic=info["deterministic"])
        t0, n = time.perf_counter(), 0
        while (b := it.get_next()) is not None:
            n += rows_of(b)
            b.release()
        dt = time.perf_counter() - t0
        print(f"epoch {epoch}{' (warm-up)' if epoch == 0 else ''}: {n} elements in {dt * 1e3:.2f} ms "
              f"({n / dt:.4g} elements/s)")
        if epoch:
            times.append(dt)
            elements = n
    med = statistics.median(times)
    print(f"median epoch: {med * 1e3:.2f} ms, {elements / med:.4g} elements/s")


if __name__ == "__main__":
    main()
