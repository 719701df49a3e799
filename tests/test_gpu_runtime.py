"""Device-pipeline runtime properties on the GPU: bounded per-epoch state
under repeat(-1), slot reuse ordered after consumer-stream work when
batches are dropped on other threads, and output independent of the
prefetch depth and of the launch-group size (the reference's
P/tests/test_parallel.cpp:297-312: settings do not change the sequence).
"""
import queue
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2101_12127_b200 import pipeline
    return pipeline


def _token_graph(dp, kind, n=4000):
    reg = dp.Registry()
    reg.register_length_filter("len<=100", 100)
    src = dp.Source.synthetic_tokens(n, 200, 3, 3)
    g = dp.Dataset.token_sequences(reg, src).filter("len<=100").shuffle(500, 5)
    if kind == "padded":
        g = g.padded_batch(64)
    elif kind == "ragged":
        g = g.batch(64)
    else:
        g = g.bucket_by_length([30, 60], [32, 16, 8])
    return g.repeat(-1).prefetch(2), src


@pytest.mark.parametrize("kind", ["padded", "ragged", "bucket"])
def test_epoch_plans_are_retired_under_repeat(dp, kind):
    """the padded kinds prefetch the next epoch's plan; the
    old ones must still be retired.  25 epochs, <= 3 live plans throughout."""
    g, _ = _token_graph(dp, kind)
    it = dp.make_iterator(g, seed_override=1)
    per_epoch = int(__import__("re").search(r"elements, (\d+) batches", it.describe()).group(1))
    peak = 0
    for k in range(25 * per_epoch):
        it.get_next().release()
        if k % per_epoch == 0:
            peak = max(peak, it.stats()["live_plans"])
    assert peak <= 3, peak


def test_image_plans_are_retired_under_repeat(dp):
    reg = dp.Registry()
    reg.register_random_crop_flip("crop", 16, 16, seed=1, flip=True)
    reg.register_normalize("norm")
    src = dp.Source.synthetic_images(640, 24, 24)
    g, _ = (dp.Dataset.tensor_slices(reg, src).shuffle(100, 2).map("crop").map("norm").batch(64).repeat(-1)
            .optimize())
    it = dp.make_iterator(g, seed_override=1)
    for _ in range(30 * 10):
        it.get_next().release()
    assert it.stats()["live_plans"] <= 3


def test_slot_reuse_waits_for_consumer_stream_work_dropped_on_other_threads(dp):
    """batches are read by slow kernels on a consumer
    stream and dropped by worker threads; a slot may be rewritten only after
    the consumer work queued before its drop.  One batch per launch group
    and a depth-2 ring make reuse immediate; the per-batch checksums taken
    on the consumer stream must equal those of an undisturbed run."""
    import torch
    reg = dp.Registry()
    reg.register_random_crop_flip("crop", 32, 32, seed=3, flip=True)
    reg.register_normalize("norm")
    src = dp.Source.synthetic_images(4096, 40, 40)
    g, _ = (dp.Dataset.tensor_slices(reg, src).shuffle(1000, 9).map("crop").map("norm").batch(64).prefetch(2)
            .optimize())
    want = []
    for b in dp.make_iterator(g, seed_override=4, launch_batches=1):
        b.wait()
        want.append(float(b.torch(1).double().sum()))
        b.release()
    cs = torch.cuda.Stream()
    it = dp.make_iterator(g, seed_override=4, consumer_stream=cs.cuda_stream, launch_batches=1)
    assert it.stats()["group_batches"] == 1
    drops = queue.Queue()
    sums = []

    def dropper():
        while (b := drops.get()) is not None:
            b.release()

    workers = [threading.Thread(target=dropper) for _ in range(3)]
    for w in workers:
        w.start()
    with torch.cuda.stream(cs):
        while (b := it.get_next()) is not None:
            torch.cuda._sleep(200_000)  # the consumer is slower than the producer
            sums.append(b.torch(1).double().sum())
            drops.put(b)
    for _ in workers:
        drops.put(None)
    for w in workers:
        w.join()
    torch.cuda.synchronize()
    assert [float(s) for s in sums] == want


@pytest.mark.parametrize("depth", [1, 2, 8, -1])
@pytest.mark.parametrize("launch_batches", [0, 1, 3, 7])
def test_output_independent_of_prefetch_and_launch_group(dp, depth, launch_batches):
    """The same batches (ids and pixels, bit for bit) for prefetch 1/2/8/
    AUTOTUNE and any launch-group size (DP max_launch_bytes), across epoch
    boundaries (repeat 3, batches spanning epochs)."""
    reg = dp.Registry()
    reg.register_random_crop_flip("crop", 24, 24, seed=5, flip=True)
    reg.register_normalize("norm")
    src = dp.Source.synthetic_images(1000, 32, 32)
    g, _ = (dp.Dataset.tensor_slices(reg, src).shuffle(300, 1).map("crop").map("norm").repeat(3).batch(48)
            .prefetch(depth).optimize())
    key = ("base",)
    if key not in _REF:
        base = dp.make_iterator(g, seed_override=7)
        _REF[key] = [(b.numpy(0), b.numpy(1)) for b in base]
    # launch_batches 0: the default group, or (depth 8) 5 batches' bytes of max_launch_bytes
    mlb = 5 * 48 * (24 * 24 * 3 * 4 + 8) if (launch_batches == 0 and depth == 8) else 0
    got = []
    it = dp.make_iterator(g, seed_override=7, max_launch_bytes=mlb, launch_batches=launch_batches)
    if launch_batches:
        assert it.stats()["group_batches"] == launch_batches
    for b in it:
        got.append((b.numpy(0), b.numpy(1)))
        b.release()
    ref = _REF[key]
    assert len(got) == len(ref) == -(-3000 // 48)
    for (i0, p0), (i1, p1) in zip(ref, got):
        assert np.array_equal(i0, i1) and np.array_equal(p0.view(np.uint32), p1.view(np.uint32))


_REF = {}


@pytest.mark.parametrize("span", [False, True])
@pytest.mark.parametrize("tiling", [(4, 3), (5, 1), (2, 7)])
def test_output_independent_of_a_first_launch_head(dp, span, tiling):
    """IteratorOptions::first_launch_batches (the bench's exact-window
    tiling): a first launch of another size, then groups of launch_batches,
    per-epoch (batch -> repeat) and spanning (repeat -> batch) stages; also
    a checkpoint seek into the tiled stream."""
    reg = dp.Registry()
    reg.register_random_crop_flip("crop", 16, 16, seed=2, flip=True)
    reg.register_normalize("norm")
    src = dp.Source.synthetic_images(700, 20, 20)
    g = dp.Dataset.tensor_slices(reg, src).shuffle(200, 4).map("crop").map("norm")
    g = g.repeat(3).batch(32) if span else g.batch(32).repeat(3)
    g, _ = g.prefetch(-1).optimize()
    ref = [(b.numpy(0), b.numpy(1)) for b in dp.make_iterator(g, seed_override=3)]
    lb, head = tiling
    it = dp.make_iterator(g, seed_override=3, launch_batches=lb, first_launch_batches=head)
    got = [(b.numpy(0), b.numpy(1)) for b in it]
    assert len(got) == len(ref)
    for (i0, p0), (i1, p1) in zip(ref, got):
        assert np.array_equal(i0, i1) and np.array_equal(p0.view(np.uint32), p1.view(np.uint32))
    it = dp.make_iterator(g, seed_override=3, launch_batches=lb, first_launch_batches=head)
    for _ in range(11):
        it.get_next().release()
    rest = [(b.numpy(0), b.numpy(1)) for b in dp.restore(g, it.save(), launch_batches=lb, first_launch_batches=head)]
    assert len(rest) == len(ref) - 11
    for (i0, p0), (i1, p1) in zip(ref[11:], rest):
        assert np.array_equal(i0, i1) and np.array_equal(p0.view(np.uint32), p1.view(np.uint32))


def test_pinned_token_staging_across_epochs(dp, orc):
    """Pinned-host token sources are staged into device memory once per
    epoch plan (dp_k_stage_rows): over repeated epochs (plans built ahead
    on the helper thread, retired behind) and a checkpoint restore, the
    batches equal those of the same sequences in HBM."""
    lens = orc.lengths(2500, 700, 9)
    toks, _ = orc.tokens(lens, 9)
    reg = dp.Registry()
    reg.register_length_filter("len<=400", 400)
    outs = []
    for pinned in (False, True):
        src = dp.Source.tokens_from_host(lens, toks, pinned=pinned)
        base = dp.Dataset.token_sequences(reg, src).filter("len<=400").shuffle(500, 3)
        got = []
        for g in (base.padded_batch(40).repeat(3), base.batch(33).repeat(3),
                  base.bucket_by_length([100, 250], [24, 16, 8]).repeat(3)):
            got += [[b.numpy(0), b.numpy(1)] for b in dp.make_iterator(g, seed_override=2)]
            it = dp.make_iterator(g, seed_override=2)
            for _ in range(17):
                it.get_next().release()
            got += [[b.numpy(0), b.numpy(1)] for b in dp.restore(g, it.save())]
        outs.append(got)
    assert len(outs[0]) == len(outs[1])
    assert all(np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) for a, b in zip(*outs))


def test_autotuned_depth_follows_the_queue_model(dp):
    """AUTOTUNE: the ring depth comes from the
    reference's M/M/1/k model (PEmpty, model.cpp:29-42, 262-266) over the
    measured producer (CUDA-event device time per group) and consumer (host
    time per group) rates, inside slots pre-allocated at the first issue --
    a consumer at about the producer's rate gets the deepest ring, a much
    slower one the minimum and (the reference's test_parallel.cpp:169-190)
    no wait: the ring refills while it works.  Slots never grow."""
    import time
    reg = dp.Registry()
    reg.register_random_crop_flip("crop", 224, 224, seed=7, flip=True)
    reg.register_normalize("norm")
    src = dp.Source.synthetic_images(2048, 256, 256)
    g, _ = (dp.Dataset.tensor_slices(reg, src).shuffle(1000, 42).map("crop").map("norm").batch(64).repeat(-1)
            .prefetch(-1).optimize())

    def run(sleep_s, n=240):
        it = dp.make_iterator(g, seed_override=1, launch_batches=2)
        waits = []
        for k in range(n):
            b = it.get_next()
            t = time.perf_counter()
            b.wait()
            waits.append(time.perf_counter() - t)
            b.release()
            if sleep_s:
                time.sleep(sleep_s)
        return it.stats(), float(np.mean(waits[n // 2:]))

    fast, _ = run(0)
    assert fast["slots"] == fast["max_depth"] >= 3  # pre-allocated, never grown
    per_group = 1.0 / fast["producer_groups_per_s"]  # device seconds per launch group (2 batches)
    equal, _ = run(per_group / 2)  # the consumer takes a group about as fast as the device writes one
    slow, slow_wait = run(per_group * 10)
    def pempty(n, x, y):  # model.cpp:29-42
        r = x / y
        return 1.0 / (n + 1.0) if abs(r - 1.0) < 1e-9 else min(max((1.0 - r) / (1.0 - r ** (n + 1.0)), 0.0), 1.0)

    def model_depth(st):
        x, y, n = st["producer_groups_per_s"], st["consumer_groups_per_s"], 1
        while n + 1 < st["max_depth"]:
            p = pempty(n, x, y)
            if p <= 0.02 or p - pempty(n + 1, x, y) < 0.005:
                break
            n += 1
        return min(max(n + 1, 2), st["max_depth"])

    for st in (fast, equal, slow):
        assert st["slots"] == st["max_depth"]
        assert st["prefetch_depth"] == model_depth(st), st
    assert equal["prefetch_depth"] == equal["max_depth"] > slow["prefetch_depth"], (equal, slow)
    assert slow["p_empty"] < 0.02 and slow_wait < per_group / 4, (slow, slow_wait, per_group)


def test_metrics_rows_per_node(dp):
    """Metrics() (runtime.hpp:76): one row per graph node, root first, with
    CUDA-event self time for the device stages."""
    reg = dp.Registry()
    reg.register_random_crop_flip("crop", 24, 24, seed=1, flip=True)
    reg.register_normalize("norm")
    src = dp.Source.synthetic_images(1000, 32, 32)
    g, _ = (dp.Dataset.tensor_slices(reg, src).shard(2, 1).shuffle(300, 5).map("crop").map("norm").batch(50)
            .repeat(2).prefetch(-1).optimize())
    it = dp.make_iterator(g, seed_override=1)
    n = sum(1 for b in it)
    rows = it.metrics()
    paths = [r[0] for r in rows]
    assert paths[0].startswith("/prefetch@0") and paths[-1].endswith("tensor_slices@0"), paths
    by = {r[0].rsplit("/", 1)[1].split("@")[0]: r for r in rows}
    assert by["map_and_batch"][2] > 0 and by["map_and_batch"][3] == n == 20
    assert by["shuffle"][2] > 0 and by["shuffle"][3] == 1000  # 500 per epoch, 2 epochs planned
    assert by["shard"][3] == 1000
