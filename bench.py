#!/usr/bin/env python
"""bench.py -- pipeline elements/s of the B200 engine on BASELINE.json's
headline configuration, with roofline, CPU-baseline, clocks and end-to-end
numbers (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
    python bench.py --impl reference ...      # the reference CPU pipeline

Workload (default cfg2 = BASELINE.json configs[1], one GPU):
    synthetic 256x256x3 uint8 images (65,536 per GPU, HBM resident)
    -> shuffle(10,000, seed=42) -> map(random crop 224 + flip) -> map(normalize
    fp32) -> batch(256) -> repeat -> prefetch(AUTOTUNE), optimized to
    map_and_batch; base seed 1.  A step = one GetNext = one batch of 256.
    N > 1: weak scaling, each rank runs the same pipeline on its own
    65,536-image shard (images with global ids rank * 65,536 + i); no
    collective on the data path, a final 8-byte order-digest all_gather.

Timing: W untimed steps, then exactly K steps between CUDA events recorded
on the iterator's stream, barrier + synchronize on both sides, max over
ranks.  Inputs (12.9 GB per GPU) and the rotating output slots (>= 2 x 154
MB) exceed the 126 MB L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

IMG_BYTES_READ = 224 * 224 * 3          # crop window (uint8)
IMG_BYTES_WRITE = 224 * 224 * 3 * 4     # fp32 output
CFG = {
    "cfg2": dict(workload="synthetic 256x256x3 u8 images -> Shuffle(10k, seed 42) -> Map(random crop 224 + flip + "
                          "normalize fp32) -> Batch(256) -> Prefetch(AUTOTUNE)",
                 in_hw=(256, 256), out_hw=(224, 224), mode=0, batch=256, n=65536,
                 bytes_per_elem=IMG_BYTES_READ + IMG_BYTES_WRITE, kernel="K3 crop_flip_normalize_batch"),
    "cfg3": dict(workload="synthetic 320x320x3 u8 images -> Shuffle(10k, seed 42) -> Map(bilinear resize 320->224 + "
                          "normalize fp32) -> Batch(256) -> Prefetch(AUTOTUNE)",
                 in_hw=(320, 320), out_hw=(224, 224), mode=1, batch=256, n=65536,
                 bytes_per_elem=320 * 320 * 3 + IMG_BYTES_WRITE,
                 kernel="K10 image_chain_roll (dp_k_resize_normalize_batch)"),
    "cfg5": dict(workload="Shard(N) over 32*N synthetic record files of 2048 256x256x3 u8 images (each GPU holds "
                          "only its 32 files) -> Interleave(cycle 4, parallel 4) -> Shuffle(10k, seed 42) -> Map(random "
                          "crop 224 + flip + normalize fp32) -> Batch(256) -> Prefetch(AUTOTUNE)",
                 in_hw=(256, 256), out_hw=(224, 224), mode=0, batch=256, n=65536, files=32, cycle=4,
                 bytes_per_elem=IMG_BYTES_READ + IMG_BYTES_WRITE, kernel="K3 crop_flip_normalize_batch"),
    # the widened UDF library (K9): no map, RandomResizedCrop, ResNet eval
    "cfg2u8": dict(workload="synthetic 256x256x3 u8 images -> Shuffle(10k, seed 42) -> Batch(256) (no map: the u8 "
                            "images themselves)",
                   in_hw=(256, 256), out_hw=(256, 256), batch=256, n=65536, udfs=[], out_f32=False,
                   bytes_per_elem=2 * 196608, kernel="K9 gather_copy_batch", dtype="u8"),
    "cfg2rrc": dict(workload="synthetic 256x256x3 u8 images -> Shuffle(10k, seed 42) -> Map(random crop 160x160 + "
                             "flip) -> Map(bilinear resize 224) -> Map(normalize fp32) -> Batch(256) "
                             "(RandomResizedCrop at a fixed scale)",
                    in_hw=(256, 256), out_hw=(224, 224), batch=256, n=65536,
                    udfs=[("random_crop", 160, 160, 7, True), ("resize", 224, 224), ("normalize",)],
                    bytes_per_elem=160 * 160 * 3 + IMG_BYTES_WRITE,
                    kernel="K10 image_chain_roll (dp_k_image_chain_batch)"),
    "cfg3e": dict(workload="synthetic 320x320x3 u8 images -> Shuffle(10k, seed 42) -> Map(bilinear resize 256) -> "
                           "Map(center crop 224) -> Map(normalize fp32) -> Batch(256) (ResNet eval)",
                  in_hw=(320, 320), out_hw=(224, 224), batch=256, n=65536,
                  udfs=[("resize", 256, 256), ("center_crop", 224, 224), ("normalize",)],
                  # source rows / columns 20..299 feed the center window: 280 x 280 x 3 read
                  bytes_per_elem=280 * 280 * 3 + IMG_BYTES_WRITE,
                  kernel="K10 image_chain_roll (dp_k_image_chain_batch)"),
    "cfg1": dict(workload="Range(2^28) int64 -> Map(x*3+1) -> Batch(1024) (cfg1 shape at the roofline size "
                          "SURVEY.md 8(d) names; Range(1M) is the parity case)",
                 kind="range", batch=1024, n=1 << 28, bytes_per_elem=8, kernel="K1 range_affine_batch",
                 unit="elements/s", dtype="int64"),
    "cfg4": dict(workload="1M int32 token sequences, len U[1,1024] -> Filter(len<=512) -> PaddedBatch(128, pad 0)",
                 kind="tokens", batch=128, n=1_000_000, max_keep=512, kernel="K5 padded_batches",
                 unit="sequences/s", dtype="int32"),
    "cfg4r": dict(workload="1M int32 token sequences, len U[1,1024] -> Filter(len<=512) -> Batch(128) (the "
                           "reference's own cfg4 graph: ragged batches, values + int64 row splits)",
                  kind="tokens", batch=128, n=1_000_000, max_keep=512, kernel="K5 ragged_batches",
                  unit="sequences/s", dtype="int32", ragged=True),
    "cfg4b": dict(workload="1M int32 token sequences, len U[1,1024] -> Filter(len<=512) -> Shuffle(10k, seed 42) -> "
                           "BucketByLength(boundaries 128/256/384, batch sizes 256/128/96/64, pad 0)",
                  kind="tokens", batch=128, n=1_000_000, max_keep=512, kernel="K8 bucket_batches",
                  unit="sequences/s", dtype="int32", bucket=([128, 256, 384], [256, 128, 96, 64])),
}
for _c in CFG.values():
    _c.setdefault("kind", "images")
    _c.setdefault("unit", "images/s")
    _c.setdefault("dtype", "u8->f32")


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 4 + k and r[4 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def config_dict(cfg, world):
    """The `config` object of both arms' JSON lines (same keys and values)."""
    if cfg["kind"] == "images":
        l2 = (f"inputs {cfg['n'] * cfg['in_hw'][0] * cfg['in_hw'][1] * 3 / 1e9:.1f} GB/GPU and the rotating output "
              f"slots exceed the 126 MB L2 (no flush needed)")
    else:
        l2 = "one launch = one epoch of output (> 126 MB L2); no flush needed"
    return {"workload": cfg["workload"], "global_batch": cfg["batch"] * world, "elements_per_gpu": cfg["n"],
            "parallelism": f"dp{world} (Shard, no data-path collective)", "l2": l2}


def expected_order_digest(config, n, world, rank):
    """tests/golden/order_check.json (generated by the oracle restatement)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "order_check.json")) as f:
            return json.load(f)["entries"].get(f"{config}/n{n}/w{world}/r{rank}")
    except (OSError, ValueError, KeyError):
        return None


def group_boundary(x, d, head, batches_per_epoch):
    """Is batch x the first batch of a launch group?  Groups of d batches tile
    each epoch from its start; with a head, epoch 0's first group holds
    `head` batches (IteratorOptions::first_launch_batches)."""
    e, k = divmod(x, batches_per_epoch)
    if k == 0:
        return True
    if e == 0 and head:
        return k == head or (k > head and (k - head) % d == 0)
    return k % d == 0


def launch_tiling_for(warmup, steps, max_group, batches_per_epoch):
    """(batches per launch, first-launch batches) with launch boundaries on
    both ends of the timed window [warmup, warmup + steps), so the window
    holds exactly `steps` batches: the largest group up to max_group, the
    warm-up as a head group when that is what makes it fit."""
    for d in range(min(max_group, batches_per_epoch), 0, -1):
        for head in (0, warmup):
            if head >= batches_per_epoch:
                continue
            if group_boundary(warmup, d, head, batches_per_epoch) and \
                    group_boundary(warmup + steps, d, head, batches_per_epoch):
                return d, head
    return 1, 0


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---- multi-rank plumbing (nccl on the GPU box; gloo in tests/test_multiproc.py) ----
def shard_layout(world, rank, n_per_rank):
    """Weak scaling: the global dataset has world * n_per_rank elements; rank
    r holds and processes shard(world, r) -- positions p % world == r."""
    global_count = world * n_per_rank
    return {"global_count": global_count, "num_shards": world, "index": rank,
            "resident": (global_count - rank + world - 1) // world}


def _coll_device(device):
    """gloo collectives run on host tensors (CPU tests, or the one-GPU
    multi-process rehearsal of the multi-rank path); nccl on the GPU."""
    import torch.distributed as distr
    return "cpu" if distr.is_initialized() and distr.get_backend() == "gloo" else device


def max_over_ranks(ms, world, device):
    import torch
    import torch.distributed as distr
    t = torch.tensor([ms], device=_coll_device(device), dtype=torch.float64)
    if world > 1:
        distr.all_reduce(t, op=distr.ReduceOp.MAX)
        distr.barrier()
    return float(t.item())


def gather_digests(digest, world):
    """The final ordering check: every rank's 8-byte order digest."""
    import torch
    import torch.distributed as distr
    digest = digest.to(_coll_device(digest.device))
    digests = [digest]
    if world > 1:
        digests = [torch.zeros_like(digest) for _ in range(world)]
        distr.all_gather(digests, digest)
    return [f"{int(d.item()) & (2**64 - 1):016x}" for d in digests]


# ---------------------------------------------------------------- CPU side --
def cpu_reference(cfg, threads, warmup_batches, steps):
    """The compiled reference pipeline (oracle/_ref) on this host's cores."""
    from tests.oracle_lib import Reference
    import ctypes
    ref = Reference.load()
    if ref is None:
        return None
    L = ref.L
    i64, u64 = ctypes.c_int64, ctypes.c_uint64
    L.ref_time_image_steps.argtypes = [ctypes.c_int] * 5 + [u64, u64, i64, i64, u64, i64, i64, i64, i64,
                                                             ctypes.c_void_p, ctypes.c_void_p]
    secs, elems = ctypes.c_double(), i64()
    sample = 2048
    if "udfs" in cfg:  # the chain configs: one reference map node per step
        from tests.oracle_lib import steps_array
        st = chain_steps(cfg["udfs"])
        L.ref_time_chain_steps.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u64, i64, i64,
                                           u64, i64, i64, i64, i64, ctypes.c_void_p, ctypes.c_void_p]
        rc = L.ref_time_chain_steps(steps_array(st), len(st), *cfg["in_hw"], 0x5EED, sample, 10000, 42, cfg["batch"],
                                    threads, warmup_batches, steps, ctypes.byref(secs), ctypes.byref(elems))
        what = f"{sample} resident synthetic images repeated, one reference map per chain step"
    elif cfg.get("files"):  # cfg5: the reference's interleave over record readers
        L.ref_time_interleave_image_steps.argtypes = [ctypes.c_int] * 5 + [u64, u64] + [i64] * 5 + [
            i64, u64, i64, i64, i64, i64, ctypes.c_void_p, ctypes.c_void_p]
        rec = cfg["n"] // cfg["files"]
        rc = L.ref_time_interleave_image_steps(cfg["mode"], *cfg["in_hw"], *cfg["out_hw"], 7, 0x5EED, sample,
                                               cfg["files"], rec, cfg["cycle"], cfg["cycle"], 10000, 42, cfg["batch"],
                                               threads, warmup_batches, steps, ctypes.byref(secs),
                                               ctypes.byref(elems))
        what = (f"interleave(cycle {cfg['cycle']}, parallel {cfg['cycle']}) over {cfg['files']} readers of {rec} "
                f"records copied from {sample} resident synthetic images")
    else:
        rc = L.ref_time_image_steps(cfg["mode"], *cfg["in_hw"], *cfg["out_hw"], 7, 0x5EED, sample, 10000, 42,
                                    cfg["batch"], threads, warmup_batches, steps, ctypes.byref(secs),
                                    ctypes.byref(elems))
        what = f"{sample} resident synthetic images repeated"
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return {"value": elems.value / secs.value, "seconds": secs.value, "elements": elems.value, "cores": threads,
            "sample": f"{what}, {steps} timed batches of {cfg['batch']} after {warmup_batches} warm-up, "
                      f"map_and_batch num_parallel_calls={threads}, prefetch(AUTOTUNE)"}


def cpu_reference_range(cfg):
    """cfg1 on the compiled reference: Range(1M) -> Map -> Batch(1024), optimized."""
    from tests.oracle_lib import Reference
    ref = Reference.load()
    if ref is None:
        return None
    n = 1_000_000
    eps = ref.time_range_map_batch(n, cfg["batch"], 1, epochs=3)
    return {"value": n / float(sorted(eps)[1]), "cores": 1, "sample": f"Range({n}) -> Map(x*3+1, p=1) -> Batch(1024), "
                                                          f"median of 3 epochs after 1 warm-up"}


def cpu_reference_tokens(cfg):
    """cfg4 on the compiled reference: sequences -> Filter(len<=512) -> Batch(128)
    (its ragged Batch: the same selection and order as PaddedBatch), one thread."""
    from tests.oracle_lib import Reference
    ref = Reference.load()
    if ref is None:
        return None
    n = 10_000  # the reference holds every token as a heap Value: a bounded sample
    eps = ref.time_filter_batch_tokens(n, 4, 1024, 4, cfg["max_keep"], cfg["batch"], epochs=3)
    return {"value": n / float(sorted(eps)[1]), "cores": 1,
            "sample": f"{n} sequences (len U[1,1024], seed 4) -> Filter(len<=512) -> Batch(128), median of 3 "
                      f"epochs after 1 warm-up"}


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if cfg["kind"] == "images":
        r = cpu_reference(cfg, threads, args.warmup, args.steps)
    else:  # the reference's sequential path (map p=1 / filter + batch): one host thread
        r = cpu_reference_range(cfg) if cfg["kind"] == "range" else cpu_reference_tokens(cfg)
        threads = 1
        r.setdefault("seconds", 1.0 / r["value"] * cfg["batch"] * args.steps)
    line = {"impl": "reference", "metric": "pipeline elements/sec", "value": round(r["value"], 2),
            "unit": cfg["unit"], "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * r["seconds"] / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg.get("dtype", "u8->f32"), "data": "synthetic",
            "config": config_dict(cfg, world),
            "cpu_baseline": {"value": round(r["value"], 2), "unit": cfg["unit"], "cores": threads,
                             "kind": "reference", "sample": r["sample"], "cpu_model": cpu_model(),
                             "host_threads": os.cpu_count()},
            "e2e": {"value": round(r["value"], 2), "unit": cfg["unit"], "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU side --
def register_udfs(dp, reg, udfs):
    names = []
    for i, st in enumerate(udfs):
        name = f"u{i}_{st[0]}"
        if st[0] == "random_crop":
            reg.register_random_crop_flip(name, st[1], st[2], seed=st[3], flip=st[4])
        elif st[0] == "center_crop":
            reg.register_center_crop(name, st[1], st[2])
        elif st[0] == "resize":
            reg.register_resize_bilinear(name, st[1], st[2])
        elif st[0] == "normalize":
            reg.register_normalize(name)
        names.append(name)
    return names


def chain_steps(udfs):
    """bench udfs -> the oracle's step tuples (tests/oracle_lib.steps_array)."""
    from tests.oracle_lib import MEAN, STD
    return [(st[0], MEAN, STD) if st[0] == "normalize" else st for st in udfs]


def build_graph(dp, cfg, src, repeat=True, shard=None, files=None):
    reg = dp.Registry()
    if "udfs" in cfg:
        names = register_udfs(dp, reg, cfg["udfs"])
    else:
        names = [reg.register_resize_bilinear("resize", *cfg["out_hw"]) if cfg["mode"] == 1
                 else reg.register_random_crop_flip("crop", *cfg["out_hw"], seed=7, flip=True),
                 reg.register_normalize("norm")]
    if cfg.get("files"):  # cfg5: Shard over the record files, then Interleave their readers
        files = files or cfg["files"] * (shard[0] if shard else 1)
        reg.register_record_reader("reader", cfg["n"] // cfg["files"])
        g = dp.Dataset.range(reg, files)
        if shard:
            g = g.shard(*shard)
        g = g.interleave("reader", cfg["cycle"], cfg["cycle"], records=src)
    else:
        g = dp.Dataset.tensor_slices(reg, src)
        if shard:
            g = g.shard(*shard)  # Shard(k, rank) right after the source
    g = g.shuffle(10000, 42)
    for nm in names:
        g = g.map(nm, -1)
    g = g.batch(cfg["batch"])
    if repeat:
        g = g.repeat(-1)
    g, report = g.prefetch(-1).optimize()
    return g, report


def build_other_graph(dp, cfg, local, rank, world, src=None):
    reg = dp.Registry()
    if cfg["kind"] == "range":  # cfg1
        reg.register_affine("affine(3,1)", 3, 1)
        g = dp.Dataset.range(reg, cfg["n"] * world)
        if world > 1:
            g = g.shard(world, rank)
        g = g.map("affine(3,1)").batch(cfg["batch"]).repeat(-1).prefetch(-1)
    else:  # cfg4 tokens
        reg.register_length_filter("len<=512", cfg["max_keep"])
        if src is None:
            src = dp.Source.synthetic_tokens(cfg["n"], 1024, 4 + rank, 4 + rank, device=local)
        g = dp.Dataset.token_sequences(reg, src).filter("len<=512")
        if cfg.get("bucket"):  # cfg4b
            g = g.shuffle(10000, 42).bucket_by_length(*cfg["bucket"])
        elif cfg.get("ragged"):  # cfg4r: the reference graph, Batch of sequences
            g = g.batch(cfg["batch"])
        else:
            g = g.padded_batch(cfg["batch"])
        g = g.repeat(-1).prefetch(-1)
    return g.optimize()


def padded_stats(dp, g, local):
    """cfg4 / cfg4b per-batch averages over one epoch: algorithmic bytes of
    K5 padded_batches / K8 bucket_batches (reads = kept tokens + (order,
    length, offset) per row; writes = the padded rows + lengths -- padding is
    the output, so it counts) and rows (the sequences a batch carries)."""
    it = dp.make_iterator(g, seed_override=1, device=local)
    per_epoch = int(re.search(r"elements, (\d+) batches", it.describe()).group(1))
    total = rows_total = 0
    for _ in range(per_epoch):
        b = it.get_next()
        if len(b.components[0][1]) == 1:  # ragged: (values, row splits)
            splits = b.numpy(1)
            rows, toks = splits.size - 1, int(splits[-1])
            total += 4 * toks + rows * (8 + 4 + 8) + 4 * toks + 8 * (rows + 1)
        else:
            lens = b.numpy(1)
            rows, lmax = b.components[0][1]
            total += 4 * int(lens.sum()) + rows * (8 + 4 + 8) + 4 * rows * lmax + 4 * rows
        rows_total += rows
        b.release()
    return total / per_epoch, rows_total / per_epoch


def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as distr
    from paper_2101_12127_b200 import pipeline as dp

    rank, world, local = dist_env()
    # DP_BENCH_ONE_GPU=1 rehearses the multi-rank path on a single GPU: every
    # rank uses cuda:0 and the (tiny) collectives go over gloo.  The ranks'
    # kernels never wait on one another (no data-path collective).
    rehearsal = os.environ.get("DP_BENCH_ONE_GPU") == "1"
    if rehearsal:
        local = 0
    if not rehearsal and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py --gpus {world}: only {torch.cuda.device_count()} CUDA device(s) visible")
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        if rehearsal:
            distr.init_process_group("gloo")
        else:
            distr.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = {"backend": distr.get_backend(), "world_size": distr.get_world_size(),
                "data_path_collectives": 0, "use": "barrier, max-over-ranks time, 8-byte digest all_gather"}
    dev = torch.device("cuda", local)

    # ---- device-resident workload (not timed) ----
    n = cfg["n"]
    if cfg["kind"] != "images":
        g, report = build_other_graph(dp, cfg, local, rank, world)
    elif cfg.get("files"):  # cfg5: each rank holds only the record files of its shard
        src = dp.Source.synthetic_records_sharded(cfg["files"] * world, n // cfg["files"], *cfg["in_hw"], world, rank,
                                                  seed=0x5EED, device=local)
        g, report = build_graph(dp, cfg, src, shard=(world, rank) if world > 1 else None)
    elif world > 1:  # each rank holds and processes shard `rank` of a world * n dataset
        lay = shard_layout(world, rank, n)
        src = dp.Source.synthetic_images_sharded(lay["global_count"], *cfg["in_hw"], world, rank, seed=0x5EED,
                                                 device=local)
        g, report = build_graph(dp, cfg, src, shard=(world, rank))
    else:
        src = dp.Source.synthetic_images(n, *cfg["in_hw"], seed=0x5EED, device=local)
        g, report = build_graph(dp, cfg, src)
    it = dp.make_iterator(g, seed_override=1, device=local)
    desc = it.describe()
    per_launch = int(re.search(r"(\d+) batch\(es\) per launch", desc).group(1))
    per_epoch = int(re.search(r"epoch: \d+ elements, (\d+) batches", desc).group(1))
    steps_requested, warmup_requested = args.steps, args.warmup
    head_batches = 0
    if cfg["kind"] == "images":
        # exactly K timed and W warm-up steps: a launch group that tiles the
        # window (largest divisor-compatible group up to the default size)
        out_bytes = cfg["batch"] * (cfg["out_hw"][0] * cfg["out_hw"][1] * 3 * (4 if cfg.get("out_f32", True) else 1)
                                    + 8)
        group, head = launch_tiling_for(args.warmup, args.steps, max(per_launch, (3200 << 20) // out_bytes),
                                        per_epoch)
        if (group, head) != (per_launch, 0):
            del it
            it = dp.make_iterator(g, seed_override=1, device=local, launch_batches=group, first_launch_batches=head)
            per_launch = group
        head_batches = head
    else:
        # token / range configs launch a whole epoch of tiny batches at once:
        # the window is whole epochs (steps and warmup rounded up to them)
        if per_epoch % per_launch:
            per_launch = per_epoch
        args.steps = max(args.steps, per_launch)
        args.warmup = max(args.warmup, per_launch)
        args.warmup = -(-args.warmup // per_launch) * per_launch
        args.steps = -(-args.steps // per_launch) * per_launch
    stream = torch.cuda.ExternalStream(it.stream, device=dev)
    it.skip(args.warmup)  # GetNext in C++, batches dropped (no-op consumer)
    torch.cuda.synchronize(dev)
    if world > 1:
        distr.barrier()
    launches0, batches0 = it.kernel_launches, it.batches_launched
    ns0, k0 = it.batch_stage_timing()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        got = it.skip(args.steps)
        e1.record(stream)
        e1.synchronize()
    assert got == args.steps
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    launches = it.kernel_launches - launches0
    batches_in_window = it.batches_launched - batches0
    ns1, k1 = it.batch_stage_timing()
    ms_max = max_over_ranks(ms, world, dev)
    # The device work inside [e0, e1] is exactly the batch-stage launches
    # issued between the two events; with W and K multiples of the launch
    # group this is K batches (checked and reported).
    if cfg.get("bytes_per_elem"):
        bytes_per_batch, rows_per_batch = cfg["bytes_per_elem"] * cfg["batch"], cfg["batch"]
    else:  # token configs: the window is whole epochs (one launch group = one epoch)
        bytes_per_batch, rows_per_batch = padded_stats(dp, g, local)
    elems = batches_in_window * rows_per_batch * world
    value = elems / (ms_max / 1e3)
    kernel_s = (ns1 - ns0) / max(k1 - k0, 1) / 1e9  # per launch
    batches_per_launch = batches_in_window / max(k1 - k0, 1)
    peak, peak_src = load_peaks()
    achieved = bytes_per_batch * batches_per_launch / kernel_s / 1e9
    del it

    # ---- end to end through the C ABI with host buffers ----
    e2e = run_e2e(dp, cfg, local, args, world, dev) if cfg["kind"] == "images" else \
        run_e2e_tokens(dp, cfg, local, args, world, dev) if cfg["kind"] == "tokens" else {
            "value": None, "note": "cfg1's range is generated in-kernel: no host input to copy"}

    # ---- the final ordering check: K7 digest of each rank's
    # first 8 emitted batches of ids, gathered (8 bytes per rank over NCCL) ----
    import ctypes
    from paper_2101_12127_b200 import _capi
    vit = dp.make_iterator(g, seed_override=1, device=local)
    digest = torch.zeros(1, dtype=torch.int64, device=dev)
    pos = 0
    for _ in range(8):
        b = vit.get_next()
        comp = 1 if cfg["kind"] == "tokens" else 0  # ids / values, or the row lengths of padded batches
        dt, shape, ptr, _ = b.components[comp]
        fn = _capi.lib().dp_k_order_digest if dt == np.int64 else _capi.lib().dp_k_word_digest
        _capi.check(fn(ctypes.c_void_p(ptr), shape[0], pos, ctypes.c_void_p(digest.data_ptr()),
                       ctypes.c_void_p(vit.stream)))
        pos += shape[0]
        b.release()
    torch.cuda.synchronize(dev)
    order_digests = gather_digests(digest, world)
    expected = [expected_order_digest(args.config, n, world, r) for r in range(world)]
    order_ok = None if None in expected else all(a == b for a, b in zip(order_digests, expected))
    del vit

    if rank != 0:
        if world > 1:
            distr.destroy_process_group()
        return
    cpu = None
    try:
        # ~10 s of CPU work on the box's 16 threads: 192 timed batches of 256
        # (49,152 images) after 4 warm-up batches
        cpu = cpu_reference(cfg, os.cpu_count() or 1, 4, 192) if cfg["kind"] == "images" else \
            cpu_reference_range(cfg) if cfg["kind"] == "range" else cpu_reference_tokens(cfg)
    except Exception as ex:  # reported, not fatal
        cpu = {"value": None, "sample": f"unavailable: {ex}"}
    one_core = None
    if cfg["kind"] == "images" and cpu is not None and cpu.get("value"):
        try:  # also the 1-core number (num_parallel_calls = 1), ~2 s
            r1 = cpu_reference(cfg, 1, 1, 4)
            one_core = {"value": round(r1["value"], 2), "cores": 1, "sample": r1["sample"]}
        except Exception as ex:
            one_core = {"value": None, "sample": f"unavailable: {ex}"}
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:  # measured on one launch of `batches` batches; scaled to this run's launch size
            t = json.load(open(prof)).get(args.config)
            traffic = None if t is None else int(t["bytes"] * batches_per_launch / t["batches"])
        except Exception:
            traffic = None
    line = {
        "metric": "pipeline elements/sec", "value": round(value, 1), "unit": cfg["unit"], "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (device-generated, SplitMix64 / PCG32 keyed)",
        "config": config_dict(cfg, world),
        "lowering": {"optimized": "map_and_batch" in report or "map_batch_fusion" in report,
                     "batches_per_launch": per_launch, "first_launch_batches": head_batches or per_launch,
                     "prefetch_depth": "AUTOTUNE"},
        **({} if (steps_requested, warmup_requested) == (args.steps, args.warmup) else
           {"steps_requested": steps_requested, "warmup_requested": warmup_requested,
            "steps_note": "whole epochs of tiny batches (one launch per epoch)"}),
        "comm": comm,
        "roofline": {"bound": "hbm", "kernel": cfg["kernel"], "achieved": round(achieved, 1), "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "algorithmic_bytes_per_launch": int(bytes_per_batch * batches_per_launch),
                     "algorithmic_bytes_per_element": round(bytes_per_batch / cfg["batch"], 1),
                     "batches_per_launch": batches_per_launch,
                     "avg_launch_us": round(kernel_s * 1e6, 3), "launches_timed": k1 - k0, "traffic": traffic,
                     **({"note": "store-only stream (the range is generated in-kernel, 8 B written per element): "
                                 "write-only HBM traffic runs above the read+write copy figure used as peak"}
                        if cfg["kind"] == "range" else {})},
        "batches_in_window": batches_in_window, "steps_per_launch_group": per_launch,
        "order_check": {"digest": "K7 position-keyed digest of each rank's first 8 batches (ids / values / row "
                                  "lengths), vs tests/golden/order_check.json (oracle restatement)",
                        "per_rank": order_digests, "expected": expected, "ok": order_ok},
        "cpu_baseline": {"value": None if cpu is None else (round(cpu["value"], 2) if cpu["value"] else None),
                         "unit": cfg["unit"], "cores": (cpu or {}).get("cores", os.cpu_count()), "kind": "reference",
                         "sample": None if cpu is None else cpu["sample"], "one_core": one_core,
                         "cpu_model": cpu_model(), "host_threads": os.cpu_count()},
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        distr.destroy_process_group()


def pcie_gbs(local, h2d=False):
    """Plain pinned-memory copy bandwidth, 512 MiB, best of 5, CUDA events (D2H, or H2D)."""
    import torch
    try:
        n = 512 << 20
        d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        s = torch.cuda.Stream(device=local)
        best = 0.0
        with torch.cuda.stream(s):
            for i in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                if h2d:
                    d.copy_(h, non_blocking=True)
                else:
                    h.copy_(d, non_blocking=True)
                e1.record(s)
                e1.synchronize()
                if i:
                    best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        del d, h
        return round(best, 1)
    except Exception:  # reported, not fatal
        return None


def pcie_d2h_gbs(local):
    """Plain pinned-memory D2H copy bandwidth (512 MiB, best of 5, CUDA events): the e2e roofline."""
    import torch
    try:
        n = 512 << 20
        d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        s = torch.cuda.Stream(device=local)
        best = 0.0
        with torch.cuda.stream(s):
            h.copy_(d, non_blocking=True)
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                h.copy_(d, non_blocking=True)
                e1.record(s)
                e1.synchronize()
                best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        del d, h
        return round(best, 1)
    except Exception:  # reported, not fatal
        return None


def e2e_image_graph(dp, cfg, local, world):
    """The config's graph over a pinned-host image dataset (4,096 images, read
    by the kernels over PCIe)."""
    import numpy as np
    n_host = 4096
    h, w = cfg["in_hw"]
    host = np.random.default_rng(0).integers(0, 256, (n_host, h, w, 3), dtype=np.uint8)
    src = dp.Source.images_pinned_host(host, device=local)
    if cfg.get("files"):  # cfg5: each rank's pinned records = its shard's files of R records
        rec = cfg["n"] // cfg["files"]
        files = n_host // rec
        if world > 1:
            src = src.as_shard(files * world * rec, world, dist_env()[0], rec)
        g, _ = build_graph(dp, cfg, src, shard=(world, dist_env()[0]) if world > 1 else None, files=files * world)
    else:
        g, _ = build_graph(dp, cfg, src)
    return g, src, host


def run_e2e(dp, cfg, local, args, world=1, dev=None):
    """Same pipeline through the C ABI with HOST inputs: the image dataset
    lives in pinned host memory and every step's inputs cross PCIe (the
    kernels read them); each step's batch is consumed on the device by a
    consumer stream (a K7 digest over every output word -- the "loss" of a
    data pipeline feeding a GPU model) and that 8-byte result is read back
    by the host before the next step.  Host wall clock over K steps, the
    slowest rank's at N GPUs.  `host_batches` repeats the run with every
    batch copied back into pinned host memory instead (the output crossing
    PCIe too)."""
    import ctypes
    import torch
    from paper_2101_12127_b200 import _capi
    g, src, host = e2e_image_graph(dp, cfg, local, world)
    launch = int(os.environ.get("DP_E2E_LAUNCH_BYTES", 160 << 20))  # one batch per launch
    out_el = 4 if cfg.get("out_f32", True) else 1
    b_out_full = cfg["batch"] * (cfg["out_hw"][0] * cfg["out_hw"][1] * 3 * out_el + 8)
    b_in = cfg["batch"] * (cfg["bytes_per_elem"] - cfg["out_hw"][0] * cfg["out_hw"][1] * 3 * out_el)
    steps = max(8, min(args.steps, 64))

    cs = torch.cuda.Stream(device=local)
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    res = torch.zeros(1, dtype=torch.int64).pin_memory()
    L = _capi.lib()
    it = dp.make_iterator(g, seed_override=1, device=local, consumer_stream=cs.cuda_stream, max_launch_bytes=launch)

    def step():
        b = it.get_next()
        _, shape, ptr, _ = b.components[1]
        words = shape[0] * shape[1] * shape[2] * shape[3] * out_el // 4
        _capi.check(L.dp_k_word_digest(ctypes.c_void_p(ptr), words, 0, ctypes.c_void_p(acc.data_ptr()),
                                       ctypes.c_void_p(cs.cuda_stream)))
        with torch.cuda.stream(cs):
            res.copy_(acc, non_blocking=True)
        cs.synchronize()  # the host reads the step's result
        b.release()
        return int(res[0])

    for _ in range(3):
        step()
    if world > 1:
        max_over_ranks(0.0, world, dev)  # barrier: start together
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    secs = time.perf_counter() - t0
    if world > 1:
        secs = max_over_ranks(secs * 1e3, world, dev) / 1e3
    del it

    # the same with the batches copied to pinned host memory
    hit = dp.make_iterator(g, seed_override=1, device=local, host_output=True, max_launch_bytes=launch)
    for _ in range(3):
        hit.get_next().wait().release()
    if world > 1:
        max_over_ranks(0.0, world, dev)
    t0 = time.perf_counter()
    for _ in range(steps):
        hit.get_next().wait().release()
    hsecs = time.perf_counter() - t0
    if world > 1:
        hsecs = max_over_ranks(hsecs * 1e3, world, dev) / 1e3
    del hit
    return {"value": round(steps * cfg["batch"] * world / secs, 1), "unit": "images/s",
            "h2d_bytes_per_step": b_in * world, "d2h_bytes_per_step": 8 * world, "steps": steps,
            "pcie": {"h2d_gbs_achieved": round(steps * b_in / secs / 1e9, 1)},
            "how": "pinned host image source read over PCIe by the kernels (every step's inputs cross PCIe); the "
                   "batch consumed on the device by a consumer stream (K7 digest over every output word) and the "
                   "8-byte result read by the host each step; host wall clock",
            "host_batches": {
                "value": round(steps * cfg["batch"] * world / hsecs, 1), "unit": "images/s",
                "h2d_bytes_per_step": b_in * world, "d2h_bytes_per_step": b_out_full * world,
                "d2h_gbs_achieved": round(steps * b_out_full / hsecs / 1e9, 1), "d2h_gbs_measured": pcie_d2h_gbs(local),
                "how": "the same with every batch copied back into pinned host slots (host_output); PCIe D2H bound"}}


def e2e_consumer():
    """tools/bin/libdpe2e.so (tools/e2e_consumer.c, built by __graft_entry__.build()): the token e2e loop in C."""
    import ctypes
    path = os.path.join(ROOT, "tools", "bin", "libdpe2e.so")
    if not os.path.exists(path):
        import __graft_entry__
        __graft_entry__._build_e2e_consumer()
    lib = ctypes.CDLL(path)
    lib.dpe2e_consume_host_batches.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_uint64),
                                               ctypes.POINTER(ctypes.c_int64)]
    return lib


def run_e2e_tokens(dp, cfg, local, args, world=1, dev=None):
    """Token configs end to end: the sequences live in pinned host memory
    (each epoch plan stages the rows it consumes over PCIe) and every batch
    is copied back into pinned host slots, waited on and read by the host.
    The consumer loop is C over the C ABI (tools/e2e_consumer.c: GetNext,
    wait, read, release -- what a C++ / FFI user writes); through ctypes the
    ~10 us Python cost per 128-sequence batch would be the bound.  Host wall
    clock over whole epochs of a 200,000-sequence host dataset."""
    import ctypes
    import numpy as np
    n_host = 200_000
    rng = np.random.default_rng(1)
    lens = rng.integers(1, 1025, n_host).astype(np.int32)
    toks = rng.integers(0, 2 ** 31 - 1, int(lens.sum()), dtype=np.int64).astype(np.int32)
    src = dp.Source.tokens_from_host(lens, toks, device=local, pinned=True)
    g, _ = build_other_graph(dp, cfg, local, 0, 1, src=src)
    C = e2e_consumer()
    ragged = 1 if cfg.get("ragged") else 0

    def consume(it, n):
        rows, chk, done = ctypes.c_int64(0), ctypes.c_uint64(0), ctypes.c_int64(0)
        st = C.dpe2e_consume_host_batches(it.h, n, ragged, ctypes.byref(rows), ctypes.byref(chk),
                                          ctypes.byref(done))
        if st:
            raise RuntimeError(f"e2e consumer: dp_status {st}")
        return rows.value

    # launch group size: the iterator's default (a 16 / 64 / 512 MB sweep measured the same: PCIe bound)
    launch = int(os.environ.get("DP_E2E_TOKEN_LAUNCH_BYTES", 0))
    it = dp.make_iterator(g, seed_override=1, device=local, host_output=True, max_launch_bytes=launch)
    per_epoch = int(re.search(r"elements, (\d+) batches", it.describe()).group(1))
    epochs = 4
    steps = per_epoch * epochs
    consume(it, per_epoch)  # one warm-up epoch on the same iterator (slots allocated, plans built ahead)
    # five timed windows of 4 epochs each on the same iterator; the median is reported
    windows = []
    for _ in range(5):
        if world > 1:
            max_over_ranks(0.0, world, dev)  # barrier: start together
        t0 = time.perf_counter()
        rows = consume(it, steps)
        secs = time.perf_counter() - t0
        if world > 1:
            secs = max_over_ranks(secs * 1e3, world, dev) / 1e3
        windows.append((secs, rows))
    secs, rows = sorted(windows)[len(windows) // 2]
    del it
    # bytes per step, from the same batches (untimed pass)
    it = dp.make_iterator(g, seed_override=1, device=local, host_output=True, max_launch_bytes=launch)
    for _ in range(per_epoch):
        it.get_next().release()
    b_in = b_out = 0
    for _ in range(per_epoch):
        b = it.get_next().wait()
        if cfg.get("ragged"):
            splits = b.numpy(1)
            r, t = splits.size - 1, int(splits[-1])
            b_in += 4 * t + r * (8 + 4 + 8)
            b_out += 4 * t + 8 * (r + 1)
        else:
            ln = b.numpy(1)
            r, lm = b.components[0][1]
            b_in += 4 * int(ln.sum()) + r * (8 + 4 + 8)
            b_out += 4 * r * lm + 4 * r
        b.release()
    del it
    b_in, b_out = b_in * epochs, b_out * epochs
    h2d_meas = pcie_gbs(local, h2d=True)
    return {"value": round(rows * world / secs, 1), "unit": cfg["unit"],
            "h2d_bytes_per_step": int(b_in / steps) * world, "d2h_bytes_per_step": int(b_out / steps) * world,
            "steps": steps, "windows_ms": [round(w[0] * 1e3, 2) for w in windows],
            "pcie": {"h2d_gbs_achieved": round(b_in / secs / 1e9, 1), "d2h_gbs_achieved": round(b_out / secs / 1e9, 1),
                     "h2d_gbs_measured": h2d_meas, "d2h_gbs_measured": pcie_d2h_gbs(local),
                     "h2d_frac": round(b_in / secs / 1e9 / h2d_meas, 3) if h2d_meas else None},
            "host_dataset": f"{n_host} sequences, len U[1,1024], pinned host memory",
            "consumer": "C loop over the C ABI (tools/e2e_consumer.c): dp_iterator_get_next, dp_batch_wait, read "
                        "the batch's first / last token on the host, dp_batch_release",
            "how": "pinned host token source staged over PCIe by each epoch plan + D2H of every batch into pinned "
                   "host slots, each batch waited on and read by the host; host wall clock over 4 epochs after a "
                   "warm-up epoch on the same iterator (median of 5 such windows)",
            "bound": "PCIe: each epoch plan stages exactly the rows it consumes from pinned host memory into HBM "
                     "(dp_k_stage_rows, one pass), the batch kernels stream HBM, every batch is copied back"}


def relaunch(n):
    """`bench.py --gpus N` outside torchrun: re-run this command as N ranks
    (one process per GPU) under torch.distributed.run on this node."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def probe_launch(args):
    """The rank plumbing of `--gpus N` without a GPU (tests/test_multiproc.py):
    every rank joins a gloo group, the max-over-ranks and digest gather run,
    rank 0 prints what it saw."""
    import torch
    import torch.distributed as distr
    rank, world, local = dist_env()
    if world > 1:
        distr.init_process_group("gloo")
    ms = max_over_ranks(1.0 + rank, world, "cpu")
    digests = gather_digests(torch.tensor([rank * 1000 + local], dtype=torch.int64), world)
    expected = [expected_order_digest(args.config, CFG[args.config]["n"], world, r) for r in range(world)]
    if rank == 0:
        print(json.dumps({"probe": True, "n_gpus": world, "gpus_requested": args.gpus, "ms_max": ms,
                          "per_rank": digests, "expected": expected}), flush=True)
    if world > 1:
        distr.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--warmup", type=int, default=32)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CFG), default="cfg2")
    ap.add_argument("--elements-per-gpu", type=int, default=0, help="override the per-GPU dataset size (tests)")
    ap.add_argument("--probe-launch", action="store_true", help=argparse.SUPPRESS)  # CPU test of the launcher
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            ap.error(f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    elif args.gpus > 1 and args.impl == "ours":
        sys.exit(relaunch(args.gpus))
    if args.probe_launch:
        return probe_launch(args)
    cfg = dict(CFG[args.config])
    if args.elements_per_gpu:
        cfg["n"] = args.elements_per_gpu
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
