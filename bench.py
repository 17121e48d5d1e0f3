"""Benchmark: CDMPP predictor training throughput on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (configs[1]): one training epoch over 262,144 synthetic compact ASTs
(327,680 generated, 8:1:1 split — SURVEY §8d C2), desk model
(init_params(desk_config(seed=0)), 354,577 parameters), batch size 64
(the reference's), hybrid loss, Adam, fp32 accumulate.  A bench "step" is one
epoch (≈4,096 optimizer steps).  Synthetic data: `synth.generate`, the
reference's generative model drawn with vectorised numpy (data="synthetic").

Printed JSON line (rank 0):
  value      training samples/s, device time of the timed epochs (CUDA events
             on the training stream, L2 flushed between epochs, max over ranks)
  e2e        the same metric through the public API per epoch: pinned-host
             H2D of the training set → K1 pack → plan upload → epoch →
             validation → D2H of per-step losses + metrics
  roofline   dominant kernel (train_kernel, fused fwd+bwd) from an uncaptured
             profiled epoch: algorithmic FLOPs / device time
  cpu_baseline  the oracle restatement of the reference step (float64 numpy)
             on this host, single thread, bounded sample
  extra      inference ASTs/s on the C1 (4,096) and 1M-AST batches
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_GEN = 327_680
METRIC = "predictor training samples/sec (train epoch, 256K synthetic ASTs)"


def desk_fwd_flops(L):
    """Algorithmic forward FLOPs/AST for the desk config:
    138,240·L + 512·L² + 13,664."""
    L = np.asarray(L, dtype=np.float64)
    return 138_240.0 * L + 512.0 * L * L + 13_664.0


# --------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------- helpers

def dist_setup(n_gpus: int):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


REF_PATH = ROOT / "baseline" / "_ref"        # the unmodified reference (install_ref.sh)
CACHE = ROOT / "bench_cache" / f"ref_synth_{N_GEN}_seed0.npz"


def _import_reference():
    """tpcost from baseline/_ref (falls back to /root/reference in the build
    container); None when neither exists."""
    for p in (REF_PATH, Path("/root/reference/pkg/src")):
        if (p / "tpcost" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import tpcost  # noqa: F401
            return p
    return None


def generate_bench_data(path: Path = CACHE) -> None:
    """The reference's own generator — generate_synthetic(327,680,
    [DEFAULT_SYNTH_DEVICE], SynthOracleConfig(noise_sigma=0.0), seed=0)
     — run once (~60 s) and cached as arrays; the 8:1:1
    split_dataset(seed=0) labels are stored with it."""
    if _import_reference() is None:
        raise RuntimeError("reference package not installed (baseline/install_ref.sh)")
    from tpcost.dataset import (DEFAULT_SYNTH_DEVICE, SynthOracleConfig, generate_synthetic,
                                split_dataset)
    ds = generate_synthetic(N_GEN, [DEFAULT_SYNTH_DEVICE], SynthOracleConfig(noise_sigma=0.0),
                            seed=0)
    sp = split_dataset(ds, seed=0)
    code = {"train": 0, "valid": 1, "test": 2}
    path.parent.mkdir(parents=True, exist_ok=True)
    tmp = path.with_suffix(".tmp.npz")
    np.savez_compressed(
        tmp, vectors=np.concatenate([s.compact.leaf_vectors for s in ds.samples]),
        ordering=np.concatenate([np.asarray(s.compact.ordering, np.int32) for s in ds.samples]),
        n_leaf=np.array([s.compact.n_leaf for s in ds.samples], np.int64),
        latency=np.array([s.latency_s for s in ds.samples]),
        task=np.array([int(s.task_id[1:]) for s in ds.samples], np.int64),
        split=np.array([code[sp.splits[s.id]] for s in ds.samples], np.int8))
    tmp.replace(path)


def make_data():
    """(all, train, valid) as SynthSet arrays of the reference-generated set;
    train / valid in the reference's subset order (ascending sample index)."""
    from paper_2311_09690_b200.synth import SynthSet
    if not CACHE.exists():
        generate_bench_data()
    z = np.load(CACHE)
    data = SynthSet(z["vectors"], z["ordering"], z["n_leaf"], z["latency"], z["task"])
    split = z["split"]
    return data, data.take(np.flatnonzero(split == 0)), data.take(np.flatnonzero(split == 1))


def bench_config(world: int, dp_mode: str, batch: int, n_steps: int) -> dict:
    """The `config` both arms print (same workload, same keys)."""
    gb = batch * world if dp_mode == "weak" else batch
    return {"workload": "train epoch, 262,144 synthetic ASTs (configs[1]): "
                        "generate_synthetic(327680, seed=0) + split_dataset(seed=0) train split",
            "model": "desk_config (354,577 params), init_params seed 0",
            "global_batch": gb, "seq_len": "1..6 leaves",
            "parallelism": (f"dp{world} ({dp_mode} scaling)" if world > 1 else "single GPU"),
            "optimizer_steps_per_epoch": int(n_steps),
            "loss": "hybrid (lambda 1e-3, transformed space), Adam lr 1e-3",
            "l2": "flushed (256 MiB write) between timed epochs"}


def rag_of(s, device_feat):
    from paper_2311_09690_b200 import engine
    dev = np.tile(device_feat.astype(np.float32), (s.n, 1))
    return engine.RaggedHost(rows=s.vectors.astype(np.float32), ordering=s.ordering,
                             n_leaf=s.n_leaf, devfeat=dev, encoded=False)


# --------------------------------------------------------------- CPU baseline

class RefTrainer:
    """The reference's own training loop body on this host: tpcost from
    baseline/_ref, costmodel.train's setup (encode_dataset once, fit_boxcox,
    init_params(desk_config(seed=0)), nn.Adam, the seeded _epoch_batches
    plan) and per step exactly `backward` + `opt.step` (costmodel.py:697-706).
    `run(budget_s)` advances through the epoch plan for a bounded sample."""

    def __init__(self, train, batch: int = 64):
        if _import_reference() is None:
            raise RuntimeError("reference package not installed (baseline/install_ref.sh)")
        from tpcost import costmodel as cm
        from tpcost.dataset import DEFAULT_SYNTH_DEVICE, Sample, fit_boxcox
        from tpcost.features import CompactAst
        self.cm = cm
        self.config = cm.desk_config(seed=0, batch_size=batch)
        off = train.offsets()
        samples = [Sample(id=f"s{i}", task_id="t0", model_id="m0",
                          device_id=DEFAULT_SYNTH_DEVICE.name,
                          compact=CompactAst(leaf_vectors=train.vectors[off[i]:off[i + 1]],
                                             ordering=tuple(train.ordering[off[i]:off[i + 1]].tolist()),
                                             serialized=(), n_leaf=int(train.n_leaf[i])),
                          latency_s=float(train.latency[i])) for i in range(train.n)]
        t0 = time.perf_counter()
        self.inputs = cm.encode_dataset(samples, {DEFAULT_SYNTH_DEVICE.name: DEFAULT_SYNTH_DEVICE})
        self.encode_s = time.perf_counter() - t0
        self.norm = fit_boxcox([s.latency_s for s in samples])
        self.targets = self.norm.encode(np.array([s.latency_s for s in samples]))
        self.params = cm.init_params(self.config)
        self.opt = cm._make_optimizer(self.config, self.params.tensors.keys())
        self.spec = cm.LossSpec(mode=self.config.loss_mode,
                                lambda_hybrid=self.config.lambda_hybrid,
                                offset=self.norm.loss_offset, mape_space=self.config.mape_space,
                                normalizer=self.norm)
        self.rng = np.random.default_rng(self.config.seed)
        self.n_leaves = [e.n_leaf for e in self.inputs]
        self.batches = cm._epoch_batches(self.rng, self.n_leaves, self.config.batch_size)
        self.pos = 0
        self.lr = cm._lr_at(self.config, 0)

    def run(self, budget_s: float, threads: int, min_steps: int = 4):
        from threadpoolctl import threadpool_limits
        cm = self.cm
        done = steps = 0
        with threadpool_limits(limits=threads):
            t0 = time.perf_counter()
            while True:
                if self.pos == len(self.batches):  # next epoch of the same run
                    self.batches = cm._epoch_batches(self.rng, self.n_leaves,
                                                     self.config.batch_size)
                    self.pos = 0
                idx = self.batches[self.pos]
                self.pos += 1
                batch = [self.inputs[i] for i in idx]
                value, grads, _ = cm.backward(self.params, batch, self.targets[idx], self.spec)
                self.opt.step(self.params.tensors, grads, self.lr)
                done += len(idx)
                steps += 1
                el = time.perf_counter() - t0
                if el >= budget_s and steps >= min_steps:
                    return done, steps, el


def _host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def cpu_baseline(train, budget_s: float = 12.0, threads: int = 1, ref: RefTrainer | None = None):
    """Bounded sample of the reference's training loop (tpcost itself) on
    this host's cores."""
    ref = ref or RefTrainer(train)
    done, steps, el = ref.run(budget_s, threads)
    return {"value": done / el, "unit": "samples/s", "cores": threads, "kind": "reference",
            "sample": f"{steps} steps of tpcost.costmodel.train's loop body (backward + "
                      f"nn.Adam.step, bs {ref.config.batch_size}, {done} samples, {el:.1f} s) "
                      f"over the same epoch plan; encode_dataset done once "
                      f"({ref.encode_s:.1f} s, outside the sample); {threads} BLAS thread(s)"}


def _ref_infer_worker(args):
    """one reference process: predict_batch over its contiguous shard"""
    vec, ordering, n_leaf, reps = args
    _import_reference()
    from tpcost import costmodel as cm
    from tpcost.dataset import DEFAULT_SYNTH_DEVICE
    from tpcost.features import CompactAst, encode_input
    off = np.concatenate([[0], np.cumsum(n_leaf)])
    inputs = [encode_input(CompactAst(vec[off[i]:off[i + 1]],
                                      tuple(ordering[off[i]:off[i + 1]].tolist()), (),
                                      int(n_leaf[i])), DEFAULT_SYNTH_DEVICE)
              for i in range(len(n_leaf))]
    params = cm.init_params(cm.desk_config(seed=0))
    cm.forward(params, inputs[:8])
    t0 = time.perf_counter()
    for _ in range(reps):
        cm.forward(params, inputs)
    return time.perf_counter() - t0


def cpu_inference_baseline(data, n: int = 4096):
    """C1 on the reference: costmodel.forward over the
    first 4,096 ASTs of the set (= generate_synthetic(4096, seed=0)), single
    process, and one process per host core on contiguous shards (summed)."""
    from multiprocessing import get_context
    sub = data.take(np.arange(n))
    off = sub.offsets()
    one = _ref_infer_worker((sub.vectors, sub.ordering, sub.n_leaf, 2))
    cores = max(1, _host_threads())
    shards = np.array_split(np.arange(n), cores)
    jobs = [(sub.vectors[off[c[0]]:off[c[-1] + 1]], sub.ordering[off[c[0]]:off[c[-1] + 1]],
             sub.n_leaf[c], 2) for c in shards if len(c)]
    with get_context("spawn").Pool(len(jobs)) as pool:
        t0 = time.perf_counter()
        times = pool.map(_ref_infer_worker, jobs)
        wall = time.perf_counter() - t0
    return {"single_process_asts_per_s": 2 * n / one,
            "all_cores_asts_per_s": 2 * n / max(times), "cores": cores,
            "all_cores_wall_s_incl_import": wall, "kind": "reference",
            "sample": f"tpcost.costmodel.forward over {n} ASTs x 2 (init_params(desk seed 0)); "
                      f"all cores: {len(jobs)} processes on contiguous shards, slowest shard's "
                      f"forward time"}


def run_reference_arm(args):
    """--impl reference: the unmodified reference (tpcost from baseline/_ref)
    on the host cores, on the repo arm's workload / metric / config; each
    step a bounded sample of the epoch (its loop body is serial: every step
    depends on the previous Adam update).  Falls back to the oracle port when
    baseline/_ref is absent."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    data, train, valid = make_data()
    ref = RefTrainer(train, args.batch_size)
    # all the host threads it can use: the steps are serial, so the only
    # parallelism is numpy's BLAS pool — probe 1 thread vs every core in the
    # warm-up and keep the faster
    n_cpu = _host_threads()
    cand = {1: 0.0}
    if n_cpu and n_cpu > 1:
        cand[int(n_cpu)] = 0.0
    for _ in range(max(args.warmup, 1)):
        for th in cand:
            d, _, el = ref.run(1.0, th)
            cand[th] = max(cand[th], d / el)
    threads = max(cand, key=cand.get)
    done = steps = 0
    el_sum = 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        d, st, el = ref.run(5.0, threads)
        done, steps, el_sum = done + d, steps + st, el_sum + el
    elapsed = time.perf_counter() - t0
    v = done / el_sum
    n_plan = len(ref.batches)
    cfg = bench_config(world, args.dp_mode, args.batch_size, n_plan)
    line = {"metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed * 1e3 / max(args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads,
                             "kind": "reference",
                             "sample": f"{steps} steps of tpcost's train loop body (backward + "
                                       f"nn.Adam.step, bs {args.batch_size}, {done} samples in "
                                       f"{args.steps} samples of 5 s) over the epoch plan; "
                                       f"encode_dataset once ({ref.encode_s:.1f} s, untimed); "
                                       f"{threads} BLAS thread(s)"},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "threads_probe_samples_per_s": {str(k): val for k, val in cand.items()}}
    print(json.dumps(line))


# ----------------------------------------------------------------- our arm

def run_full_config(args, data, norm, dv, dev, world, comm, n_steps: int = 12):
    import torch
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import engine
    from paper_2311_09690_b200.large_training import LargeTrainer
    from paper_2311_09690_b200.training import plan_epoch
    cfg = pb.full_reference_config()
    sub = data.take(np.arange(65536))
    loss = engine.loss_struct("hybrid", cfg.lambda_hybrid, norm.loss_offset)
    params = pb.init_params(cfg)
    tr = LargeTrainer(cfg, params.tensors, rag_of(sub, dv), norm.encode(sub.latency), loss,
                      device=dev, comm=comm)
    flat, steps = plan_epoch(np.random.default_rng(0), tr.n_leaf, cfg.batch_size, world,
                             tr.rank)
    full_steps = steps[steps[:, 3] == cfg.batch_size * world]  # full global batches
    tr.run_epoch(cfg.lr, flat, full_steps[:3])
    torch.cuda.synchronize()
    barrier(world)
    sel = full_steps[3:3 + n_steps]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tr.run_epoch(cfg.lr, flat, sel)
    b.record()
    torch.cuda.synchronize()
    t = max_over_ranks(a.elapsed_time(b) / 1e3, world)
    samples = int(sel[:, 3].sum())  # global samples
    losses = tr.losses[:len(sel)].cpu().numpy()
    out = {"model": "full_reference_config (d 716, 11 layers, 4 heads, d_ff 985, 46.7 M params)",
           "train_samples_per_s": samples / t, "train_ms_per_step": t / len(sel) * 1e3,
           "train_global_batch": cfg.batch_size * world, "train_steps_timed": len(sel),
           "train_model_tflops": samples * 3 * 281.0e6 / t / 1e12,
           "train_loss_first_last": [float(losses[0]), float(losses[-1])],
           "paper_v100_train_samples_per_s": 14241,
           "dtype": "3xTF32 tcgen05 GEMMs (fp32-class), fp32 params / Adam"}
    del tr
    p = pb.Predictor(params)
    n = 4096
    s2 = data.take((np.arange(n) + (world > 1) * 0) % data.n)
    rows, ordering, leaf_off, devfeat = engine.upload_ragged(rag_of(s2, dv), dev)
    f = lambda: p.forward_device(rows, ordering, leaf_off, devfeat, n, False, norm,  # noqa
                                 latents=False, n_leaf=s2.n_leaf)
    for _ in range(2):
        f()
    barrier(world)
    a.record()
    for _ in range(5):
        f()
    b.record()
    torch.cuda.synchronize()
    t = max_over_ranks(a.elapsed_time(b) / 1e3, world)
    out["infer_asts_per_s"] = n * world * 5 / t
    out["infer_batch_per_rank"] = n
    return out


def run_large_batch(cfg, train, targets, norm, dv, dev, flush_l2, batch: int = 600):
    """Desk config at global batch 600, one epoch (device time, L2 flushed
    before it): fused FFMA trainer vs the layer-by-layer tcgen05 path."""
    import torch
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import engine
    from paper_2311_09690_b200.large_training import LargeTrainer
    from paper_2311_09690_b200.training import Trainer
    cfg6 = pb.desk_config(seed=0, batch_size=batch)
    params = pb.init_params(cfg6)
    loss = engine.loss_struct("hybrid", cfg6.lambda_hybrid, norm.loss_offset, 0.0, 5,
                              "transformed", norm)
    out = {"global_batch": batch,
           "semantics": "the reference's train loop at batch_size 600 (per-bucket batches of "
                        "<= 600, ~437 optimizer steps per epoch): a different optimisation "
                        "trajectory from bs 64, same per-sample work",
           "variants": "fused_ffma: train4 + slot reduce + Adam; fused_ffma_wgrad_tcgen05: "
                       "the encoder weight gradients as tcgen05 3xTF32 GEMMs over the "
                       "step's token rows (wgrad.cu); tcgen05_3xtf32_layerwise: large.cu"}
    for name, mk in (("fused_ffma", lambda: Trainer(cfg6, params.tensors, rag_of(train, dv),
                                                    targets, loss, device=dev)),
                     ("fused_ffma_wgrad_tcgen05",
                      lambda: Trainer(cfg6, params.tensors, rag_of(train, dv), targets, loss,
                                      device=dev, wgrad_tc=True)),
                     ("tcgen05_3xtf32_layerwise",
                      lambda: LargeTrainer(cfg6, params.tensors, rag_of(train, dv), targets,
                                           loss, device=dev))):
        tr = mk()
        rng = np.random.default_rng(0)
        flat, steps = tr.plan(rng)
        with torch.cuda.stream(tr.stream):
            tr.run_epoch(cfg6.lr, flat, steps[:8])   # warm-up (+ graph capture)
        torch.cuda.synchronize()
        flat, steps = tr.plan(rng)
        flush_l2()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(tr.stream):
            a.record()
            tr.run_epoch(cfg6.lr, flat, steps)
            b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 1e3
        out[name] = {"samples_per_s": train.n / t, "ms_per_step": t * 1e3 / len(steps),
                     "optimizer_steps": int(len(steps))}
        del tr
    # the A/B at the headline batch (64): the same fused trainer with the
    # encoder weight gradients on tcgen05 (the bs-64 fused number is `value`)
    cfg64 = pb.desk_config(seed=0, batch_size=64)
    tr = Trainer(cfg64, params.tensors, rag_of(train, dv), targets, loss, device=dev,
                 wgrad_tc=True)
    rng = np.random.default_rng(0)
    flat, steps = tr.plan(rng)
    with torch.cuda.stream(tr.stream):
        tr.run_epoch(cfg64.lr, flat, steps[:8])
    torch.cuda.synchronize()
    flat, steps = tr.plan(rng)
    flush_l2()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(tr.stream):
        a.record()
        tr.run_epoch(cfg64.lr, flat, steps)
        b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 1e3
    out["bs64_fused_ffma_wgrad_tcgen05"] = {"samples_per_s": train.n / t,
                                            "ms_per_step": t * 1e3 / len(steps),
                                            "optimizer_steps": int(len(steps))}
    del tr
    return out


def _ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/r02/ncu_traffic.json)."""
    p = ROOT / "profiles" / "r02" / "ncu_traffic.json"
    try:
        return int(json.loads(p.read_text())[kernel]["dram_bytes_per_launch"])
    except Exception:
        return None


def run_ours(args):
    import torch
    import paper_2311_09690_b200 as pb
    from paper_2311_09690_b200 import _lib, engine
    from paper_2311_09690_b200.dataset import fit_boxcox
    from paper_2311_09690_b200.training import Trainer, epoch_batches

    world, rank, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    lib = _lib.load()
    cfg = pb.desk_config(seed=0, batch_size=args.batch_size)
    data, train, valid = make_data()
    norm = fit_boxcox(train.latency)
    targets = norm.encode(train.latency)
    dspec = pb.DeviceSpec("synth0", 1000.0, 16.0, 1024.0, 16, 2048.0, 4.0)
    dv = pb.device_vector(dspec)
    # data parallel (N > 1): --dp-mode weak (default: bs 64 per rank, global
    # batch 64·N) or strong (each reference batch of 64 split across the
    # ranks, the reference's step count); gradients reduced in rank order
    # over NCCL inside the captured epoch; each rank holds the whole training
    # set and takes its share of every global batch from the common plan
    comm = engine.Comm(rank, world) if world > 1 else None
    params = pb.init_params(cfg)
    loss = engine.loss_struct("hybrid", cfg.lambda_hybrid, norm.loss_offset, 0.0, 5,
                              "transformed", norm)
    tr = Trainer(cfg, params.tensors, rag_of(train, dv), targets, loss, rag_of(valid, dv),
                 valid.latency, norm, device=dev, comm=comm, overlap=bool(args.overlap),
                 dp_mode=args.dp_mode)
    rng = np.random.default_rng(cfg.seed)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def flush_l2():
        with torch.cuda.stream(tr.stream):
            _lib.check(lib.tpcb_flush_l2(flush.data_ptr(), flush.numel(), engine.stream_ptr()),
                       "flush")

    # warm-up epochs (first one captures the epoch graph)
    for w in range(max(args.warmup, 1)):
        flat, steps = tr.plan(rng)
        n = tr.run_epoch(cfg.lr, flat, steps)
        tr.evaluate_async()
        tr.collect(n, w)
    plans = [tr.plan(rng) for _ in range(args.steps)]
    n_steps = plans[0][1].shape[0]
    # timed: K epochs, device time per epoch, L2 flushed in between
    barrier(world)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for k, (flat, steps) in enumerate(plans):
            flush_l2()
            with torch.cuda.stream(tr.stream):
                ev[k][0].record()
            tr.run_epoch(cfg.lr, flat, steps)
            with torch.cuda.stream(tr.stream):
                ev[k][1].record()
        tr.stream.synchronize()
    barrier(world)
    ms = sum(a.elapsed_time(b) for a, b in ev)
    ms = max_over_ranks(ms, world)
    tr.collect(n_steps, 0)
    samples = train.n * args.steps  # the epoch is shared by all ranks
    value = samples / (ms / 1e3)

    # ------------------------------------------------ e2e through the public API
    # per epoch: pinned-host H2D of the training set + K1 pack, plan upload,
    # epoch, validation, D2H of losses and metrics
    pinned = {
        "rows": torch.from_numpy(train.vectors.astype(np.float32)).pin_memory(),
        "ordering": torch.from_numpy(train.ordering.astype(np.int32)).pin_memory(),
        "leaf_off": torch.from_numpy(train.offsets()).pin_memory(),
        "y": torch.from_numpy(np.asarray(targets, dtype=np.float64)).pin_memory(),
    }
    h2d = sum(t.numel() * t.element_size() for t in pinned.values())
    e2e_k = max(3, min(args.steps, 5))
    e2e_times = []
    for k in range(e2e_k):
        barrier(world)
        t0 = time.perf_counter()
        with torch.cuda.stream(tr.stream):
            rows_d = pinned["rows"].to(dev, non_blocking=True)
            ord_d = pinned["ordering"].to(dev, non_blocking=True)
            off_d = pinned["leaf_off"].to(dev, non_blocking=True)
            tr.src.y.copy_(pinned["y"], non_blocking=True)
            engine.pack(rows_d, ord_d, off_d, train.n, cfg.n_leaf_max, False, tr.status,
                        out=tr.src.pk)
        flat, steps = plans[k % len(plans)]
        n = tr.run_epoch(cfg.lr, flat, steps)
        tr.evaluate_async()
        losses, _, met = tr.collect(n, k)
        barrier(world)
        e2e_times.append(max_over_ranks(time.perf_counter() - t0, world))
    e2e_s = statistics.median(e2e_times)
    d2h = n_steps * 8 + 3 * 8 + 4
    plan_bytes = plans[0][0].nbytes + plans[0][1].nbytes
    e2e = {"value": train.n / e2e_s, "unit": "samples/s",
           "h2d_bytes_per_step": int(h2d + plan_bytes), "d2h_bytes_per_step": int(d2h),
           "steps": e2e_k, "statistic": "median over the epochs (wall clock, max over ranks)",
           "epoch_s": [round(t, 4) for t in e2e_times],
           "includes": "H2D of training set + K1 + epoch + validation"}

    # --------------------------------------- roofline of the dominant kernel
    prof = np.zeros(3)
    flat, steps = plans[0]
    tr.run_epoch(cfg.lr, flat, steps, profile=prof)
    tr.collect(n_steps, 0)
    launches = n_steps
    # this rank's share of the epoch's algorithmic FLOPs
    flops_epoch = 3.0 * float(desk_fwd_flops(train.n_leaf).sum()) / world
    avg_ms = prof[0] / launches
    achieved = flops_epoch / launches / (avg_ms / 1e3) / 1e12
    import ctypes as C
    scratch = torch.empty(4096, dtype=torch.float32, device=dev)
    tf = C.c_double()
    _lib.check(lib.tpcb_probe_ffma(scratch.data_ptr(), C.byref(tf), engine.stream_ptr()), "probe")
    ffma = tf.value
    peaks = {}
    pk_path = ROOT / "MEASURED_PEAKS.json"
    if pk_path.exists():
        peaks = json.loads(pk_path.read_text())
    bf16 = peaks.get("bf16_tflops", 1590.0)
    roofline = {"bound": "tensor", "kernel": "train4_kernel (fused fwd+bwd per sample, desk fast path)",
                "achieved": achieved, "peak": bf16, "unit": "TFLOP/s",
                "frac": achieved / bf16, "traffic": _ncu_traffic("train4_kernel"),
                "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if peaks else
                               "fallback 1.59 PFLOP/s",
                "fp32_ffma_peak_measured": ffma, "frac_of_fp32_ffma": achieved / ffma,
                "share_of_step": prof[0] / prof.sum(),
                "per_launch": {"flops": flops_epoch / launches, "avg_ms": avg_ms},
                "other_kernels_ms_per_epoch": {"reduce_adam": prof[1], "allreduce_opt_dp": prof[2]}}

    # ----------------------------------------------- inference (extra keys)
    # batch inference sharded with no communication: every rank runs the
    # forward over its own contiguous shard of n ASTs of the global batch
    # (n · world); throughput = global batch / max-over-ranks device time.
    # e2e: the public bulk API (Predictor.forward_batch: host CompactBatch in
    # — arrays in pinned host memory — decoded latencies out), wall clock.
    infer = {"model": "the desk model after the timed training epochs (decodes inside the "
                      "Box-Cox domain)"}
    trained = pb.CostModelParams(cfg, tr.tensors())
    for prec in ("fp32", "bf16"):
        p = pb.Predictor(trained, precision=prec)
        tag = "" if prec == "fp32" else "bf16_"
        for n in (4096, 1 << 20):
            sub = data.take((np.arange(n) + rank * n) % data.n)
            rows, ordering, leaf_off, devfeat = engine.upload_ragged(rag_of(sub, dv), dev)
            for _ in range(3):
                p.forward_device(rows, ordering, leaf_off, devfeat, n, False, norm, latents=False)
            barrier(world)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20 if n <= 4096 else 5
            a.record()
            for _ in range(reps):
                p.forward_device(rows, ordering, leaf_off, devfeat, n, False, norm, latents=False)
            b.record()
            torch.cuda.synchronize()
            t_inf = max_over_ranks(a.elapsed_time(b) / 1e3, world)
            infer[f"infer_{tag}asts_per_s_{n * world}"] = n * world * reps / t_inf
            # e2e through the public API from pinned host arrays
            pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa
            batch = pb.CompactBatch(pin(sub.vectors.astype(np.float32)),
                                    pin(sub.ordering.astype(np.int32)), pin(sub.n_leaf),
                                    np.zeros(n, np.int32), [dspec])
            p.forward_batch(batch, norm)
            calls = []
            for _ in range(max(reps, 7)):
                barrier(world)
                t0 = time.perf_counter()
                _, _, _, _, lat_h = p.forward_batch(batch, norm)
                calls.append(max_over_ranks(time.perf_counter() - t0, world))
            t_e2e = statistics.median(calls)  # per call (host jitter: median)
            infer[f"infer_{tag}e2e_asts_per_s_{n * world}"] = n * world / t_e2e
            infer[f"infer_e2e_h2d_bytes_{n}"] = int(batch.vectors.nbytes + batch.ordering.nbytes
                                                    + 8 * (n + 1) + 4 * 6 * n)
            infer[f"infer_e2e_d2h_bytes_{n}"] = int(8 * n + 4 * n)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        infer["cpu_reference_c1"] = cpu_inference_baseline(data)

    # ------------------------------------------ large-batch desk variant
    # the same epoch at global batch 600 (the paper's batch;
    # the reference's semantics at that batch size, ~437 optimizer steps):
    # the fused FFMA trainer (one CTA per sample) and the layer-by-layer
    # tcgen05 3xTF32 path (large.cu), device time of one epoch each
    large_batch = None
    if world == 1 and not args.no_large_batch:
        large_batch = run_large_batch(cfg, train, targets, norm, dv, dev, flush_l2)

    # ------------------------- full_reference_config (extra keys)
    # d 716 × 11 layers, 46.7 M params: the layer-by-layer tcgen05 path
    # (3xTF32 GEMMs).  Training: bs 600 per rank (weak scaling, gradient
    # all-reduced over NCCL), forward + loss + backward + Adam + weight-image
    # rebuild per step, device time max over ranks; inference: 4,096 ASTs per
    # rank.  The paper's V100 training figure for this config: 14,241
    # samples/s.
    full = None
    if not args.no_full:
        full = run_full_config(args, data, norm, dv, dev, world, comm)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(train)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True,
                "scaling": "weak" if (world == 1 or args.dp_mode == "weak") else "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": bench_config(world, args.dp_mode, args.batch_size, n_steps),
                "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu,
                "gpu_launches": int(args.steps * n_steps * (2 if world == 1 else 4)),
                "clocks": clk.summary(), "extra": infer, "large_batch": large_batch,
                "full_reference_config": full,
                "final_val_mape": float(met[0]), "final_train_loss": float(np.mean(losses))}
        print(json.dumps(line))
    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch-size", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full", action="store_true",
                    help="skip the full_reference_config training/inference block")
    ap.add_argument("--dp-mode", choices=["weak", "strong"], default="weak",
                    help="data parallel (N > 1): weak = bs per rank, strong = the reference "
                         "batch split across ranks")
    ap.add_argument("--no-large-batch", action="store_true",
                    help="skip the desk large-batch (600) variant")
    ap.add_argument("--overlap", type=int, default=1,
                    help="1: reduce + Adam of each step overlapped with its backward (default); "
                         "0: sequential reduce kernel (A/B)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
