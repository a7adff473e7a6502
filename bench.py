#!/usr/bin/env python
"""FPS-SFT throughput on B200: transforms/s over a batch of independent
instances (BASELINE.json config 2 by default: 4096 x 256x256 complex64,
K=100, noiseless, profile P32).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2]
    python bench.py --impl reference ...      # the CPU reference arm

One step = one ``fpssft_run_batch`` (one fused kernel launch) over the
rank's batch, cubes resident in HBM.  L2 is flushed (256 MiB write) before
every timed step and only the step is inside the CUDA events.  Multi-GPU
(torchrun): every rank owns its own slice of the instance stream (weak
scaling, no data-path collective); time = max over ranks.

The JSON line adds ``roofline`` (algorithmic gather bytes per launch over
the launch time vs the measured HBM copy peak), ``cpu_baseline`` (the CPU
oracle port on this host's cores over a bounded sample of the same
inputs), ``e2e`` (through the public API from pinned host buffers, copies
included) and ``clocks`` (nvidia-smi sampled during the run).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FPS-SFT transforms/sec"
UNIT = "transforms/s"
# recovered-set capacity per config (power of two >= K plus false positives);
# an overflow seen in the untimed warm-up doubles it (reported in config)
K_CAP = {1: 64, 2: 128, 3: 512, 4: 2048, 5: 1024}
FLUSH_BYTES = 256 << 20


def _cfg(w, seed):
    import paper_1711_11407_b200 as P

    return P.FpsSftConfig(seed=seed, **P.PROFILES[w.profile])


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _probe_rate():
    """Random 64-byte-segment fetch rate of this GPU measured by
    tools/gather_probe.cu (variant 2: 8-byte loads with the .L2::64B fetch
    size, 2^28-element array, all SMs)."""
    import re

    try:
        for line in open(os.path.join(ROOT, "profiles", "r01_gather_probe.txt")):
            m = re.search(r"2\^28 x8B\s+ctas\s+1184\s+variant 2:.*?([0-9.]+) Gsamples/s", line)
            if m:
                return float(m.group(1)) * 1e9
    except OSError:
        pass
    return None


def _segments_per_launch(shape, schedule, iterations, sched_index=None, seg=8, group=1):
    """Distinct 64-byte DRAM segments (seg = 8 complex64 samples) the gathers
    of one launch touch: per iteration, the (D+1) L sample offsets of the
    lines (row-major cube), counted once per instance that runs it.  With the
    .L2::64B fetch size a miss moves one such segment (config 2: 6.7 M
    segments, 427 MB of DRAM reads under ncu).  Interleaved layout (group G):
    a group's G samples of an offset share segments, counted once per group
    for as many iterations as its longest-running instance."""
    if group > 1:
        iters = np.asarray(iterations)
        pad = (-len(iters)) % group
        gi = np.concatenate([iters, np.zeros(pad, iters.dtype)]).reshape(-1, group).max(1)
        si = None
        if sched_index is not None:  # one schedule per group is what the model assumes
            si = np.asarray(sched_index)[::group]
        return _segments_per_launch(shape, schedule, gi, si, seg, -group)
    G = -group if group < 0 else 1
    dims = np.asarray(shape.dims, np.int64)
    strides = np.cumprod(np.concatenate([[1], dims[::-1][:-1]]))[::-1]
    L = shape.line_len
    l = np.arange(L, dtype=np.int64)[:, None]
    iters = np.asarray(iterations)
    sidx = np.zeros(len(iters), np.int64) if sched_index is None else np.asarray(sched_index)
    total = 0
    for s in np.unique(sidx):
        its = iters[sidx == s]
        per_t = []
        for t in range(int(its.max())):
            al, ta = schedule[s, t, 0].astype(np.int64), schedule[s, t, 1].astype(np.int64)
            offs = []
            for i in range(shape.ndim + 1):
                tau = ta.copy()
                if i:
                    tau[i - 1] = (tau[i - 1] + 1) % dims[i - 1]
                offs.append((((l * al + tau) % dims) * strides).sum(1))
            o = np.concatenate(offs)
            if G > 1:  # element index in the group block: offset * G + member
                o = (o[:, None] * G + np.arange(G)[None, :]).ravel()
            per_t.append(len(np.unique(o // seg)))
        per_t = np.asarray(per_t)
        total += int(sum(per_t[:n].sum() for n in its))
    return total


def _traffic(workload_name, batch=None):
    """DRAM bytes per launch from the committed ncu capture, if any (a capture
    of a subset, "<cfgN>_recover_subset<n>", scaled to ``batch`` instances)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
    except Exception:
        return None
    if workload_name in d:
        return d[workload_name]
    pre = workload_name.split("_")[0] + "_recover_subset"
    for k, v in d.items():
        if k.startswith(pre) and batch:
            return int(v * batch / int(k[len(pre):]))
    return None


# ---------------------------------------------------------------- CPU arm
_SAMPLE = None  # (cubes, dims, profile kwargs, seed) inherited by forked workers


def _oracle_chunk(idx):
    from oracle import fps_oracle as O

    cubes, dims, prof, seed, synth = _SAMPLE
    p = O.Profile(**prof)
    t0 = time.perf_counter()
    its = 0
    for i in idx:
        rep = O.recover(cubes[i], dims, p, seed=seed)
        its += rep.iterations_run
        if synth:  # config 5 also re-synthesises the image (numpy ifftn of the spectrum)
            O.synthesize(dims, rep.freqs, rep.amps)
    return time.perf_counter() - t0, its


def cpu_oracle_throughput(cubes: np.ndarray, dims, prof: dict, seed: int, workers: int,
                          synth: bool = False):
    """instances/s of the CPU oracle port over ``cubes`` on ``workers``
    processes (the reference's own ProcessPoolExecutor parallelism,
    oracle.py:275-277): instances / max worker busy time."""
    import multiprocessing as mp

    global _SAMPLE
    _SAMPLE = (cubes, tuple(dims), prof, seed, synth)
    n = len(cubes)
    parts = [list(range(i, n, workers)) for i in range(workers)]
    parts = [p for p in parts if p]
    t0 = time.perf_counter()
    if len(parts) == 1:
        res = [_oracle_chunk(parts[0])]
    else:
        with mp.get_context("fork").Pool(len(parts)) as pool:
            res = pool.map(_oracle_chunk, parts)
    wall = time.perf_counter() - t0
    busy = max(r[0] for r in res)
    return n / busy, wall, sum(r[1] for r in res) / n


def _host_sample(w, count, start=0):
    from paper_1711_11407_b200 import workloads as W

    return np.stack([W.make_instance(w, r)[2] for r in W.instance_rngs(w.seed, count, start)])


def _estimate_oracle_seconds(cubes, dims, prof, seed):
    from oracle import fps_oracle as O

    t0 = time.perf_counter()
    for c in cubes[:2]:
        O.recover(c, dims, O.Profile(**prof), seed=seed)
    return (time.perf_counter() - t0) / min(2, len(cubes))


def run_reference(args, w):
    import paper_1711_11407_b200 as P

    cores = os.cpu_count() or 1
    prof = P.PROFILES[w.profile]
    probe = _host_sample(w, 2)
    per = _estimate_oracle_seconds(probe, w.dims, prof, args.config)
    # each step: a bounded sample sized for ~args.ref_step_seconds of wall time
    count = int(max(cores, min(w.batch, args.ref_step_seconds * cores / max(per, 1e-4))))
    cubes = _host_sample(w, count)
    for _ in range(args.warmup_ref):
        cpu_oracle_throughput(cubes[:cores], w.dims, prof, args.config, cores)
    times, its = [], []
    for _ in range(args.steps):
        rate, wall, mean_it = cpu_oracle_throughput(cubes, w.dims, prof, args.config, cores,
                                                    synth=args.config == 5)
        times.append(count / rate)
        its.append(mean_it)
    total = sum(times)
    value = count * args.steps / total
    sample = (f"{count} of the {w.batch} instances of {w.name} (instances 0..{count - 1}), "
              f"numpy float64 oracle port, {cores} worker processes"
              + (", recovery + numpy re-synthesis" if args.config == 5 else ""))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; BASELINE.json names no dataset)",
        "config": {"workload": w.name, "batch_per_step": count, "profile": w.profile,
                   "mean_iterations": float(np.mean(its))},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait(timeout=10)
        rows = []
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 8:
                    rows.append(f)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [r for r in rows if r[2].isdigit() and int(r[2]) > 0] or rows
        sm = [int(r[0]) for r in loaded if r[0].isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in loaded for n, v in zip(names, r[4:8]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": int(rows[0][1]) if rows[0][1].isdigit() else None,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--layout", default="auto", choices=["auto", "batch_major", "interleaved"],
                    help="HBM layout of the batch: [B, *dims], or [B/G, *dims, G] with G "
                         "instances interleaved sample by sample (--group); auto = "
                         "interleaved for batches of >= 64 instances")
    ap.add_argument("--group", type=int, default=8)
    ap.add_argument("--mode", default="auto", choices=["auto", "warp", "cta"],
                    help="kernel family (auto: the planner's choice for this batch)")
    ap.add_argument("--batch", type=int, default=None, help="override instances per rank")
    ap.add_argument("--k-cap", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU-seconds budget of the cpu_baseline sample")
    ap.add_argument("--ref-step-seconds", type=float, default=4.0)
    ap.add_argument("--warmup-ref", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-synth", action="store_true", help="config 5 without re-synthesis")
    ap.add_argument("--l2-fetch", type=int, default=32,
                    help="cudaLimitMaxL2FetchGranularity in bytes (0 = leave the driver default)")
    ap.add_argument("--load-seconds", type=float, default=1.0,
                    help="back-to-back steps before the timed region (clock ramp/sampling)")
    args = ap.parse_args()

    from paper_1711_11407_b200 import workloads as W

    w = W.CONFIGS[args.config]
    if args.batch:
        w = W.Workload(w.name, w.dims, args.batch, w.k, w.placement, w.magnitude, w.noise_var,
                       w.profile, w.seed)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, w)
        return

    import torch

    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import ops
    from paper_1711_11407_b200.shard import instance_range

    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    l2_default = P._native.get_l2_fetch_granularity(dev)
    if args.l2_fetch:
        P._native.set_l2_fetch_granularity(args.l2_fetch, dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    B = w.batch
    b0, b1 = instance_range(rank, world, per_rank=B)
    shape = P.CubeShape(w.dims)
    cfg = _cfg(w, args.config)
    k_cap = args.k_cap or K_CAP[args.config]

    # ---- inputs: spectra on the host, cubes synthesised on the device
    spectra = W.make_spectra(w, B, b0)
    cubes = W.synthesize_batch_torch(w.dims, spectra, dev, w.noise_var,
                                     noise_seed=w.seed * 1000003 + b0)
    torch.cuda.synchronize()
    layout = args.layout
    if layout == "auto":
        layout = "interleaved" if B >= 64 else "batch_major"
    group = args.group if layout == "interleaved" else 1
    run_cubes = P.interleave(cubes, group) if group > 1 else cubes
    torch.cuda.synchronize()
    runner = P.BatchRunner(shape, cfg, B, k_cap=k_cap, precision=args.precision, device=dev,
                           mode=args.mode, group=group)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    res = runner.run(run_cubes)
    while int((res.terminated_by == 3).sum()) > 0:  # k_cap overflow: widen, untimed
        k_cap *= 2
        runner = P.BatchRunner(shape, cfg, B, k_cap=k_cap, precision=args.precision, device=dev,
                               mode=args.mode, group=group)
        res = runner.run(run_cubes)
    for _ in range(max(3, args.warmup)):
        res = runner.run(run_cubes)
    torch.cuda.synchronize()
    count = res.count.cpu().numpy()
    term = res.terminated_by.cpu().numpy()
    samples = res.samples_used.cpu().numpy()
    iters = res.iterations.cpu().numpy()
    bytes_per_launch = int(samples.sum()) * 8  # complex64 samples gathered (driver.py:208)

    gpu_id = str(local)
    try:
        uuid = torch.cuda.get_device_properties(dev).uuid
        gpu_id = f"GPU-{uuid}"
    except Exception:
        pass
    clocks = ClockSampler(gpu_id)
    clocks.start()
    t_end = time.perf_counter() + args.load_seconds
    while time.perf_counter() < t_end:  # sustained load so sampled clocks reflect it
        for _ in range(10):
            runner.run(run_cubes)
        torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed before each, events around each
    # config 5 recovers *and* re-synthesises every image (BASELINE.json)
    synth = args.config == 5 and not args.no_synth
    img = torch.empty_like(cubes) if synth else None
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if synth:
        ops.synthesize(runner.run(run_cubes), out=img)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(i)
        starts[i].record(stream)
        r = runner.run(run_cubes)
        mids[i].record(stream)
        if synth:
            ops.synthesize(r, out=img)
        ends[i].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    recover_ms = [s.elapsed_time(e) for s, e in zip(starts, mids)]
    synth_ms = [s.elapsed_time(e) for s, e in zip(mids, ends)]
    total_ms = sum(step_ms)
    clk = clocks.stop()
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * B / (ms_per_step / 1e3)

    peak, peak_kind = _peaks()
    rec_ms = sum(recover_ms) / args.steps
    achieved = bytes_per_launch / (rec_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": _traffic(w.name, B),
                "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": bytes_per_launch,
                "kernel": "recover (" + runner.plan["mode"] + " per instance)",
                "kernel_ms": rec_ms,
                "note": "achieved = sum(samples_used)*8 B gathered per launch / mean launch time"}
    if roofline["traffic"]:
        # useful sample bytes per DRAM byte moved (ceiling ~0.33 for scattered 8-byte
        # samples in 64-byte segments)
        roofline["sector_efficiency"] = bytes_per_launch / roofline["traffic"]
    probe = _probe_rate()
    segs = _segments_per_launch(shape, runner.schedule_host, iters, group=group)
    roofline["gather"] = {
        "segments_per_launch": segs, "achieved_segments_per_s": segs / (rec_ms / 1e3),
        "peak_segments_per_s": probe,
        "frac": (segs / (rec_ms / 1e3) / probe) if probe else None,
        "note": "distinct random 64-byte DRAM segments the line gathers touch vs the measured "
                "random-fetch rate of this B200 (tools/gather_probe.cu variant 2, "
                "profiles/r01_gather_probe.txt): the bound of a scattered-sample gather"}
    if synth:
        s_ms = sum(synth_ms) / args.steps
        wbytes = cubes.numel() * cubes.element_size()
        roofline["synthesis"] = {"kernel_ms": s_ms, "bytes_written": wbytes,
                                 "achieved_gbs": wbytes / (s_ms / 1e3) / 1e9,
                                 "frac": wbytes / (s_ms / 1e3) / 1e9 / peak}

    # ---- e2e through the public API: cubes in pinned host memory -> recovered
    #      spectra (and config-5 images) in pinned host memory.  HostBatchRunner
    #      splits each host batch between zero-copy gathers (only the sampled
    #      bytes cross the host link) and double-buffered bulk copies, with the
    #      split tuned untimed on this batch (hostpath.py).
    e2e = None
    if not args.no_e2e:
        from paper_1711_11407_b200.hostpath import HostBatchRunner

        cube_bytes = cubes[0].numel() * cubes.element_size()
        hb = max(1, min(B, (4 << 30) // cube_bytes))  # instances per pinned host batch
        while B % hb:
            hb -= 1
        n_host = B // hb
        host = torch.empty((hb, *cubes.shape[1:]), dtype=cubes.dtype, pin_memory=True)
        host.copy_(cubes[:hb])
        himg = torch.empty_like(host, pin_memory=True) if synth else None
        hr = HostBatchRunner(shape, cfg, hb, k_cap=k_cap, precision=args.precision, device=dev)
        frac = hr.tune(host, himg)
        bz = hr.split_count()
        e_steps = max(1, min(args.steps, 5))
        e_ms = []
        for i in range(e_steps):
            flush.fill_(i)
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            for _ in range(n_host):
                o = hr.run(host, himg)
            b_.record(stream)
            b_.synchronize()
            e_ms.append(a_.elapsed_time(b_))
        zc_samples = int(o["samples_used"][:bz].sum())
        h2d = n_host * ((hb - bz) * cube_bytes + 16 * zc_samples)
        d2h = n_host * (sum(v.numel() * v.element_size() for v in o.values() if v is not None)
                        + (himg.numel() * himg.element_size() if synth else 0))
        e_total = sum(e_ms)
        if dist:
            t = torch.tensor([e_total], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_total = float(t.item())
        e2e = {"value": world * B * e_steps / (e_total / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e_total / e_steps,
               "path": f"{n_host} x {hb} instances from pinned host memory per step: "
                       f"{bz} gathered in place (zero copy), {hb - bz} copied in "
                       f"{hr.chunk}-instance double-buffered chunks (split {frac:.2f} tuned "
                       f"untimed); results{' and images' if synth else ''} to pinned host",
               "note": "h2d counts whole cubes for the copied part and 16 B per gathered "
                       "sample (one 16-byte read request each) for the zero-copy part"}
        del host, himg, hr

    # ---- CPU baseline on this host (rank 0, N=1), same inputs
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        probe = cubes[:2].cpu().numpy()
        per = _estimate_oracle_seconds(probe, w.dims, P.PROFILES[w.profile], args.config)
        n = int(max(cores, min(B, args.cpu_seconds / max(per, 1e-4))))
        sample = cubes[:n].cpu().numpy()
        rate, wall, mean_it = cpu_oracle_throughput(sample, w.dims, P.PROFILES[w.profile],
                                                    args.config, cores, synth=synth)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"instances 0..{n - 1} of this run's {w.name} batch (same complex64 "
                         f"cubes), numpy float64 oracle port, {cores} processes, "
                         f"{wall:.1f} s wall",
               "mean_iterations": mean_it}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "f64",
            "data": "synthetic (seeded; BASELINE.json names no dataset)",
            "config": {"workload": w.name, "instances_per_gpu": B, "dims": list(w.dims),
                       "k": w.k, "profile": w.profile, "k_cap": k_cap,
                       "kernel": runner.plan,
                       "precision": args.precision, "parallelism": f"dp{world} (instances)",
                       "layout": (f"interleaved [B/{group}, *dims, {group}] complex64 (group of "
                                  f"{group} instances per 64-byte sample segment, DESIGN.md 4)"
                                  if group > 1 else "batch-major [B, *dims] complex64"),
                       "l2": "flushed (256 MiB write) before every timed step",
                       "l2_fetch_granularity": {"set": args.l2_fetch, "driver_default": l2_default},
                       "mean_iterations": float(iters.mean()),
                       "recovered_per_instance_mean": float(count.mean()),
                       "terminated_clean": int((term == 0).sum())},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": args.steps * (int(P._native.lib().fpssft_launches_per_batch())
                                          + (1 if synth else 0)),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
