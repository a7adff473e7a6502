#!/usr/bin/env python
"""FPS-SFT throughput on B200: transforms/s over a batch of independent
instances (BASELINE.json config 2 by default: 4096 x 256x256 complex64,
K=100, noiseless, profile P32).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--scaling weak|strong]
    python bench.py --impl reference ...      # the CPU reference arm

One step = one ``fpssft_run_batch`` (one fused kernel launch) over the
rank's batch, cubes resident in HBM.  L2 is flushed (256 MiB write) before
every timed step and only the step is inside the CUDA events.

Multi-GPU: ``--gpus N`` is N ranks, one process per GPU -- started by
torchrun, or spawned here (``shard.launch``) when the environment has no
``WORLD_SIZE``.  ``--scaling weak`` (default: instances are independent, so
the path shards with no data-path collective) gives every rank the config's
whole batch; ``strong`` splits the global batch (4096 instances for config 2,
16384 frames for config 5) into N contiguous slices.  A weak-scaling run with
N > 1 also times the strong-scaling split and reports it as ``strong``.  No
collective sits on the data path: each rank times its own launches, the job
time is the max over ranks, and the padded results are gathered to rank 0
over NCCL after the timed region (timed separately, ``gather``).

The JSON line adds ``roofline`` (algorithmic gather bytes per launch over
the launch time vs the measured HBM copy peak), ``cpu_baseline`` (the CPU
oracle port on this host's cores over a bounded sample of the same
inputs), ``parity`` (the GPU results of exactly those instances against the
oracle's), ``batch_major`` (the same step on the drop-in [B, *dims] layout),
``e2e`` (through the public API from pinned host buffers, copies included)
and ``clocks`` (nvidia-smi sampled during the run).
"""

from __future__ import annotations

import argparse
import glob
import json
import os
import re
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FPS-SFT transforms/sec"
UNIT = "transforms/s"
# recovered-set capacity per config (power of two >= K plus false positives);
# an overflow seen in the untimed warm-up doubles it (reported in run.k_cap)
K_CAP = {1: 64, 2: 128, 3: 512, 4: 2048, 5: 1024}
FLUSH_BYTES = 256 << 20
# north-star amplitude tolerance (BASELINE.json): noiseless / noisy profiles
AMP_TOL = {"P32": 1e-4, "P64": 1e-4, "PN": 1e-3}
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


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


def _traffic(workload_name, batch, full_batch):
    """DRAM bytes per launch of ``batch`` instances from the committed ncu
    capture: a capture of the config's full batch (``full_batch``) or of a
    subset ("<cfgN>_recover_subset<n>"), scaled linearly to ``batch``."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
    except Exception:
        return None
    if workload_name in d:
        return int(d[workload_name] * batch / full_batch)
    pre = workload_name.split("_")[0] + "_recover_subset"
    for k, v in d.items():
        if k.startswith(pre):
            return int(v * batch / int(k[len(pre):]))
    return None


def batch_plan(args, w, world):
    """(global batch, instances per rank) for the scaling mode."""
    B = args.batch or w.batch
    if args.scaling == "weak":
        return B * world, B
    if B % world:
        raise SystemExit(f"strong scaling: global batch {B} is not divisible by {world} ranks")
    return B, B // world


def workload_config(args, w, world):
    """The ``config`` dict of both arms (static: what was asked for, not
    what the run observed), so the driver can match the two lines."""
    B, per = batch_plan(args, w, world)
    return {"workload": w.name, "global_batch": B, "instances_per_rank": per,
            "dims": list(w.dims), "k": w.k, "profile": w.profile,
            "precision": args.precision, "scaling": args.scaling,
            "parallelism": f"dp{world} (instances)",
            "l2": "flushed (256 MiB write) before every timed step"}


# ---------------------------------------------------------------- CPU arms
_SAMPLE = None  # (cubes, dims, profile kwargs, seed, synth, kind) inherited by forked workers


def _ref_module():
    """The unmodified reference package installed in baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "fps_sft")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import fps_sft
    except Exception:
        return None
    if not os.path.abspath(fps_sft.__file__).startswith(REF_DIR):
        return None
    return fps_sft


def _cpu_chunk(idx):
    """Worker: recover ``cubes[idx]`` (and re-synthesise, config 5) with the
    oracle port or the unmodified reference.  Returns (busy seconds,
    per-instance results)."""
    cubes, dims, prof, seed, synth, kind = _SAMPLE
    out = []
    if kind == "reference":
        R = _ref_module()
        shape = R.CubeShape(tuple(dims))
        cfg = R.FpsSftConfig(seed=seed, **prof)
        grid = np.indices(dims).reshape(len(dims), -1).T if synth else None
        t0 = time.perf_counter()
        for i in idx:
            rep = R.fps_sft(R.make_dense_source(cubes[i], shape), cfg)
            if synth:  # the reference's own evaluation of the recovered mixture
                R.make_synthetic_source(rep.recovered).sample_many(grid)
            out.append((i, rep.iterations_run, rep.terminated_by, None, None))
        return time.perf_counter() - t0, out
    from oracle import fps_oracle as O

    p = O.Profile(**prof)
    t0 = time.perf_counter()
    for i in idx:
        rep = O.recover(cubes[i], dims, p, seed=seed)
        if synth:  # config 5 also re-synthesises the image (numpy ifftn of the spectrum)
            O.synthesize(dims, rep.freqs, rep.amps)
        out.append((i, rep.iterations_run, rep.terminated_by, rep.freqs, rep.amps))
    return time.perf_counter() - t0, out


def cpu_throughput(cubes: np.ndarray, dims, prof: dict, seed: int, workers: int,
                   synth: bool = False, kind: str = "port"):
    """instances/s of the CPU path over ``cubes`` on ``workers`` processes
    (the reference's own ProcessPoolExecutor parallelism, oracle.py:275-277):
    instances / max worker busy time.  Also returns the per-instance results
    in instance order."""
    import multiprocessing as mp

    global _SAMPLE
    _SAMPLE = (cubes, tuple(dims), prof, seed, synth, kind)
    n = len(cubes)
    parts = [list(range(i, n, workers)) for i in range(workers)]
    parts = [p for p in parts if p]
    t0 = time.perf_counter()
    if len(parts) == 1:
        res = [_cpu_chunk(parts[0])]
    else:
        with mp.get_context("fork").Pool(len(parts)) as pool:
            res = pool.map(_cpu_chunk, parts)
    wall = time.perf_counter() - t0
    busy = max(r[0] for r in res)
    reports = sorted((x for r in res for x in r[1]), key=lambda x: x[0])
    return n / busy, wall, reports


def _host_sample(w, count, start=0):
    from paper_1711_11407_b200 import workloads as W

    return np.stack([W.make_instance(w, r)[2] for r in W.instance_rngs(w.seed, count, start)])


def _estimate_seconds(cubes, dims, prof, seed, kind, synth=False):
    global _SAMPLE
    _SAMPLE = (cubes, tuple(dims), prof, seed, synth, kind)
    n = min(2, len(cubes))
    busy, _ = _cpu_chunk(list(range(n)))
    return busy / n


def run_reference(args, w, world):
    """``--impl reference``: the unmodified reference (baseline/_ref, its
    public ``fps_sft`` over ``make_dense_source``) on this host's cores, or
    the oracle port when baseline/_ref is absent; bounded sample per step."""
    import paper_1711_11407_b200 as P

    cores = os.cpu_count() or 1
    kind = "reference" if _ref_module() is not None else "port"
    prof = P.PROFILES[w.profile]
    synth = args.config == 5
    probe = _host_sample(w, 2)
    per = _estimate_seconds(probe, w.dims, prof, args.config, kind, synth)
    B, _ = batch_plan(args, w, world)
    # each step: a bounded sample sized for ~args.ref_step_seconds of wall time
    count = int(max(cores, min(B, args.ref_step_seconds * cores / max(per, 1e-4))))
    cubes = _host_sample(w, count)
    for _ in range(args.warmup_ref):
        cpu_throughput(cubes[:cores], w.dims, prof, args.config, cores, synth, kind)
    times, its = [], []
    for _ in range(args.steps):
        rate, wall, reps = cpu_throughput(cubes, w.dims, prof, args.config, cores, synth, kind)
        times.append(count / rate)
        its.append(np.mean([r[1] for r in reps]))
    total = sum(times)
    value = count * args.steps / total
    what = ("unmodified reference fps_sft 0.1.0 (baseline/_ref) on make_dense_source"
            if kind == "reference" else "numpy float64 oracle port (baseline/_ref absent)")
    sample = (f"{count} of the {B} instances of {w.name} (instances 0..{count - 1}) per step, "
              f"{what}, {cores} worker processes"
              + (", recovery + re-synthesis of each frame" if synth else ""))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; BASELINE.json names no dataset)",
        "config": workload_config(args, w, world),
        "impl": "reference",
        "run": {"mean_iterations": float(np.mean(its)), "batch_per_step": count},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
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


# ---------------------------------------------------------------- parity
def parity_summary(gpu: dict, reports, tol: float) -> dict:
    """GPU results of the sampled instances vs the oracle's reports of the
    same cubes: support, iterations/termination and amplitudes (north-star
    tolerance ``tol``, relative, on identical supports)."""
    from paper_1711_11407_b200 import _native as N

    n = len(reports)
    same_sup = same_it = 0
    worst = 0.0
    for i, its, term, freqs, amps in reports:
        c = int(gpu["count"][i])
        f = gpu["freqs"][i, :c].astype(np.int64)
        a = gpu["amps"][i, :c]
        if f.shape == freqs.shape and np.array_equal(f, freqs):
            same_sup += 1
            if c:
                worst = max(worst, float(np.max(np.abs(a - amps) / np.abs(amps))))
        same_it += (int(gpu["iterations"][i]) == its
                    and N.TERM_NAMES[int(gpu["terminated_by"][i])] == term)
    return {"instances": n, "identical_support": same_sup, "identical_iterations": same_it,
            "max_rel_amp_err": worst, "tolerance": tol,
            "pass": same_sup == n and same_it == n and worst <= tol,
            # BASELINE.json north star: support bit-exact, amplitudes within tolerance
            "north_star_pass": same_sup == n and worst <= tol,
            "oracle": "oracle/fps_oracle.py (float64 numpy port, pinned to the reference's "
                      "golden runs), same complex64 cubes and schedule"}


# ---------------------------------------------------------------- NCCL evidence
def _nccl_log_setup(rank):
    if "NCCL_DEBUG" in os.environ:
        return None
    path = os.path.join(tempfile.gettempdir(), f"fpssft_bench_nccl.{os.getpid()}.log")
    os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT,NVLS",
                      NCCL_DEBUG_FILE=path)
    return path


def _nccl_log_summary(path):
    if not path:
        return None
    txt = ""
    for p in glob.glob(path + "*") + [path]:
        try:
            txt += open(p).read()
        except OSError:
            pass
    m = re.findall(r"nRanks (\d+)", txt)
    return {"nranks": int(m[-1]) if m else None,
            "nvls": bool(re.search(r"NVLS multicast support is available", txt)),
            "version": (re.findall(r"NCCL version ([0-9.]+)", txt) or [None])[-1]}


# ---------------------------------------------------------------- GPU arm
def _time_steps(run, steps, stream, flush, after=None):
    """Per-step CUDA-event times (ms) of ``run()`` (and ``after(result)``),
    L2 flushed before each step, outside the events."""
    import torch

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i)
        starts[i].record(stream)
        r = run()
        mids[i].record(stream)
        if after is not None:
            after(r)
        ends[i].record(stream)
    torch.cuda.synchronize()
    return ([s.elapsed_time(e) for s, e in zip(starts, ends)],
            [s.elapsed_time(e) for s, e in zip(starts, mids)],
            [s.elapsed_time(e) for s, e in zip(mids, ends)])


def gpu_rank(args):
    import torch

    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import ops
    from paper_1711_11407_b200 import shard
    from paper_1711_11407_b200 import workloads as W

    rank, local, world = shard.env_rank()
    w = W.CONFIGS[args.config]
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the GPU arm has no CPU path)")
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} wants cuda:{local} but only "
                         f"{torch.cuda.device_count()} GPU(s) are visible")
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    l2_default = P._native.get_l2_fetch_granularity(dev)
    if args.l2_fetch:
        P._native.set_l2_fetch_granularity(args.l2_fetch, dev)
    dist = None
    nccl_log = None
    if world > 1:
        import torch.distributed as dist

        nccl_log = _nccl_log_setup(rank)
        dist.init_process_group("nccl", device_id=dev)
        ones = torch.ones(1, device=dev)
        dist.all_reduce(ones)  # communicator up; its size is checked below
        comm_check = int(ones.item())

    B_total, B = batch_plan(args, w, world)
    if args.scaling == "weak":
        b0, b1 = shard.instance_range(rank, world, per_rank=B)
    else:
        b0, b1 = shard.instance_range(rank, world, total=B_total)
    shape = P.CubeShape(w.dims)
    cfg = _cfg(w, args.config)
    k_cap = args.k_cap or K_CAP[args.config]

    # ---- inputs: this rank's spectra on the host, cubes synthesised on its device
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

    def make_runner(kc, grp, batch=B):
        return P.BatchRunner(shape, cfg, batch, k_cap=kc, precision=args.precision, device=dev,
                             mode=args.mode, group=grp)

    runner = make_runner(k_cap, group)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    res = runner.run(run_cubes)
    while int((res.terminated_by == 3).sum()) > 0:  # k_cap overflow: widen, untimed
        k_cap *= 2
        runner = make_runner(k_cap, group)
        res = runner.run(run_cubes)
    for _ in range(max(3, args.warmup)):
        res = runner.run(run_cubes)
    torch.cuda.synchronize()
    host_res = {k: v.cpu().numpy() for k, v in runner.out.items() if v is not None}
    count, term = host_res["count"], host_res["terminated_by"]
    samples, iters = host_res["samples_used"], host_res["iterations"]
    bytes_per_launch = int(samples.sum()) * 8  # complex64 samples gathered (driver.py:208)

    gpu_id = str(local)
    try:
        gpu_id = f"GPU-{torch.cuda.get_device_properties(dev).uuid}"
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
    if synth:
        ops.synthesize(runner.run(run_cubes), out=img)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, recover_ms, synth_ms = _time_steps(
        lambda: runner.run(run_cubes), args.steps, stream, flush,
        (lambda r: ops.synthesize(r, out=img)) if synth else None)
    if dist:
        dist.barrier()
    clk = clocks.stop()
    total_ms = shard.max_over_ranks(sum(step_ms), dev)
    ms_per_step = total_ms / args.steps
    value = B_total / (ms_per_step / 1e3)

    # ---- the same step on the batch-major layout the drop-in receives
    batch_major = None
    if group > 1 and not args.no_batch_major:
        bm = make_runner(k_cap, 1)
        for _ in range(max(3, args.warmup)):
            bm.run(cubes)
        torch.cuda.synchronize()
        bm_ms, _, _ = _time_steps(lambda: bm.run(cubes), args.steps, stream, flush)
        bm_total = shard.max_over_ranks(sum(bm_ms), dev)
        same = all(torch.equal(bm.out[k], runner.out[k]) for k in bm.out if bm.out[k] is not None)
        batch_major = {"value": B_total / (bm_total / args.steps / 1e3), "unit": UNIT,
                       "ms_per_step": bm_total / args.steps,
                       "layout": "batch-major [B, *dims] complex64 (what fps_sft_batch and "
                                 "make_dense_source users hand in)",
                       "outputs_identical_to_interleaved": bool(same)}
        del bm

    # ---- N > 1, weak scaling: the strong-scaling point too -- the config's
    #      global batch split over the ranks (instances r*B/N .. (r+1)*B/N-1
    #      of the same instance stream), timed the same way
    strong = None
    if world > 1 and args.scaling == "weak" and B % world == 0 and not args.no_strong:
        sb = B // world
        s0, _ = shard.instance_range(rank, world, total=B)
        s_cubes = W.synthesize_batch_torch(w.dims, W.make_spectra(w, sb, s0), dev, w.noise_var,
                                           noise_seed=w.seed * 1000003 + s0)
        s_group = group if sb % group == 0 else 1
        s_run = P.interleave(s_cubes, s_group) if s_group > 1 else s_cubes
        sr = make_runner(k_cap, s_group, sb)
        for _ in range(max(3, args.warmup)):
            sr.run(s_run)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        s_ms, _, _ = _time_steps(lambda: sr.run(s_run), args.steps, stream, flush,
                                 (lambda r: ops.synthesize(r, out=s_cubes)) if synth else None)
        s_total = shard.max_over_ranks(sum(s_ms), dev)
        strong = {"value": B / (s_total / args.steps / 1e3), "unit": UNIT,
                  "ms_per_step": s_total / args.steps, "global_batch": B,
                  "instances_per_rank": sb,
                  "note": "strong scaling: the config's global batch split over the ranks "
                          "(the main line is weak scaling: every rank a whole batch)"}
        del sr, s_run, s_cubes

    # ---- result gather to rank 0 over NCCL (after the timed region, timed alone)
    gather = None
    if dist:
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        got = shard.gather_results(runner.out, dst=0)
        g1.record(stream)
        torch.cuda.synchronize()
        g_ms = shard.max_over_ranks(g0.elapsed_time(g1), dev)
        ok = None
        if rank == 0:
            ok = int(got["count"].shape[0]) == B * world
        gather = {"ms": g_ms, "bytes_per_rank": shard.result_bytes(runner.out),
                  "collective": "torch.distributed.gather to rank 0 (NCCL)",
                  "rows_on_rank0": int(got["count"].shape[0]) if rank == 0 else None,
                  "complete": ok}

    peak, peak_kind = _peaks()
    rec_ms = sum(recover_ms) / args.steps
    achieved = bytes_per_launch / (rec_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": _traffic(w.name, B, w.batch),
                "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": bytes_per_launch,
                "kernel": "recover (" + runner.plan["mode"] + " per instance)",
                "kernel_ms": rec_ms,
                "note": "achieved = sum(samples_used)*8 B gathered per launch / mean launch time"}
    if roofline["traffic"]:
        # useful sample bytes per DRAM byte moved
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
    #      spectra (and config-5 images) in pinned host memory (hostpath.py)
    e2e = e2e_bm = None
    if not args.no_e2e:
        from paper_1711_11407_b200.hostpath import HostBatchRunner

        e_steps = max(1, min(args.steps, 5))

        def time_host(hr, host, himg, n_host):
            e_ms = []
            for i in range(e_steps):
                flush.fill_(i)
                torch.cuda.synchronize()
                a_ = torch.cuda.Event(enable_timing=True)
                b_ = torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                for _ in range(n_host):
                    o = hr.run(host, himg)
                b_.record(stream)
                b_.synchronize()
                e_ms.append(a_.elapsed_time(b_))
            return o, shard.max_over_ranks(sum(e_ms), dev)

        def out_bytes(o):
            return sum(v.numel() * v.element_size() for v in o.values() if v is not None)

        # (a) batch-major host cubes, what a user of make_dense_source holds:
        #     zero-copy / bulk-copy split tuned untimed
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
        o, e_total = time_host(hr, host, himg, n_host)
        zc_samples = int(o["samples_used"][:bz].sum())
        h2d = n_host * ((hb - bz) * cube_bytes + 16 * zc_samples)
        d2h = n_host * (out_bytes(o) + (himg.numel() * himg.element_size() if synth else 0))
        e2e_bm = {"value": B_total * e_steps / (e_total / 1e3), "unit": UNIT,
                  "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                  "ms_per_step": e_total / e_steps,
                  "path": f"batch-major [B, *dims] pinned host cubes, {n_host} x {hb} instances "
                          f"per step per rank: {bz} gathered in place (zero copy), {hb - bz} "
                          f"copied in {hr.chunk}-instance double-buffered chunks (split "
                          f"{frac:.2f} tuned untimed); results"
                          f"{' and images' if synth else ''} to pinned host",
                  "note": "h2d counts whole cubes for the copied part and 16 B per gathered "
                          "sample (one 16-byte read request each) for the zero-copy part"}
        del host, himg, hr
        e2e = e2e_bm
        # (b) the same batch in the interleaved layout on the host (the layout
        #     `value` is measured on): every instance gathered in place by the
        #     group kernel, one 64-byte PCIe read per segment serving `group`
        #     instances
        hg = args.host_group
        if group > 1 and not synth and hg > 1 and B % hg == 0:
            host_il = P.interleave(cubes, hg)
            host = torch.empty(host_il.shape, dtype=host_il.dtype, pin_memory=True)
            host.copy_(host_il)
            del host_il
            hr = HostBatchRunner(shape, cfg, B, k_cap=k_cap, precision=args.precision,
                                 device=dev, group=hg)
            hr.run(host)
            o, e_total = time_host(hr, host, None, 1)
            segs_h = _segments_per_launch(shape, hr._runner(0, B).schedule_host,
                                          o["iterations"].numpy(), group=hg)
            e2e_il = {"value": B_total * e_steps / (e_total / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": int(64 * segs_h), "d2h_bytes_per_step": out_bytes(o),
                   "ms_per_step": e_total / e_steps,
                   "path": f"interleaved [B/{hg}, *dims, {hg}] pinned host cubes, all {B} "
                           f"instances per step gathered in place by the group kernel (zero "
                           f"copy: one {8 * hg}-byte PCIe read per sample position serves {hg} "
                           f"instances); results to pinned host",
                   "note": "h2d = distinct 64-byte segments the gathers touch x 64 B",
                   "outputs_identical_to_device_run": bool(all(
                       torch.equal(o[k], runner.out[k].cpu()) for k in o if o[k] is not None))}
            del host, hr
            # the interleaved host layout pays off where the group-gather kernel
            # serves it (one read per segment for the group); elsewhere each
            # instance reads its own chunks and the batch-major split is faster:
            # e2e is the faster of the two, both are reported
            if e2e_il["value"] > e2e_bm["value"]:
                e2e = e2e_il
            else:
                e2e_il["note"] += " (slower than the batch-major path for this shape: not e2e)"
                e2e["e2e_interleaved_host"] = e2e_il
        # (c) interleaved by --host-stage-group (32: 256-byte segments) with the
        #     first --host-stage-iterations iterations' line samples staged
        #     through HBM by TMA bulk copies (fpssft_run_batch_staged): the link's
        #     bulk rate instead of the SM loads' request rate
        sg, st0 = args.host_stage_group, args.host_stage_iterations
        if st0 == 0:  # auto: the slowest instance's iterations in the device run (untimed)
            st0 = int(runner.out["iterations"].max())
        # (re-synthesis configs: the same host batches as (a), images back to the host)
        hb_c, n_c = (hb, n_host) if synth else (B, 1)
        if group > 1 and sg > 1 and st0 > 0 and hb_c % sg == 0:
            try:
                pipe = (args.host_stage_pipeline
                        if not synth and hb_c % (sg * args.host_stage_pipeline) == 0 else 1)
                hr = HostBatchRunner(shape, cfg, hb_c, k_cap=k_cap, precision=args.precision,
                                     device=dev, group=sg, stage_iterations=st0, pipeline=pipe)
                host_il = P.interleave(cubes[:hb_c], sg)
                host = torch.empty(host_il.shape, dtype=host_il.dtype, pin_memory=True)
                host.copy_(host_il)
                del host_il
                himg = (torch.empty((hb_c, *shape.dims), dtype=torch.complex64, pin_memory=True)
                        if synth else None)
                hr.run(host, himg)
            except ValueError:  # no staged read path for this shape / precision
                hr = None
            if hr is not None:
                o, e_total = time_host(hr, host, himg, n_c)
                nll = (shape.ndim + 1) * shape.line_len
                its = o["iterations"].numpy().astype(np.int64)
                t0 = min(st0, hr.t_max)
                if shape.ndim == 2 and shape.line_len == 256:  # the group-gather kernel
                    late_b = np.maximum(its.reshape(-1, 8).max(axis=1) - t0, 0).sum() * nll * 64
                else:  # per-instance kernels: one 32-byte sector per late sample
                    late_b = np.maximum(its - t0, 0).sum() * nll * 32
                staged_b = (hb_c // sg) * t0 * nll * 8 * sg
                img_b = himg.numel() * himg.element_size() if synth else 0
                chunks = (f"{pipe} chunks pipelined (chunk i+1 staged while chunk i recovers and "
                          f"its results return)" if not synth else
                          f"{n_c} x {hb_c} instances per step in {hr.chunk}-instance chunks over "
                          f"three streams (staging || recovery + re-synthesis || images back)")
                e2e_st = {"value": B_total * e_steps / (e_total / 1e3), "unit": UNIT,
                          "h2d_bytes_per_step": int(n_c * (staged_b + late_b)),
                          "d2h_bytes_per_step": int(n_c * (out_bytes(o) + img_b)),
                          "ms_per_step": e_total / e_steps,
                          "path": f"interleaved [B/{sg}, *dims, {sg}] pinned host cubes: the line "
                                  f"samples of iterations 0..{t0 - 1} staged through HBM by one "
                                  f"TMA bulk copy per {8 * sg}-byte segment "
                                  f"(fpssft_run_batch_staged), later iterations gathered in place; "
                                  f"{chunks}; results{' and images' if synth else ''} to pinned "
                                  f"host",
                          "note": "h2d = staged segments x segment bytes + the in-place reads of "
                                  "iterations past the staged ones (64 B per position and "
                                  "8-instance team, or 32 B per sample for per-instance kernels)",
                          "outputs_identical_to_device_run": bool(all(
                              torch.equal(o[k], runner.out[k][:hb_c].cpu()) for k in o
                              if o[k] is not None))}
                del host, hr, himg
                if e2e_st["value"] > e2e["value"]:
                    prev = e2e
                    e2e = e2e_st
                    if prev is not e2e_bm:
                        e2e["e2e_zero_copy_interleaved"] = prev
                else:
                    e2e["e2e_staged"] = e2e_st

    # ---- CPU baseline on this host (rank 0, N=1), same inputs; parity of the
    #      GPU results of exactly those instances against the oracle's
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        prof = P.PROFILES[w.profile]
        probe_c = cubes[:2].cpu().numpy()
        per = _estimate_seconds(probe_c, w.dims, prof, args.config, "port", synth)
        n = int(max(cores, min(B, args.cpu_seconds / max(per, 1e-4))))
        sample = cubes[:n].cpu().numpy()
        rate, wall, reps = cpu_throughput(sample, w.dims, prof, args.config, cores,
                                          synth=synth)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"instances 0..{n - 1} of this run's {w.name} batch (same complex64 "
                         f"cubes), numpy float64 oracle port, {cores} processes, "
                         f"{wall:.1f} s wall",
               "mean_iterations": float(np.mean([r[1] for r in reps]))}
        parity = parity_summary(host_res, reps, AMP_TOL[w.profile])

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic (seeded; BASELINE.json names no dataset)",
            "config": workload_config(args, w, world),
            "run": {"k_cap": k_cap, "kernel": runner.plan,
                    "arithmetic": {0: "fp32", 1: "fp64", 2: "fp32-guarded"}[runner.prec],
                    "layout": (f"interleaved [B/{group}, *dims, {group}] complex64 (group of "
                               f"{group} instances per 64-byte sample segment, DESIGN.md 4)"
                               if group > 1 else "batch-major [B, *dims] complex64"),
                    "l2_fetch_granularity": {"set": args.l2_fetch, "driver_default": l2_default},
                    "mean_iterations": float(iters.mean()),
                    "recovered_per_instance_mean": float(count.mean()),
                    "terminated_clean": int((term == 0).sum()),
                    "rank0_instances": [b0, b1]},
            "roofline": roofline, "parity": parity, "cpu_baseline": cpu,
            "batch_major": batch_major, "e2e": e2e, "e2e_batch_major": e2e_bm, "clocks": clk,
            "gpu_launches": args.steps * (int(P._native.lib().fpssft_launches_per_batch())
                                          + (1 if synth else 0)),
        }
        if world > 1:
            line["comm"] = {"backend": "nccl", "world": world, "allreduce_ones": comm_check,
                            "log": _nccl_log_summary(nccl_log)}
            line["gather"] = gather
            line["strong"] = strong
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-strong", action="store_true",
                    help="N > 1, weak scaling: skip the strong-scaling point")
    ap.add_argument("--scaling", default="weak", choices=["strong", "weak"],
                    help="strong: the config's global batch split over the ranks; weak: the "
                         "whole batch on every rank")
    ap.add_argument("--precision", default="auto",
                    choices=["auto", "fp32", "fp32-guarded", "fp64"],
                    help="auto: float32, guarded (exact float64 decisions) for the noisy "
                         "profile; see driver._precision_code")
    ap.add_argument("--layout", default="auto", choices=["auto", "batch_major", "interleaved"],
                    help="HBM layout of the batch: [B, *dims], or [B/G, *dims, G] with G "
                         "instances interleaved sample by sample (--group); auto = "
                         "interleaved for batches of >= 64 instances")
    ap.add_argument("--group", type=int, default=8)
    ap.add_argument("--host-group", type=int, default=16,
                    help="interleave group of the e2e host batch (16: one 128-byte PCIe read "
                         "per position serves 16 instances; 1 = batch-major only)")
    ap.add_argument("--mode", default="auto", choices=["auto", "warp", "cta"],
                    help="kernel family (auto: the planner's choice for this batch)")
    ap.add_argument("--batch", type=int, default=None,
                    help="override the global batch (strong) / per-rank batch (weak)")
    ap.add_argument("--k-cap", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU-seconds budget of the cpu_baseline sample")
    ap.add_argument("--ref-step-seconds", type=float, default=4.0)
    ap.add_argument("--warmup-ref", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--host-stage-group", type=int, default=32,
                    help="interleave group of the staged e2e host batch (32: 256-byte segments, "
                         "one TMA bulk copy each; 0 = off)")
    ap.add_argument("--host-stage-pipeline", type=int, default=4,
                    help="chunks of the staged e2e batch pipelined over two streams")
    ap.add_argument("--host-stage-iterations", type=int, default=0,
                    help="iterations whose line samples the staged e2e path copies up front "
                         "(0 = the slowest instance's count in the device run, found untimed)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-batch-major", action="store_true")
    ap.add_argument("--no-synth", action="store_true", help="config 5 without re-synthesis")
    ap.add_argument("--l2-fetch", type=int, default=32,
                    help="cudaLimitMaxL2FetchGranularity in bytes (0 = leave the driver default)")
    ap.add_argument("--load-seconds", type=float, default=1.0,
                    help="back-to-back steps before the timed region (clock ramp/sampling)")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")

    from paper_1711_11407_b200 import shard
    from paper_1711_11407_b200 import workloads as W

    if args.impl == "reference":
        rank, _, world = shard.env_rank()
        if "WORLD_SIZE" not in os.environ:
            world = args.gpus
        if rank == 0:  # one CPU measurement for the job; other ranks have no work
            run_reference(args, W.CONFIGS[args.config], world)
        return
    shard.launch(args.gpus, gpu_rank, args)


if __name__ == "__main__":
    main()
