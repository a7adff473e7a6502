"""Recovery of batches whose cubes live in pinned HOST memory.

The reference's users hand ``fps_sft`` a host array (``make_dense_source``,
``/root/reference/pkg/src/fps_sft/core.py:276-278``); at batch scale the
cost of reaching the GPU is the host link, not the recovery kernel (config 2:
2 GiB of cubes at ~55 GB/s = 39 ms against 0.2 ms of recovery).  FPS-SFT
reads only ``samples_used`` of the N samples of each cube (sub-linear sample
complexity, ``driver.py:208``), so a cube need not cross the link at all: the
recovery kernel can gather its samples straight out of the pinned host
buffer (zero copy, UVA).  This module moves every batch through two
concurrent paths and splits the instances between them:

* zero copy: the first ``Bz`` instances are recovered by ``BatchRunner.run``
  on the pinned host tensor itself -- only the gathered samples cross the
  link, at the host's random-read rate (~3.6e8 samples/s measured, 16-byte
  requests; ``tools/host_gather_probe.cu``);
* bulk copy: the remaining instances stream through double-buffered device
  chunks (H2D on one stream, recovery on another, results back on a third),
  at the host link's bulk rate.

``mode="auto"`` sizes the split from a cost model (``zero_copy_split``) fed
with the mean ``samples_used`` of the previous batch (the first batch goes
through the copy path); ``tune()`` replaces the model by measuring a few
splits on a real batch (untimed, like a cuFFT plan); ``"zero_copy"`` /
``"copy"`` force one path, ``"split"`` takes an explicit fraction.  Results
are identical whichever path an instance takes (the kernels are the same;
tested).  Outputs land in pinned host tensors.

Measured on one B200 behind PCIe Gen5 (``profiles/r01_hostpath.jsonl``):
config 2 batches cross 2x faster split 0.8/0.2 than copied whole, config 4
4.5x faster zero-copied; config 5 (30 % of each cube sampled, images
returned) stays on the copy path, where H2D and D2H overlap.
"""

from __future__ import annotations

import numpy as np

from .core import CubeShape
from .driver import BatchRunner, FpsSftConfig, allocate_outputs, default_max_iterations

# measured on the B200 pool (tools/host_gather_probe.cu, tools/zero_copy_probe.py)
ZC_SAMPLES_PER_S = 3.6e8
H2D_BYTES_PER_S = 5.5e10


def zero_copy_split(mean_samples: float, cube_samples: int, *, zc_rate: float = ZC_SAMPLES_PER_S,
                    h2d_rate: float = H2D_BYTES_PER_S) -> float:
    """Fraction of a batch to gather in place from host memory: the split at
    which the zero-copy part (``mean_samples`` random reads per instance at
    ``zc_rate``) and the copied part (whole complex64 cubes at ``h2d_rate``)
    take equal time.  Fractions below 5 % are not worth a second launch."""
    if mean_samples <= 0:
        return 1.0
    t_z = mean_samples / zc_rate
    t_c = cube_samples * 8 / h2d_rate
    f = t_c / (t_z + t_c)
    return f if f > 0.05 else 0.0


class HostBatchRunner:
    """Recover ``[batch, *dims]`` complex64 cubes held in pinned host memory.

    ``run(host_cubes)`` returns the per-instance outputs as pinned host
    tensors (the ``allocate_outputs`` dict); ``run(host_cubes, images)`` also
    re-synthesises every recovered spectrum (config 5) into the pinned host
    tensor ``images``.
    """

    def __init__(self, shape: CubeShape, config: FpsSftConfig, batch: int, *,
                 k_cap: int = 256, precision: str = "auto", device=None, mode: str = "auto",
                 zero_copy_fraction: float | None = None, chunk: int | None = None,
                 chunk_bytes: int = 256 << 20, schedule=None, sched_index=None,
                 graphs: bool = True, group: int = 1, stage_iterations: int = 0,
                 pipeline: int = 1):
        import torch

        if mode not in ("auto", "copy", "zero_copy", "split"):
            raise ValueError("mode must be auto, copy, zero_copy or split")
        # group > 1: the host batch is interleaved [ceil(B/G), *dims, G] (the
        # producer's layout choice, like the device bench's): every batch is
        # gathered in place by the group kernel, one PCIe read per 64-byte
        # segment serving G instances (config 2: 6.7 vs 23 ms per batch
        # batch-major, tools/zc_group_probe.py)
        self.group = int(group)
        # stage_iterations > 0: the first iterations' line samples cross the
        # link as TMA bulk copies of whole 8 G-byte segments into an HBM staging
        # buffer (fpssft_run_batch_staged; G = 32: 256-byte segments at the
        # link's bulk rate, tools/seg_probe.cu), later iterations in place
        self.stage_iterations = int(stage_iterations)
        if self.stage_iterations and self.group < 2:
            raise ValueError("staged lines need an interleaved host batch (group >= 2)")
        # pipeline > 1 (staged lines): the batch goes in that many chunks, chunk
        # i+1 staged over the host link while chunk i recovers and its results
        # return (two streams, the recovery one at high priority)
        self.pipeline = max(1, int(pipeline))
        if self.pipeline > 1 and (not self.stage_iterations
                                  or int(batch) % (self.group * self.pipeline)):
            raise ValueError("pipeline needs staged lines and a batch of whole groups per chunk")
        if self.group > 1:
            if mode not in ("auto", "zero_copy"):
                raise ValueError("an interleaved host batch is gathered in place (zero_copy)")
            if sched_index is not None:
                raise ValueError("an interleaved host batch shares one schedule")
            mode = "zero_copy"
        if mode == "split" and zero_copy_fraction is None:
            raise ValueError("split mode needs zero_copy_fraction")
        self.shape, self.config, self.batch = shape, config, int(batch)
        self.mode = mode
        self.fraction = zero_copy_fraction
        self.device = torch.device(device if device is not None else "cuda")
        self.k_cap, self.precision = k_cap, precision
        self.t_max = config.max_iterations or default_max_iterations(shape)
        cube_bytes = shape.n_total * 8
        self.chunk = int(chunk or max(1, min(self.batch, chunk_bytes // cube_bytes)))
        self._schedule = schedule
        self._sched_index = None if sched_index is None else np.asarray(sched_index, np.int32)
        self.out = allocate_outputs(self.batch, shape, k_cap, self.t_max, "cpu", pin=True)
        self.last_mean_samples: float | None = None
        self.tuned: dict | None = None
        self.graphs = graphs
        self._graphs: dict = {}
        self._runners: dict = {}
        self._bufs: list = []
        self._img_bufs: list = []
        self._streams = None
        self._pipe_streams = None

    # ------------------------------------------------------------------ plan
    def split_count(self) -> int:
        """Instances that take the zero-copy path in the next ``run``."""
        if self.mode == "copy":
            return 0
        if self.mode == "zero_copy":
            return self.batch
        if self.mode == "split":
            return int(round(self.fraction * self.batch))
        if self.last_mean_samples is None:
            return 0
        return int(self.batch * zero_copy_split(self.last_mean_samples, self.shape.n_total))

    def tune(self, host_cubes, images=None, fractions=None) -> float:
        """Measure a few zero-copy fractions on ``host_cubes`` (one timed run
        each after a warm run) and keep the fastest (mode becomes "split").
        Returns the chosen fraction."""
        import time

        if fractions is None:
            self.run(host_cubes, images)  # learns the sample count
            f0 = self.split_count() / max(1, self.batch)
            fractions = sorted({0.0, 1.0, round(f0, 3), 0.35, 0.5, 0.65, 0.7, 0.75, 0.8, 0.85,
                                0.9, 0.95})
        best = None
        for f in fractions:
            self.mode, self.fraction = "split", float(f)
            self.run(host_cubes, images)
            t0 = time.perf_counter()
            self.run(host_cubes, images)
            dt = time.perf_counter() - t0
            if best is None or dt < best[0]:
                best = (dt, float(f))
        self.fraction = best[1]
        self.tuned = {"fraction": best[1], "ms": best[0] * 1e3}
        return best[1]

    def _runner(self, b0: int, n: int) -> BatchRunner:
        key = (b0, n)
        r = self._runners.get(key)
        if r is None:
            si = None if self._sched_index is None else self._sched_index[b0:b0 + n]
            r = BatchRunner(self.shape, self.config, n, schedule=self._schedule, sched_index=si,
                            k_cap=self.k_cap, precision=self.precision, device=self.device,
                            group=self.group, stage_iterations=self.stage_iterations)
            self._runners[key] = r
        return r

    def _ensure_buffers(self, synth: bool):
        import torch

        if self._streams is None:
            self._streams = [torch.cuda.Stream(self.device) for _ in range(4)]
        nbuf = 2
        while len(self._bufs) < nbuf:
            self._bufs.append(torch.empty((self.chunk, *self.shape.dims), dtype=torch.complex64,
                                          device=self.device))
        while synth and len(self._img_bufs) < nbuf:
            self._img_bufs.append(torch.empty((self.chunk, *self.shape.dims),
                                              dtype=torch.complex64, device=self.device))

    def _launch_in_place(self, host_cubes):
        """Everything of an in-place / staged run, enqueued behind the current
        stream: one launch (pair) and the result copy, or the staged chunks
        pipelined over two streams."""
        import torch

        if self.pipeline == 1:
            r = self._runner(0, self.batch)
            r.run(host_cubes)
            self._copy_out(r, 0, self.batch)
            return
        if self._pipe_streams is None:
            self._pipe_streams = (torch.cuda.Stream(self.device),
                                  torch.cuda.Stream(self.device, priority=-1))
        s_stage, s_run = self._pipe_streams
        cur = torch.cuda.current_stream(self.device)
        s_stage.wait_stream(cur)
        s_run.wait_stream(cur)
        n, G = self.batch // self.pipeline, self.group
        for i in range(self.pipeline):
            b0 = i * n
            r = self._runner(b0, n)
            hc = host_cubes[b0 // G:(b0 + n) // G]
            with torch.cuda.stream(s_stage):
                r.stage(hc)
                ev = torch.cuda.Event()
                ev.record(s_stage)
            with torch.cuda.stream(s_run):
                s_run.wait_event(ev)
                r.run(hc, staged=True)
                self._copy_out(r, b0, n)
        cur.wait_stream(s_stage)
        cur.wait_stream(s_run)

    def _run_staged_synth(self, host_cubes, images) -> dict:
        """Interleaved host batch, staged lines, images back to the host
        (config 5): chunk by chunk over three streams -- the line samples of
        chunk i+1 cross the link (TMA staging) while chunk i recovers and
        re-synthesises and the images of chunk i-1 return.  Only the sampled
        segments go up, so the link's downstream direction carries the images
        at its full rate."""
        import torch

        from .ops import synthesize

        G = self.group
        n = max(G, self.chunk // G * G)
        if self._pipe_streams is None:
            self._pipe_streams = (torch.cuda.Stream(self.device),
                                  torch.cuda.Stream(self.device, priority=-1))
        if self._streams is None:
            self._streams = [torch.cuda.Stream(self.device) for _ in range(4)]
        # recovery at high priority: its CTAs are placed before the staging
        # grid's pending ones
        (s_stage, s_run), s_d2h = self._pipe_streams, self._streams[2]
        while len(self._img_bufs) < 2:
            self._img_bufs.append(torch.empty((min(n, self.batch), *self.shape.dims),
                                              dtype=torch.complex64, device=self.device))
        cur = torch.cuda.current_stream(self.device)
        for s in (s_stage, s_run, s_d2h):
            s.wait_stream(cur)
        ev_free = [None, None]
        for k, b0 in enumerate(range(0, self.batch, n)):
            m = min(n, self.batch - b0)
            i = k & 1
            r = self._runner(b0, m)
            hc = host_cubes[b0 // G:(b0 + m + G - 1) // G]
            with torch.cuda.stream(s_stage):
                r.stage(hc)
                ev_st = torch.cuda.Event()
                ev_st.record(s_stage)
            with torch.cuda.stream(s_run):
                s_run.wait_event(ev_st)
                if ev_free[i] is not None:
                    s_run.wait_event(ev_free[i])
                res = r.run(hc, staged=True)
                self._copy_out(r, b0, m)
                img = self._img_bufs[i][:m]
                synthesize(res, out=img)
                ev_img = torch.cuda.Event()
                ev_img.record(s_run)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_img)
                images[b0:b0 + m].copy_(img, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_d2h)
                ev_free[i] = ev
        for s in (s_stage, s_run, s_d2h):
            cur.wait_stream(s)
        cur.synchronize()
        if self.mode == "auto":
            self.last_mean_samples = float(self.out["samples_used"].double().mean())
        return self.out

    def _graph_for(self, host_cubes):
        """CUDA graph of (zero-copy recovery + result copy) for this host
        buffer: the launch sequence of a small batch costs more on the host
        than on the device (config 1: one instance, 24 us of kernel).  None if
        the capture is refused (then the stream path runs)."""
        import torch

        key = (host_cubes.data_ptr(), tuple(host_cubes.shape))
        if key in self._graphs:
            return self._graphs[key]
        g = None
        try:
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):  # warm: plans and attributes set outside capture
                self._launch_in_place(host_cubes)
            side.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self._launch_in_place(host_cubes)
        except RuntimeError:
            g = None
            torch.cuda.synchronize(self.device)
        self._graphs[key] = g
        return g

    def _copy_out(self, r: BatchRunner, b0: int, n: int):
        if b0 == 0 and n == self.batch:  # same packed layout: one copy
            self.out.buf.copy_(r.out.buf, non_blocking=True)
            return
        for k, v in r.out.items():
            if v is not None:
                self.out[k][b0:b0 + n].copy_(v, non_blocking=True)

    # ------------------------------------------------------------------- run
    def run(self, host_cubes, images=None) -> dict:
        """Recover every instance of the pinned host tensor ``host_cubes``;
        with ``images`` (pinned host, same shape) also write each instance's
        re-synthesised grid.  Blocks until the outputs are on the host."""
        import torch

        from .ops import synthesize

        if not (isinstance(host_cubes, torch.Tensor) and not host_cubes.is_cuda
                and host_cubes.is_pinned()):
            raise ValueError("host_cubes must be a pinned host tensor")
        G = self.group
        want = ((self.batch, *self.shape.dims) if G == 1
                else (-(-self.batch // G), *self.shape.dims, G))
        if tuple(host_cubes.shape) != want or host_cubes.dtype != torch.complex64:
            raise ValueError(f"host_cubes must be complex64 {list(want)}")
        if not host_cubes.is_contiguous():
            raise ValueError("host_cubes must be contiguous")
        synth = images is not None
        if synth and G > 1 and not self.stage_iterations:
            raise ValueError("re-synthesis from an interleaved host batch needs staged lines")
        if synth and not (not images.is_cuda and images.is_pinned()
                          and tuple(images.shape) == (self.batch, *self.shape.dims)
                          and images.dtype == torch.complex64 and images.is_contiguous()):
            raise ValueError("images must be a contiguous pinned complex64 host tensor "
                             "[batch, *dims]")
        if synth and G > 1:
            return self._run_staged_synth(host_cubes, images)
        bz = self.split_count()
        if bz == self.batch and not synth:
            # all gathered in place: one launch and the result copy, in stream order,
            # replayed from a CUDA graph once captured for this host buffer
            g = self._graph_for(host_cubes) if self.graphs else None
            if g is not None:
                g.replay()
            else:
                self._launch_in_place(host_cubes)
            torch.cuda.current_stream(self.device).synchronize()
            if self.mode == "auto":
                self.last_mean_samples = float(self.out["samples_used"].double().mean())
            return self.out
        self._ensure_buffers(synth)
        if bz == 0 and self.chunk >= self.batch and not synth:
            # one chunk, nothing to overlap: copy, recover, copy back in stream order
            buf = self._bufs[0][:self.batch]
            buf.copy_(host_cubes, non_blocking=True)
            r = self._runner(0, self.batch)
            r.run(buf)
            self._copy_out(r, 0, self.batch)
            torch.cuda.current_stream(self.device).synchronize()
            self.last_mean_samples = float(self.out["samples_used"].double().mean())
            return self.out
        s_h2d, s_run, s_d2h, s_zc = self._streams
        cur = torch.cuda.current_stream(self.device)
        for s in self._streams:
            s.wait_stream(cur)

        # zero-copy part: gathered in place from host memory (one launch)
        ev_zc = None
        if bz:
            with torch.cuda.stream(s_zc):
                rz = self._runner(0, bz)
                rz.run(host_cubes[:bz])
                self._copy_out(rz, 0, bz)
                ev_zc = torch.cuda.Event()
                ev_zc.record(s_zc)

        # bulk-copy part: double-buffered chunks, H2D || recovery || D2H
        ev_free = [None, None]
        k = 0
        b0 = bz
        while b0 < self.batch:
            n = min(self.chunk, self.batch - b0)
            i = k & 1
            buf = self._bufs[i][:n]
            with torch.cuda.stream(s_h2d):
                if ev_free[i] is not None:
                    s_h2d.wait_event(ev_free[i])
                buf.copy_(host_cubes[b0:b0 + n], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_h2d)
            with torch.cuda.stream(s_run):
                s_run.wait_event(ev_in)
                r = self._runner(b0, n)
                res = r.run(buf)
                self._copy_out(r, b0, n)
                ev_done = torch.cuda.Event()
                ev_done.record(s_run)
                if synth:
                    img = self._img_bufs[i][:n]
                    synthesize(res, out=img)
                    ev_img = torch.cuda.Event()
                    ev_img.record(s_run)
            if synth:
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_img)
                    images[b0:b0 + n].copy_(img, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(s_d2h)
                    ev_free[i] = ev
            else:
                ev_free[i] = ev_done
            b0 += n
            k += 1

        if synth and bz:
            # the zero-copy instances' images: synthesised chunk-wise, sent back
            s_run.wait_event(ev_zc)
            c0 = 0
            while c0 < bz:
                n = min(self.chunk, bz - c0)
                i = k & 1
                with torch.cuda.stream(s_run):
                    if ev_free[i] is not None:
                        s_run.wait_event(ev_free[i])
                    img = self._img_bufs[i][:n]
                    o = self._runners[(0, bz)].out
                    synthesize(o["freqs"][c0:c0 + n], o["amps"][c0:c0 + n],
                               o["count"][c0:c0 + n], shape=self.shape, out=img)
                    ev_img = torch.cuda.Event()
                    ev_img.record(s_run)
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_img)
                    images[c0:c0 + n].copy_(img, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(s_d2h)
                    ev_free[i] = ev
                c0 += n
                k += 1

        for s in self._streams:
            cur.wait_stream(s)
        cur.synchronize()
        self.last_mean_samples = float(self.out["samples_used"].double().mean())
        return self.out
