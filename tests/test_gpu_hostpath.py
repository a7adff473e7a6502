"""Pinned-host batches (hostpath.HostBatchRunner): every path an instance can
take -- gathered in place from host memory (zero copy), or copied through the
double-buffered device chunks -- gives bit-identical outputs to the
device-resident run, and config-5 images written back to the host equal the
device re-synthesis."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1711_11407_b200 as P  # noqa: E402
from paper_1711_11407_b200 import ops  # noqa: E402
from paper_1711_11407_b200 import workloads as W  # noqa: E402
from paper_1711_11407_b200.hostpath import HostBatchRunner  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

DEV = torch.device("cuda:0")


def _cubes(cfg_id, count):
    w = W.CONFIGS[cfg_id]
    spectra = W.make_spectra(w, count, 0)
    cubes = W.synthesize_batch_torch(w.dims, spectra, DEV, w.noise_var, noise_seed=w.seed)
    cfg = P.FpsSftConfig(seed=cfg_id, **P.PROFILES[w.profile])
    return w, cubes, cfg


@pytest.mark.parametrize("mode,frac", [("copy", None), ("zero_copy", None), ("split", 0.4),
                                       ("auto", None)])
@pytest.mark.parametrize("cfg_id,count,k_cap", [(2, 37, 128), (4, 5, 2048), (3, 9, 512)])
def test_host_paths_match_device(cfg_id, count, k_cap, mode, frac):
    w, cubes, cfg = _cubes(cfg_id, count)
    shape = P.CubeShape(w.dims)
    dev_run = P.BatchRunner(shape, cfg, count, k_cap=k_cap, device=DEV)
    dev_run.run(cubes)
    want = {k: v.cpu() for k, v in dev_run.out.items() if v is not None}
    host = torch.empty(cubes.shape, dtype=cubes.dtype, pin_memory=True)
    host.copy_(cubes)
    hr = HostBatchRunner(shape, cfg, count, k_cap=k_cap, device=DEV, mode=mode,
                         zero_copy_fraction=frac, chunk=4)  # several chunks per batch
    for _ in range(2):  # auto: the second run splits with the learnt sample count
        got = hr.run(host)
        for k in want:
            assert torch.equal(got[k], want[k]), k
    if mode == "zero_copy":
        assert hr.split_count() == count
    if mode == "copy":
        assert hr.split_count() == 0


def test_pinned_host_tensor_runs_in_place():
    w, cubes, cfg = _cubes(2, 16)
    shape = P.CubeShape(w.dims)
    r = P.BatchRunner(shape, cfg, 16, k_cap=128, device=DEV)
    r.run(cubes)
    want = r.out["amps"].clone()
    host = cubes.cpu().pin_memory()
    r.run(host)
    assert torch.equal(r.out["amps"], want)
    with pytest.raises(ValueError):
        r.run(cubes.cpu())  # pageable host memory is not device-accessible


def test_cfg5_images_to_pinned_host():
    w, cubes, cfg = _cubes(5, 6)
    shape = P.CubeShape(w.dims)
    r = P.BatchRunner(shape, cfg, 6, k_cap=1024, device=DEV)
    want = ops.synthesize(r.run(cubes)).cpu()
    host = torch.empty(cubes.shape, dtype=cubes.dtype, pin_memory=True)
    host.copy_(cubes)
    for mode, frac in (("copy", None), ("split", 0.5)):
        images = torch.zeros(cubes.shape, dtype=cubes.dtype, pin_memory=True)
        hr = HostBatchRunner(shape, cfg, 6, k_cap=1024, device=DEV, mode=mode,
                             zero_copy_fraction=frac, chunk=2)
        hr.run(host, images)
        assert torch.equal(images, want), mode


@pytest.mark.parametrize("G,B,chunk", [(8, 22, 8), (4, 6, 2), (32, 40, 32)])
def test_cfg5_images_from_staged_interleaved_host_batch(G, B, chunk):
    """Config 5 from an interleaved host batch: lines staged chunk by chunk,
    recovery, re-synthesis, images and reports back in pinned host memory --
    identical to the device run (partial last group and chunk included)."""
    w, cubes, cfg = _cubes(5, B)
    shape = P.CubeShape(w.dims)
    r = P.BatchRunner(shape, cfg, B, k_cap=1024, device=DEV, precision="fp32")
    res = r.run(cubes)
    want = ops.synthesize(res).cpu()
    il = P.interleave(cubes, G)
    host = torch.empty(il.shape, dtype=il.dtype, pin_memory=True)
    host.copy_(il)
    images = torch.zeros(cubes.shape, dtype=cubes.dtype, pin_memory=True)
    hr = HostBatchRunner(shape, cfg, B, k_cap=1024, device=DEV, group=G, chunk=chunk,
                         precision="fp32",
                         stage_iterations=int(r.out["iterations"].max()) - 3)
    for _ in range(2):
        out = hr.run(host, images)
        assert torch.equal(images, want)
        for k, v in out.items():
            if v is not None:
                assert torch.equal(v, r.out[k].cpu()), k
    with pytest.raises(ValueError):  # no staged lines: interleaved re-synthesis refused
        HostBatchRunner(shape, cfg, B, k_cap=1024, device=DEV, group=G).run(host, images)
    with pytest.raises(ValueError):  # the guarded team kernel has no staged read path
        HostBatchRunner(shape, cfg, B, k_cap=1024, device=DEV, group=G, chunk=chunk,
                        stage_iterations=5).run(host, images)


def test_tune_picks_a_measured_fraction():
    w, cubes, cfg = _cubes(2, 64)
    host = torch.empty(cubes.shape, dtype=cubes.dtype, pin_memory=True)
    host.copy_(cubes)
    hr = HostBatchRunner(P.CubeShape(w.dims), cfg, 64, k_cap=128, device=DEV, chunk=16)
    f = hr.tune(host, fractions=[0.0, 0.5, 1.0])
    assert f in (0.0, 0.5, 1.0) and hr.mode == "split" and hr.tuned["fraction"] == f


@pytest.mark.parametrize("cfg_id,count,k_cap,group", [(2, 37, 128, 8), (2, 16, 128, 16),
                                                      (3, 9, 512, 8), (4, 5, 2048, 4),
                                                      (5, 6, 1024, 8), (1, 1, 64, 8)])
def test_interleaved_layout_matches_batch_major(cfg_id, count, k_cap, group):
    """The interleaved batch layout [ceil(B/G), *dims, G] (fpssft_run_batch_grouped)
    gives bit-identical outputs, partial last group included."""
    w, cubes, cfg = _cubes(cfg_id, count)
    shape = P.CubeShape(w.dims)
    ref = P.BatchRunner(shape, cfg, count, k_cap=k_cap, device=DEV)
    ref.run(cubes)
    g = P.BatchRunner(shape, cfg, count, k_cap=k_cap, device=DEV, group=group)
    gi = P.interleave(cubes, group)
    assert gi.shape == ((count + group - 1) // group, *w.dims, group)
    g.run(gi)
    for k, v in ref.out.items():
        if v is not None:
            assert torch.equal(v, g.out[k]), k
    with pytest.raises(ValueError):
        g.run(cubes)  # batch-major tensor handed to a grouped runner


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_interleaved_layout_with_per_instance_schedules(prec):
    """Grouped layout with one schedule per instance (Monte Carlo style) and in
    float64: still bit-identical to the batch-major run."""
    import numpy as np

    w, cubes, cfg = _cubes(2, 20)
    shape = P.CubeShape(w.dims)
    t_max = P.default_max_iterations(shape)
    sch = np.stack([P.schedule_from_seed(shape, s, t_max) for s in range(3)])
    si = np.random.default_rng(4).integers(0, 3, 20)
    kw = dict(k_cap=128, device=DEV, precision=prec, schedule=sch, sched_index=si)
    ref = P.BatchRunner(shape, cfg, 20, **kw)
    ref.run(cubes)
    g = P.BatchRunner(shape, cfg, 20, group=8, **kw)
    g.run(P.interleave(cubes, 8))
    for k, v in ref.out.items():
        if v is not None:
            assert torch.equal(v, g.out[k]), k


def test_zero_copy_graph_replay_sees_new_host_data():
    """The captured graph (zero copy + result copy) replays on whatever the
    pinned host buffer holds now."""
    w, cubes, cfg = _cubes(2, 12)
    shape = P.CubeShape(w.dims)
    other = W.synthesize_batch_torch(w.dims, W.make_spectra(w, 12, 100), DEV, 0.0, noise_seed=3)
    ref = P.BatchRunner(shape, cfg, 12, k_cap=128, device=DEV)
    host = torch.empty(cubes.shape, dtype=cubes.dtype, pin_memory=True)
    hr = HostBatchRunner(shape, cfg, 12, k_cap=128, device=DEV, mode="zero_copy")
    for src in (cubes, other, cubes):
        host.copy_(src)
        got = {k: v.clone() for k, v in hr.run(host).items() if v is not None}
        ref.run(src)
        for k, v in ref.out.items():
            if v is not None:
                assert torch.equal(v.cpu(), got[k]), k
    assert hr._graphs and all(g is not None for g in hr._graphs.values())


@pytest.mark.parametrize("G", [8, 16])
def test_interleaved_host_batch_gathered_in_place(G):
    """An interleaved pinned host batch [B/8, *dims, 8] is recovered in place by
    the group kernel (one PCIe read per 64-byte segment for 8 instances), with
    outputs identical to the device run of the same batch."""
    import numpy as np

    import paper_1711_11407_b200 as P
    from paper_1711_11407_b200 import workloads as W
    from paper_1711_11407_b200.hostpath import HostBatchRunner

    w = W.CONFIGS[2]
    B = 64
    inst = [W.make_instance(w, r) for r in W.instance_rngs(w.seed, B)]
    cubes = torch.as_tensor(np.stack([c for _, _, c in inst])).cuda()
    cfg = P.FpsSftConfig(seed=2, **P.PROFILES["P32"])
    shape = P.CubeShape(w.dims)
    dev = P.BatchRunner(shape, cfg, B, k_cap=128)  # batch-major device run
    dev.run(cubes)
    il = P.interleave(cubes, G)
    host = torch.empty(il.shape, dtype=il.dtype, pin_memory=True)
    host.copy_(il)
    hr = HostBatchRunner(shape, cfg, B, k_cap=128, group=G)
    assert hr._runner(0, B).plan["instances_per_cta"] == G  # the G-wide group kernel
    out = hr.run(host)
    for k, v in out.items():
        if v is not None:
            assert torch.equal(v, dev.out[k].cpu()), k
    with pytest.raises(ValueError):
        hr.run(torch.empty((B, *w.dims), dtype=torch.complex64, pin_memory=True))


@pytest.mark.parametrize("G,T0,B,pipe", [(32, 3, 96, 1), (32, 1, 70, 1), (16, 2, 64, 1),
                                         (8, 50, 40, 1), (64, 3, 64, 1), (32, 4, 128, 2),
                                         (16, 5, 128, 4)])
def test_staged_lines_from_interleaved_host_batch(G, T0, B, pipe):
    """fpssft_run_batch_staged: the first T0 iterations' line samples staged
    through HBM by TMA bulk copies of whole 8 G-byte host segments, later
    iterations gathered in place -- outputs bit-identical to the batch-major
    device run (partial last group, T0 beyond the iteration cap, and chunks
    pipelined over two streams included)."""
    import numpy as np

    w = W.CONFIGS[2]
    inst = [W.make_instance(w, r) for r in W.instance_rngs(w.seed, B)]
    cubes = torch.as_tensor(np.stack([c for _, _, c in inst])).cuda()
    cfg = P.FpsSftConfig(seed=2, **P.PROFILES["P32"])
    shape = P.CubeShape(w.dims)
    dev = P.BatchRunner(shape, cfg, B, k_cap=128)
    dev.run(cubes)
    assert int(dev.out["iterations"].max()) > 1
    il = P.interleave(cubes, G)
    host = torch.empty(il.shape, dtype=il.dtype, pin_memory=True)
    host.copy_(il)
    hr = HostBatchRunner(shape, cfg, B, k_cap=128, group=G, stage_iterations=T0, pipeline=pipe)
    for _ in range(2):  # second run: the captured graph
        out = hr.run(host)
        for k, v in out.items():
            if v is not None:
                assert torch.equal(v, dev.out[k].cpu()), k
    # the same from a device-resident interleaved batch
    st = P.BatchRunner(shape, cfg, B, k_cap=128, group=G, stage_iterations=T0)
    st.run(il)
    for k, v in st.out.items():
        if v is not None:
            assert torch.equal(v, dev.out[k]), k


@pytest.mark.parametrize("cfg_id,B,G,T0,k_cap,dims", [(3, 20, 32, 400, 512, None),
                                                      (3, 9, 8, 30, 512, None),
                                                      (1, 6, 4, 2, 64, (32, 64)),
                                                      (4, 6, 4, 3, 2048, None),
                                                      (5, 10, 8, 60, 512, "fp32")])
def test_staged_lines_per_instance_kernels(cfg_id, B, G, T0, k_cap, dims):
    """Staged lines read by the per-instance kernels (guarded float32 on the
    noisy 64^3 shape, tens of iterations; the runtime-shape warp kernel on a
    generic power-of-two shape; the team kernels of configs 4 and 5):
    bit-identical to the batch-major device run."""
    import dataclasses

    w = W.CONFIGS[cfg_id]
    prec = "auto"
    if dims == "fp32":  # config 5's team kernel, plain float32 (its guarded form has no staged reads)
        dims, prec = None, "fp32"
    if dims is not None:
        w = dataclasses.replace(w, dims=dims, k=8)
    spectra = W.make_spectra(w, B, 0)
    cubes = W.synthesize_batch_torch(w.dims, spectra, DEV, w.noise_var, noise_seed=w.seed)
    cfg = P.FpsSftConfig(seed=cfg_id, **P.PROFILES[w.profile])
    shape = P.CubeShape(w.dims)
    dev = P.BatchRunner(shape, cfg, B, k_cap=k_cap, precision=prec)
    dev.run(cubes)
    assert dev.plan["mode"] == ("cta" if cfg_id in (4, 5) else "warp")
    il = P.interleave(cubes, G)
    host = torch.empty(il.shape, dtype=il.dtype, pin_memory=True)
    host.copy_(il)
    hr = HostBatchRunner(shape, cfg, B, k_cap=k_cap, group=G, stage_iterations=T0,
                         precision=prec)
    for _ in range(2):
        out = hr.run(host)
        for k, v in out.items():
            if v is not None:
                assert torch.equal(v, dev.out[k].cpu()), k


def test_staged_lines_argument_errors():
    w = W.CONFIGS[2]
    shape = P.CubeShape(w.dims)
    cfg = P.FpsSftConfig(seed=2, **P.PROFILES["P32"])
    with pytest.raises(ValueError):
        P.BatchRunner(shape, cfg, 8, k_cap=128, group=1, stage_iterations=3)
    with pytest.raises(ValueError):
        P.BatchRunner(shape, cfg, 8, k_cap=128, group=8, stage_iterations=3,
                      sched_index=[0] * 8)
    with pytest.raises(ValueError):  # the runtime-shape CTA kernel has no staged read path
        r = P.BatchRunner(P.CubeShape((12, 18)), cfg, 8, k_cap=64, group=8,
                          stage_iterations=3)
        r.run(torch.zeros((1, 12, 18, 8), dtype=torch.complex64, device=DEV))
    with pytest.raises(ValueError):  # float64
        r = P.BatchRunner(shape, cfg, 8, k_cap=128, group=8, stage_iterations=3,
                          precision="fp64")
        r.run(torch.zeros((1, 256, 256, 8), dtype=torch.complex64, device=DEV))
