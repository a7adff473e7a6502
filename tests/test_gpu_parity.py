"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (tests/golden, generated from the unmodified reference) and against
the CPU oracle (oracle/fps_oracle.py) on identical inputs and schedules.

Tolerances (north_star): recovered support bit-exact; amplitudes within
1e-4 relative (noiseless) / 1e-3 (noisy profile) in float32.  The float64
mode is held to 1e-9.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import fixtures as G  # noqa: E402
from oracle import fps_oracle as O  # noqa: E402

import paper_1711_11407_b200 as P  # noqa: E402
from paper_1711_11407_b200 import ops  # noqa: E402
from paper_1711_11407_b200 import workloads as W  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

RUNS = G.meta()["runs"]
OPS = G.meta()["ops"]
DEV = torch.device("cuda:0")


def _cfg(entry):
    return P.FpsSftConfig(**entry["cfg"], **G.PROFILES[entry["profile"]])


def _fp32_resolvable(exp) -> bool:
    """False when the reference recovered entries at the complex64 rounding
    level of the cube (|a| < 1e-5 sum|a|): float32 arithmetic cannot resolve
    those, float64 can."""
    a = np.abs(exp["amps"])
    return a.size == 0 or a.min() > 1e-5 * a.sum()


def _amp_tol(entry):
    return 1e-3 if entry["profile"] == "PN" else 1e-4


# ------------------------------------------------------------- per-step ops
@pytest.mark.parametrize("prec,tol", [("fp32", 2e-6), ("fp64", 1e-13)])
@pytest.mark.parametrize("entry", [e for e in OPS["line"]
                                   if f"{e['key']}/cube" in G.npz("ops.npz")],
                         ids=lambda e: e["key"])
def test_line_spectra_vs_reference(entry, prec, tol):
    ops_ = G.npz("ops.npz")
    cube = torch.as_tensor(ops_[f"{entry['key']}/cube"])[None].to(DEV)
    got = ops.line_spectra(cube, entry["alpha"], entry["tau"], precision=prec)[0].cpu().numpy()
    want = ops_[f"{entry['key']}/spectra"]
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= tol * scale * np.sqrt(want.shape[1])


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 6, 7, 8, 11, 12, 13, 16, 30, 36, 48, 60, 64, 256,
                               512, 2048, 4608, 243, 343, 1000])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_dft_forward_vs_numpy(L, prec, rng):
    v = rng.standard_normal((3, L)) + 1j * rng.standard_normal((3, L))
    x = torch.as_tensor(v).to(DEV)
    try:
        got = ops.dft_forward(x, precision=prec).cpu().numpy()
    except ValueError as e:  # UnsupportedError for lengths beyond one CTA
        pytest.skip(str(e))
    want = np.fft.fft(v, axis=-1) / L
    tol = (3e-7 if prec == "fp32" else 1e-15) * max(1.0, np.log2(L)) * np.abs(v).max()
    assert np.abs(got - want).max() <= tol


def test_dft_goldens():  # pkg/tests/test_transform.py:13-19
    x = torch.tensor([[1, 1, 1, 1]], dtype=torch.complex128, device=DEV)
    assert np.allclose(ops.dft_forward(x, precision="fp64").cpu().numpy(), [[1, 0, 0, 0]],
                       atol=1e-15)
    tone = torch.as_tensor(np.exp(2j * np.pi * np.arange(4) / 4))[None].to(DEV)
    assert np.allclose(ops.dft_forward(tone, precision="fp64").cpu().numpy(), [[0, 1, 0, 0]],
                       atol=1e-15)


@pytest.mark.parametrize("entry", OPS["decode"], ids=lambda e: e["key"])
@pytest.mark.parametrize("pname,prec", [("P64", "fp64"), ("P32", "fp64"), ("P32", "fp32")])
def test_decode_spectra_vs_reference(entry, pname, prec):
    ops_ = G.npz("ops.npz")
    k = entry["key"]
    shape = P.CubeShape(entry["dims"])
    kw = {a: b for a, b in G.PROFILES[pname].items() if a != "residual_stop"}
    acc, nc = ops.decode_spectra(ops_[f"{k}/spectra"], entry["tau"], shape, precision=prec, **kw)
    assert nc == int(ops_[f"{k}/{pname}/ncand"])
    assert [b for b, _ in acc] == list(ops_[f"{k}/{pname}/bins"])
    assert [s.freq for _, s in acc] == [tuple(f) for f in ops_[f"{k}/{pname}/freqs"]]
    got = np.asarray([s.amp for _, s in acc])
    want = ops_[f"{k}/{pname}/amps"]
    tol = 1e-12 if prec == "fp64" else 1e-5
    assert np.all(np.abs(got - want) <= tol * np.abs(want))


@pytest.mark.parametrize("entry", OPS["project"], ids=lambda e: e["key"])
@pytest.mark.parametrize("prec,tol", [("fp64", 1e-13), ("fp32", 1e-6)])
def test_project_onto_bins_vs_reference(entry, prec, tol):
    ops_ = G.npz("ops.npz")
    k = entry["key"]
    shape = P.CubeShape(entry["dims"])
    got = ops.project_onto_bins(ops_[f"{k}/freqs"], ops_[f"{k}/amps"], entry["alpha"],
                                entry["tau"], shape, precision=prec).cpu().numpy()
    want = ops_[f"{k}/out"]
    assert np.abs(got - want).max() <= tol * np.abs(ops_[f"{k}/amps"]).sum()


def test_project_empty_set_is_zero():  # pkg/tests/test_decoder.py:146-150
    out = ops.project_onto_bins(np.zeros((0, 2)), np.zeros(0), (1, 1), (0, 0), P.CubeShape((8, 8)))
    assert torch.count_nonzero(out).item() == 0


# -------------------------------------------------------- the fused loop
def _check_report(rep, exp, amp_rtol, log=True, amp_atol_rel=0.0):
    assert rep.terminated_by == exp["terminated_by"]
    assert rep.iterations_run == exp["iterations_run"]
    assert rep.samples_used == exp["samples_used"]
    got_f = rep.recovered.freq_array.reshape(-1, exp["freqs"].shape[1])
    np.testing.assert_array_equal(got_f, exp["freqs"])
    got_a = rep.recovered.amp_array
    atol = amp_atol_rel * (np.abs(exp["amps"]).max() if len(exp["amps"]) else 0.0)
    assert np.all(np.abs(got_a - exp["amps"]) <= amp_rtol * np.abs(exp["amps"]) + atol)
    if log:
        assert [s.alpha for s in rep.iteration_log] == [tuple(a) for a in exp["log_alpha"]]
        assert [s.tau for s in rep.iteration_log] == [tuple(t) for t in exp["log_tau"]]
        got = [(s.candidates, s.accepted, s.rejected) for s in rep.iteration_log]
        want = [tuple(int(v) for v in c) for c in exp["log_counts"]]
        assert got == want


@pytest.mark.parametrize("mode", ["auto", "cta"])
@pytest.mark.parametrize("entry", RUNS, ids=lambda e: e["name"])
def test_fps_sft_fp64_matches_reference(entry, mode):
    cube = G.run_cube(entry)
    shape = P.CubeShape(cube.shape)
    if P.max_k_cap(shape, "fp64", mode) < max(1, len(G.run_expected(entry)["amps"])):
        pytest.skip("recovered set does not fit one CTA in float64")
    rep = P.fps_sft(P.make_dense_source(cube, shape), _cfg(entry), precision="fp64", mode=mode)
    # float64 amplitudes carry ~1e-16 * max|a| absolute rounding, which is
    # large relative to complex64-rounding-level entries
    _check_report(rep, G.run_expected(entry), 1e-9, amp_atol_rel=1e-13)


@pytest.mark.parametrize("mode", ["auto", "cta"])
@pytest.mark.parametrize("entry", [e for e in RUNS if e["profile"] != "P64"],
                         ids=lambda e: e["name"])
def test_fps_sft_fp32_matches_reference(entry, mode):
    exp = G.run_expected(entry)
    if not _fp32_resolvable(exp):
        pytest.skip("reference recovered complex64-rounding-level entries")
    cube = G.run_cube(entry)
    shape = P.CubeShape(cube.shape)
    # "auto": plain float32 for the noiseless profiles, guarded float32 (the
    # float64 reference's decisions, csrc/fpssft_guard.cuh) for the noisy one
    rep = P.fps_sft(P.make_dense_source(cube, shape), _cfg(entry), precision="auto", mode=mode)
    _check_report(rep, exp, _amp_tol(entry))


# ----------------------------------------------------- batches vs oracle
def _batch(w: W.Workload, count: int):
    inst = [W.make_instance(w, r) for r in W.instance_rngs(w.seed, count)]
    cubes = torch.as_tensor(np.stack([c for _, _, c in inst])).to(DEV)
    return inst, cubes


@pytest.mark.parametrize("cfg_id,count,prec,mode", [
    (2, 48, "fp32", "warp"), (2, 16, "fp32", "cta"), (2, 16, "fp64", "warp"), (1, 1, "fp32", "auto"),
    (4, 32, "fp32", "auto"), (3, 32, "auto", "warp"), (3, 32, "auto", "cta"),
    (5, 32, "auto", "auto"), (3, 2, "fp64", "auto"), (5, 2, "fp64", "auto")])
def test_config_batches_match_oracle(cfg_id, count, prec, mode):
    """Every instance identical to the oracle: support, iterations,
    termination and the per-iteration (candidates, accepted, rejected) log;
    amplitudes within the north-star tolerance (1e-4 noiseless, 1e-3 noisy;
    the noisy configs run guarded float32 under "auto")."""
    w = W.CONFIGS[cfg_id]
    inst, cubes = _batch(w, count)
    prof = O.Profile(**G.PROFILES[w.profile])
    cfg = P.FpsSftConfig(seed=cfg_id, **G.PROFILES[w.profile])
    shape = P.CubeShape(w.dims)
    k_cap = 2048 if cfg_id == 4 else (1024 if cfg_id in (3, 5) else 256)
    if prec == "fp64":
        k_cap = min(k_cap, P.max_k_cap(shape, "fp64"))
    res = P.fps_sft_batch(cubes, cfg, k_cap=k_cap, precision=prec, iter_stats=True, mode=mode)
    tol = 1e-9 if prec == "fp64" else (1e-3 if w.noise_var else 1e-4)
    for b, (f, a, cube) in enumerate(inst):
        ref = O.recover(cube, w.dims, prof, seed=cfg_id)
        rep = res.report(b)
        exp = dict(freqs=ref.freqs, amps=ref.amps, terminated_by=ref.terminated_by,
                   iterations_run=ref.iterations_run, samples_used=ref.samples_used,
                   log_alpha=[x[0] for x in ref.log], log_tau=[x[1] for x in ref.log],
                   log_counts=[x[2:] for x in ref.log])
        _check_report(rep, exp, tol, amp_atol_rel=1e-13 if prec == "fp64" else 0.0)


def test_cfg2_full_batch_recovers_truth():
    """BASELINE config 2 at full size (4096 instances): every instance's
    recovered spectrum equals its generating spectrum (size-independent
    property; the oracle checks a subset above)."""
    w = W.CONFIGS[2]
    spectra = W.make_spectra(w)
    cubes = W.synthesize_batch_torch(w.dims, spectra, DEV)
    cfg = P.FpsSftConfig(seed=2, **G.PROFILES["P32"])
    res = P.fps_sft_batch(cubes, cfg, k_cap=256)
    count = res.count.cpu().numpy()
    term = res.terminated_by.cpu().numpy()
    assert (term == 0).all()
    assert (count == w.k).all()
    freqs = res.freqs.cpu().numpy()
    amps = res.amps.cpu().numpy()
    for b in range(0, w.batch, 97):
        f, a = spectra[b]
        order = np.lexsort(f.T[::-1])
        np.testing.assert_array_equal(freqs[b, :w.k], f[order])
        assert np.all(np.abs(amps[b, :w.k] - a[order]) <= 1e-4 * np.abs(a[order]))


# ------------------------------------------------------------ properties
@pytest.mark.parametrize("mode", ["warp", "cta"])
def test_determinism_bitwise(mode):
    w = W.CONFIGS[5]
    _, cubes = _batch(w, 3)
    cfg = P.FpsSftConfig(seed=5, **G.PROFILES["PN"])
    prec = "fp32" if mode == "warp" else "auto"  # cta: the guarded team kernel
    r1 = P.fps_sft_batch(cubes, cfg, k_cap=1024, mode=mode, precision=prec)
    a1 = (r1.freqs.clone(), r1.amps.clone(), r1.count.clone())
    r2 = P.fps_sft_batch(cubes, cfg, k_cap=1024, mode=mode, precision=prec)
    assert torch.equal(a1[0], r2.freqs) and torch.equal(a1[1], r2.amps)
    assert torch.equal(a1[2], r2.count)


def test_amplitude_scale_equivariance():  # pkg/tests/test_driver.py:119-128
    f, a = W.reference_generate((16, 12), 8, 4)
    shape = P.CubeShape((16, 12))
    cfg = P.FpsSftConfig(max_iterations=15, seed=123, **G.PROFILES["P32"])
    base = P.fps_sft(P.make_dense_source(W.synthesize_np((16, 12), f, a), shape), cfg)
    other = P.fps_sft(P.make_dense_source(W.synthesize_np((16, 12), f, a * (3 - 4j)), shape), cfg)
    assert set(base.recovered.entries) == set(other.recovered.entries)
    for k, v in base.recovered.entries.items():
        assert abs(other.recovered.entries[k] - v * (3 - 4j)) <= 1e-4 * abs(v * (3 - 4j))


def test_sample_accounting_and_certificate():  # test_driver.py:78-84, 106-117
    f, a = W.reference_generate((16, 16), 12, 8)
    shape = P.CubeShape((16, 16))
    cube = W.synthesize_np((16, 16), f, a)
    rep = P.fps_sft(P.make_dense_source(cube, shape),
                    P.FpsSftConfig(max_iterations=20, seed=9, **G.PROFILES["P32"]))
    assert rep.samples_used == rep.iterations_run * 3 * 16
    assert rep.terminated_by == "residual_clean"
    rebuilt = W.synthesize_np((16, 16), rep.recovered.freq_array, rep.recovered.amp_array)
    assert np.abs(rebuilt - cube).max() <= 1e-5 * np.abs(cube).max()


@pytest.mark.parametrize("mode", ["warp", "cta"])
def test_zero_cube_terminates_clean_with_nothing(mode):
    cubes = torch.zeros((2, 16, 16), dtype=torch.complex64, device=DEV)
    res = P.fps_sft_batch(cubes, P.FpsSftConfig(max_iterations=5, seed=1), k_cap=64, mode=mode)
    assert res.count.tolist() == [0, 0]
    assert res.terminated_by.tolist() == [0, 0]
    assert res.iterations.tolist() == [1, 1]


def test_empty_batch_is_a_noop():
    cubes = torch.zeros((0, 16, 16), dtype=torch.complex64, device=DEV)
    res = P.fps_sft_batch(cubes, P.FpsSftConfig(max_iterations=5), k_cap=64)
    assert res.count.numel() == 0


@pytest.mark.parametrize("mode", ["warp", "cta"])
def test_k_cap_overflow_is_reported(mode):
    w = W.CONFIGS[2]
    _, cubes = _batch(w, 2)
    res = P.fps_sft_batch(cubes, P.FpsSftConfig(seed=2, **G.PROFILES["P32"]), k_cap=32, mode=mode)
    assert res.terminated_by.tolist() == [3, 3]
    assert (res.count.cpu().numpy() <= 32).all()


@pytest.mark.parametrize("mode", ["warp", "cta"])
def test_per_instance_schedules_and_strided_input(mode):
    w = W.CONFIGS[2]
    inst, cubes = _batch(w, 4)
    shape = P.CubeShape(w.dims)
    cfg = P.FpsSftConfig(max_iterations=12, **G.PROFILES["P32"])
    sched = np.stack([P.schedule_from_seed(shape, s, 12) for s in (11, 12)])
    idx = np.asarray([1, 0, 1, 0])
    # a transposed (non-contiguous) view of the same data: recover on x^T,
    # whose spectrum is the transposed spectrum
    cubes_t = cubes.transpose(1, 2)
    res = P.fps_sft_batch(cubes_t, cfg, schedule=sched, sched_index=idx, k_cap=256, mode=mode)
    prof = O.Profile(**G.PROFILES["P32"], max_iterations=12)
    for b, (_, _, cube) in enumerate(inst):
        ref = O.recover(np.ascontiguousarray(cube.T), w.dims, prof,
                        schedule=sched[idx[b]].astype(np.int64))
        rep = res.report(b)
        np.testing.assert_array_equal(rep.recovered.freq_array.reshape(-1, 2), ref.freqs)
        assert rep.iterations_run == ref.iterations_run


def test_invalid_schedule_rejected():
    cubes = torch.zeros((1, 8, 8), dtype=torch.complex64, device=DEV)
    bad = np.zeros((3, 2, 2), np.int32)
    bad[0, 1] = (8, 0)
    with pytest.raises(ValueError):
        P.fps_sft_batch(cubes, P.FpsSftConfig(max_iterations=3), schedule=bad, k_cap=64)


def test_lazy_source_is_materialised():
    class Lazy:
        def __init__(self, f, a, dims):
            self.f, self.a, self.dims = f, a, dims

        def shape(self):
            return P.CubeShape(self.dims)

        def sample_many(self, idx):
            ph = (idx[:, None, :] * self.f[None] / np.asarray(self.dims)).sum(-1)
            return (np.exp(2j * np.pi * ph) * self.a).sum(-1)

    f, a = W.reference_generate((12, 12), 10, 31)
    rep = P.fps_sft(Lazy(f, a, (12, 12)),
                    P.FpsSftConfig(max_iterations=12, seed=5, **G.PROFILES["P32"]))
    order = np.lexsort(f.T[::-1])
    np.testing.assert_array_equal(rep.recovered.freq_array, f[order])


# ------------------------------------------------------------ re-synthesis
@pytest.mark.parametrize("dims,k", [((512, 512), 500), ((12, 18), 9), ((4, 6, 5), 7), ((32,), 5),
                                    ((64, 64, 64), 200), ((256, 256), 100), ((10, 15), 150),
                                    # synth512_kernel (512-point rows) with other row counts /
                                    # line lengths and crowded columns (its quarter-image chunks,
                                    # column ranking and entry sort)
                                    ((128, 512), 300), ((48, 512), 300), ((1024, 512), 700),
                                    ((64, 512), 2000)])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_synthesize_matches_dense_evaluation(dims, k, prec, rng):
    """a15: dense re-synthesis vs the float64 evaluation of the same spectra
    (SyntheticSource.sample_many semantics, core.py:176-217)."""
    B = 3
    k = min(k, int(np.prod(dims)))
    kc = 1 << (k - 1).bit_length()
    fr = np.zeros((B, kc, len(dims)), np.int32)
    am = np.zeros((B, kc), np.complex128)
    cnt = np.zeros(B, np.int32)
    want = []
    for b in range(B):
        n = k - b  # ragged counts
        flat = rng.choice(int(np.prod(dims)), size=n, replace=False)
        f = np.stack(np.unravel_index(flat, dims), axis=-1)
        a = rng.rayleigh(1.0, n) * np.exp(2j * np.pi * rng.random(n))
        fr[b, :n], am[b, :n], cnt[b] = f, a, n
        want.append(W.synthesize_np(dims, f, a))
    got = ops.synthesize(torch.as_tensor(fr).to(DEV), torch.as_tensor(am).to(DEV),
                         torch.as_tensor(cnt).to(DEV), shape=P.CubeShape(dims),
                         precision=prec).cpu().numpy()
    for b in range(B):
        scale = np.abs(am[b]).sum()
        # the grid is written as complex64 in both modes (rounding ~6e-8 |x|)
        tol = (2e-6 if prec == "fp32" else 1.2e-7) * scale
        assert np.abs(got[b] - want[b]).max() <= tol


def test_cfg5_recover_then_resynthesise():
    """Config 5 end to end on a few frames: recover, re-synthesise, compare
    with the oracle's re-synthesis of its own recovered spectrum."""
    w = W.CONFIGS[5]
    inst, cubes = _batch(w, 3)
    cfg = P.FpsSftConfig(seed=5, **G.PROFILES["PN"])
    res = P.fps_sft_batch(cubes, cfg, k_cap=1024, precision="fp64")
    img = ops.synthesize(res).cpu().numpy()
    prof = O.Profile(**G.PROFILES["PN"])
    for b, (_, _, cube) in enumerate(inst):
        ref = O.recover(cube, w.dims, prof, seed=5)
        want = O.synthesize(w.dims, ref.freqs, ref.amps)
        assert np.abs(img[b] - want).max() <= 2e-6 * np.abs(ref.amps).sum()


# ------------------------------------------------------- Monte Carlo sweeps
def test_sweep_small_shapes_recover():  # cf. pkg/tests/test_driver.py:57-69
    from paper_1711_11407_b200 import sweep as S
    row, per = S.run_cell(P.CubeShape((16, 12)), 16, "uniform", 100, 7,
                          P.FpsSftConfig(max_iterations=30, stall_limit=10, **G.PROFILES["P32"]))
    assert row.p_success >= 0.99
    np.testing.assert_array_equal(per["samples_used"], per["iterations"] * 3 * 48)


@pytest.mark.slow
def test_sweep_paper_anchors_c5_c6():
    """pkg/tests/test_acceptance.py:182-219 on the GPU: p(K=5 N0) >= 0.90 and
    p(K=6 N0) <= 0.05 on 256x256 with T_max=85; mean samples for K=N0 in [4%, 8%]."""
    from paper_1711_11407_b200 import sweep as S
    cfg = P.FpsSftConfig(max_iterations=85, stall_limit=12, **G.PROFILES["P32"])
    rows = S.run_sweep([(256, 256)], [1280, 1536], ["uniform"], 100, 505, cfg)
    p = {r.k: r.p_success for r in rows}
    assert p[1280] >= 0.90 and p[1536] <= 0.05, p
    row = S.run_sweep([(256, 256)], [256], ["uniform"], 100, 606, cfg)[0]
    assert row.p_success >= 0.99
    assert 0.04 <= row.mean_percent_samples <= 0.08, row


def test_lazy_spectrum_source_synthesised_on_device():
    """A lazy mixture exposing ``spectrum`` (like the reference's
    SyntheticSource) is materialised with fpssft_synthesize and recovered."""
    f, a = W.reference_generate((16, 12), 16, 3)

    class Spec:
        freq_array, amp_array = f, a

    class Lazy:
        spectrum = Spec()

        def shape(self):
            return P.CubeShape((16, 12))

    cfg = P.FpsSftConfig(max_iterations=30, stall_limit=10, seed=1003, **G.PROFILES["P32"])
    rep = P.fps_sft(Lazy(), cfg)
    order = np.lexsort(f.T[::-1])
    np.testing.assert_array_equal(rep.recovered.freq_array, f[order])
    assert np.all(np.abs(rep.recovered.amp_array - a[order]) <= 1e-4 * np.abs(a[order]))


# ------------------------------------------------------------- baseline_sft
BASE = G.meta().get("baseline", [])


@pytest.mark.parametrize("entry", BASE, ids=lambda e: e["name"])
def test_baseline_sft_matches_reference(entry):  # driver.py:219-314
    a = G.npz("runs.npz")
    n = entry["name"]
    cube = a[f"{n}/cube"] if f"{n}/cube" in a else G.cube_from_recipe(entry["recipe"])
    assert G.sha(cube) == entry["sha256"]
    shape = P.CubeShape(cube.shape)
    cfg = P.FpsSftConfig(**entry["cfg"], **G.PROFILES[entry["profile"]])
    rep = P.baseline_sft(P.make_dense_source(cube, shape), cfg)
    assert rep.terminated_by == entry["terminated_by"]
    assert rep.iterations_run == entry["iterations_run"]
    assert rep.samples_used == entry["samples_used"]
    np.testing.assert_array_equal(rep.recovered.freq_array.reshape(-1, 2), a[f"{n}/freqs"])
    want = a[f"{n}/amps"]
    assert np.all(np.abs(rep.recovered.amp_array - want) <= 1e-4 * np.abs(want))
    assert [(s.candidates, s.accepted, s.rejected) for s in rep.iteration_log] == \
        [tuple(int(v) for v in c) for c in a[f"{n}/log_counts"]]


def test_baseline_sft_rejects_bad_shapes():  # pkg/tests/test_driver.py:170-183
    for dims in ((8, 12), (6, 6), (4, 4, 4)):
        cube = np.zeros(dims, np.complex64)
        with pytest.raises(ValueError):
            P.baseline_sft(P.make_dense_source(cube, P.CubeShape(dims)))


@pytest.mark.parametrize("dims,k", [((1, 8), 3), ((8, 1), 3), ((11, 13), 6), ((3, 4, 5, 6), 9),
                                    ((7,), 2), ((2, 2), 2), ((5, 5, 5), 8), ((9, 12), 10)])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_unusual_shapes_match_oracle(dims, k, prec, rng):
    """Degenerate (N_k = 1), prime, 4-D and tiny shapes through the generic
    kernels, against the oracle on the same cube and schedule."""
    f, a = W.reference_generate(dims, k, 17)
    cube = W.synthesize_np(dims, f, a).astype(np.complex64)
    prof = dict(G.PROFILES["P32"])
    cfg = P.FpsSftConfig(max_iterations=12, stall_limit=6, seed=5, **prof)
    rep = P.fps_sft(P.make_dense_source(cube, P.CubeShape(dims)), cfg, precision=prec)
    ref = O.recover(cube, dims, O.Profile(max_iterations=12, stall_limit=6, **prof), seed=5)
    if prec == "fp32" and len(ref.amps) and np.abs(ref.amps).min() < 1e-5 * np.abs(ref.amps).sum():
        pytest.skip("reference recovered complex64-rounding-level entries")
    exp = dict(freqs=ref.freqs, amps=ref.amps, terminated_by=ref.terminated_by,
               iterations_run=ref.iterations_run, samples_used=ref.samples_used,
               log_alpha=[x[0] for x in ref.log], log_tau=[x[1] for x in ref.log],
               log_counts=[x[2:] for x in ref.log])
    _check_report(rep, exp, 1e-9 if prec == "fp64" else 1e-4,
                  amp_atol_rel=1e-13 if prec == "fp64" else 0.0)


@pytest.mark.parametrize("dims,k_cap", [((1024, 2048), 64), ((512, 512), 16), ((256, 256), 8),
                                        ((64, 64, 64), 16)])
def test_tiny_k_cap_overflows_cleanly(dims, k_cap):
    """Every kernel family with a recovered-set capacity far below K: the
    overflow is reported per instance and nothing faults."""
    f, a = W.reference_generate(dims, 4 * k_cap, 3)
    cube = torch.as_tensor(W.synthesize_np(dims, f, a).astype(np.complex64))[None].to(DEV)
    cfg = P.FpsSftConfig(max_iterations=6, **G.PROFILES["P32"])
    for mode in ("auto", "cta"):
        res = P.fps_sft_batch(cube, cfg, k_cap=k_cap, mode=mode)
        torch.cuda.synchronize()
        assert res.terminated_by.item() == 3
        assert 0 <= res.count.item() <= k_cap


@pytest.mark.parametrize("dims,k,k_cap,mode", [((256, 256), 100, 128, "auto"),
                                               ((256, 256), 100, 128, "cta"),
                                               ((64, 64, 64), 200, 512, "auto"),
                                               ((512, 512), 500, 1024, "cta"),
                                               ((1024, 2048), 1000, 2048, "cta")])
def test_misaligned_and_padded_rows_match_contiguous(dims, k, k_cap, mode):
    """The staged 16-byte gathers read the aligned chunk around each sample:
    a cube whose base is 8 bytes off a 16-byte boundary, with an odd row
    pitch (so the half-select flips from row to row) and rows that end at
    the chunk edge, must give bit-identical results to the contiguous copy."""
    f, a = W.reference_generate(dims, k, 23)
    cube = torch.as_tensor(W.synthesize_np(dims, f, a).astype(np.complex64)).to(DEV)
    cubes = torch.stack([cube, cube.roll(1, -1)])
    padded = torch.zeros((2, *dims[:-1], dims[-1] + 1), dtype=torch.complex64, device=DEV)
    padded[..., 1:] = cubes
    view = padded[..., 1:]
    assert view.data_ptr() % 16 == 8 and view.stride(-2) % 2 == 1
    cfg = P.FpsSftConfig(max_iterations=8, **G.PROFILES["P32"])
    r0 = P.fps_sft_batch(cubes, cfg, k_cap=k_cap, mode=mode)
    r1 = P.fps_sft_batch(view, cfg, k_cap=k_cap, mode=mode)
    for name in ("count", "iterations", "terminated_by", "freqs", "amps"):
        assert torch.equal(getattr(r0, name), getattr(r1, name)), name
    assert int(r0.count[0]) > 0


def test_spectrum_files_round_trip_through_the_device(tmp_path):
    """fps_sft_batch -> save_batch (reference text format) -> load_batch ->
    fpssft_synthesize gives the same grids as synthesising the device result."""
    from paper_1711_11407_b200 import spectrum_io as S

    w = W.CONFIGS[2]
    _, cubes = _batch(w, 3)
    res = P.fps_sft_batch(cubes, P.FpsSftConfig(**G.PROFILES["P32"]), k_cap=128)
    paths = S.save_batch(res, tmp_path)
    f, a, c, shape = S.load_batch(paths, k_cap=128)
    assert shape == res.shape
    assert torch.equal(c, res.count)
    for b in range(3):
        n = int(c[b])
        assert torch.equal(f[b, :n], res.freqs[b, :n]) and torch.equal(a[b, :n], res.amps[b, :n])
    assert torch.equal(ops.synthesize(f, a, c, shape=shape), ops.synthesize(res))
