"""CPU-only checks of the host side: schedule replay against the reference's
draws, slope validity, the C ABI library (loads, exports every symbol the
header declares, validates arguments before touching a GPU), and the
reference-mirroring types."""

import ctypes
import os
import re

import numpy as np
import pytest

import fixtures as G
import paper_1711_11407_b200 as P
from paper_1711_11407_b200 import _native as N
from paper_1711_11407_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = G.meta()["ops"]


@pytest.mark.parametrize("entry", OPS["schedule"], ids=lambda e: e["key"])
def test_schedule_replays_reference_draws(entry):
    got = P.schedule_from_seed(P.CubeShape(entry["dims"]), entry["seed"], entry["T"])
    np.testing.assert_array_equal(got, G.npz("ops.npz")[entry["key"]])


def test_schedule_matches_reference_iteration_logs():
    for entry in G.meta()["runs"]:
        exp = G.run_expected(entry)
        T = len(exp["log_alpha"])
        sch = P.schedule_from_seed(P.CubeShape(entry["recipe"]["dims"]),
                                   entry["cfg"].get("seed", 0), T)
        np.testing.assert_array_equal(sch[:, 0], exp["log_alpha"])
        np.testing.assert_array_equal(sch[:, 1], exp["log_tau"])


@pytest.mark.parametrize("alpha,ok", [((1, 1), True), ((1, 5), True), ((3, 1), True),
                                      ((2, 1), False), ((1, 3), False), ((2, 3), False)])
def test_slope_validity_4x6(alpha, ok):  # pkg/tests/test_numtheory.py:46-54
    assert P.is_valid_slope(alpha, P.CubeShape((4, 6))) == ok


def test_slope_validation_errors():  # numtheory.py:64-69
    with pytest.raises(ValueError):
        P.is_valid_slope((1,), P.CubeShape((4, 6)))
    with pytest.raises(ValueError):
        P.is_valid_slope((4, 1), P.CubeShape((4, 6)))


def test_bins_of_frequencies_goldens():
    for e in OPS["project"]:
        got = P.bins_of_frequencies(G.npz("ops.npz")[f"{e['key']}/freqs"], e["alpha"],
                                    P.CubeShape(e["dims"]))
        np.testing.assert_array_equal(got, G.npz("ops.npz")[f"{e['key']}/bins"])


def test_config_validation_mirrors_reference():  # pkg/tests/test_driver.py:27-34
    with pytest.raises(ValueError):
        P.FpsSftConfig(max_iterations=0)
    with pytest.raises(ValueError):
        P.FpsSftConfig(stall_limit=0)
    with pytest.raises(ValueError):
        P.FpsSftConfig(mag_tol=0)
    assert P.default_max_iterations(P.CubeShape((256, 256))) == 85
    assert P.default_max_iterations(P.CubeShape((2, 2))) == 1


def test_shape_and_spectrum_types():  # pkg/tests/test_core.py
    s = P.CubeShape((4, 6))
    assert (s.n_total, s.line_len, s.cofactors) == (24, 12, (3, 2))
    with pytest.raises(ValueError):
        P.CubeShape(())
    with pytest.raises(ValueError):
        P.CubeShape((0, 3))
    with pytest.raises(ValueError):
        P.SparseSpectrum(s, {(0, 0): 0})
    sp = P.SparseSpectrum(s, {(3, 1): 1j, (0, 5): 2.0})
    assert list(sp.entries) == [(0, 5), (3, 1)]
    with pytest.raises(ValueError):
        P.make_dense_source(np.zeros((3, 3), np.complex64), s)


def test_reference_generator_draw_order():
    f, a = W.reference_generate((16, 12), 16, 0)
    assert f.shape == (16, 2) and np.allclose(np.abs(a), 1.0)


# ------------------------------------------------------------- the C ABI
def _header_symbols():
    src = open(os.path.join(ROOT, "include", "fpssft.h")).read()
    return sorted(set(re.findall(r"\b(fpssft_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = N.lib()
    syms = _header_symbols()
    assert len(syms) >= 10
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(N.EXPORTS)
    assert lib.fpssft_abi_version() == 1


def _byref(x):
    return ctypes.byref(x)


def test_abi_rejects_bad_arguments_without_a_gpu():
    lib = N.lib()
    sh = N.make_shape((16, 16))
    p = P.driver._params(P.FpsSftConfig(), 0, 64, N.F32)  # t_max 0
    with pytest.raises(ValueError):
        N.check(lib.fpssft_run_batch(None, 0, 0, _byref(sh), _byref(p), None, None, 1, None, None))
    p = P.driver._params(P.FpsSftConfig(), 4, 60, N.F32)  # k_cap not a power of two
    with pytest.raises(ValueError):
        N.check(lib.fpssft_run_batch(None, 0, 0, _byref(sh), _byref(p), None, None, 1, None, None))
    p = P.driver._params(P.FpsSftConfig(), 4, 64, N.F32)
    big = N.make_shape((65536, 65536))
    with pytest.raises(OverflowError):
        N.check(lib.fpssft_run_batch(None, 0, 0, _byref(big), _byref(p), None, None, 1, None,
                                     None))
    bad = N.Shape()
    bad.ndim = 5
    with pytest.raises(ValueError):
        N.check(lib.fpssft_run_batch(None, 0, 0, _byref(bad), _byref(p), None, None, 1, None,
                                     None))
    with pytest.raises(ValueError):
        N.check(lib.fpssft_dft_forward(None, 1, 0, None, 0, None))


@pytest.mark.parametrize("dims,prec,threads", [((256, 256), N.F32, 256), ((1024, 2048), N.F32, 1024),
                                               ((64, 64, 64), N.F32, 64), ((512, 512), N.F32, 512),
                                               ((4, 6), N.F32, 64)])
def test_block_plan(dims, prec, threads):
    assert N.lib().fpssft_block_threads(_byref(N.make_shape(dims)), prec) == threads


def test_smem_budget_fits_configs():
    for dims, k_cap in (((256, 256), 256), ((64, 64, 64), 1024), ((1024, 2048), 2048),
                        ((512, 512), 1024)):
        p = P.driver._params(P.FpsSftConfig(), 8, k_cap, N.F32)
        need = N.lib().fpssft_smem_bytes(_byref(N.make_shape(dims)), _byref(p))
        assert 0 < need <= 227 * 1024, (dims, need)


@pytest.mark.parametrize("dims,k_cap,mode", [((256, 256), 256, "warp"), ((512, 512), 1024, "cta"),
                                           ((64, 64, 64), 512, "warp"), ((1024, 2048), 2048, "cta"),
                                           ((12, 18), 64, "cta")])
def test_launch_plan_picks_kernel(dims, k_cap, mode):
    p = P.driver._params(P.FpsSftConfig(), 8, k_cap, N.F32)
    plan = P.driver.launch_plan(P.CubeShape(dims), p)
    assert plan["mode"] == mode
    assert 0 < plan["smem_bytes"] <= 227 * 1024
    if mode == "warp":
        assert plan["threads_per_cta"] == 32 * plan["instances_per_cta"]


def test_sweep_seeds_and_generator_match_reference():  # oracle.py:88-139, 215-227
    from paper_1711_11407_b200 import sweep as S
    ops = G.npz("ops.npz")
    got = np.asarray(S.trial_seeds(505, 8), dtype=np.uint64)
    np.testing.assert_array_equal(got, ops["trial_seeds"])
    for e in OPS["sweep"]:
        kind = "clustered" if e["placement"] == "clustered" else "uniform"
        f, a = S.generate_spectrum(P.CubeShape(e["dims"]), e["k"], e["seed"], kind,
                                   e["cluster_size"])
        order = np.lexsort(f.T[::-1])
        np.testing.assert_array_equal(f[order], ops[f"{e['key']}/freqs"])
        np.testing.assert_array_equal(a[order], ops[f"{e['key']}/amps"])


def test_zero_copy_split_model():
    from paper_1711_11407_b200.hostpath import zero_copy_split

    # config 2: ~2300 of 65536 samples per instance -> mostly zero copy
    f2 = zero_copy_split(2322.0, 256 * 256)
    assert 0.5 < f2 < 1.0
    # config 4: 1 % sampled -> almost all zero copy
    assert zero_copy_split(21972.0, 1024 * 2048) > 0.8
    # sampling every sample many times over -> copy everything
    assert zero_copy_split(1e9, 64) == 0.0
    assert zero_copy_split(0.0, 64) == 1.0
    # monotone in the sample count
    fs = [zero_copy_split(s, 512 * 512) for s in (1e3, 1e4, 1e5, 1e6)]
    assert fs == sorted(fs, reverse=True)


def test_interleave_layout_cpu():
    import torch

    from paper_1711_11407_b200 import interleave

    x = torch.arange(5 * 3 * 4, dtype=torch.float32).reshape(5, 3, 4).to(torch.complex64)
    y = interleave(x, 2)
    assert y.shape == (3, 3, 4, 2)
    for b in range(5):
        assert torch.equal(y[b // 2, ..., b % 2], x[b])
    assert torch.equal(y[2, ..., 1], torch.zeros(3, 4, dtype=torch.complex64))


def test_schedules_from_seeds_pool_matches_serial():
    from paper_1711_11407_b200 import CubeShape
    from paper_1711_11407_b200.schedule import schedule_from_seed, schedules_from_seeds

    shape = CubeShape((32, 24))
    seeds = [3, 99, 12345, 7, 2**40 + 1]
    want = np.stack([schedule_from_seed(shape, s, 40) for s in seeds])
    np.testing.assert_array_equal(schedules_from_seeds(shape, seeds, 40, workers=1), want)
    # forced through the process pool
    np.testing.assert_array_equal(schedules_from_seeds(shape, seeds * 30, 40, workers=2),
                                  np.concatenate([want] * 30))


def test_segment_model_batch_major_and_interleaved():
    """bench.py's DRAM-segment model: batch-major counts a segment per instance
    that runs the iteration; the interleaved layout (group 8) counts each
    sample position once per group, for its longest-running instance."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    from paper_1711_11407_b200 import CubeShape, schedule_from_seed

    shape = CubeShape((16, 16))
    sch = schedule_from_seed(shape, 3, 5)[None]
    one = bench._segments_per_launch(shape, sch, np.array([1]))
    assert bench._segments_per_launch(shape, sch, np.full(16, 1)) == 16 * one
    # group of 8 with equal iteration counts: every (line, sample) position is its own
    # segment, shared by the group
    positions = bench._segments_per_launch(shape, sch, np.array([1]), seg=1)
    assert bench._segments_per_launch(shape, sch, np.full(16, 1), group=8) == 2 * positions
    # a group runs as long as its slowest member
    its = np.array([1] * 7 + [2] + [1] * 8)
    two = bench._segments_per_launch(shape, sch, np.array([2]), seg=1)
    assert bench._segments_per_launch(shape, sch, its, group=8) == two + positions


def test_bench_scaling_plan():
    """bench.py: weak scaling by default (every rank a whole batch, the
    instance ranges disjoint); strong splits the config's global batch."""
    import argparse
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    from paper_1711_11407_b200 import workloads as W

    w = W.CONFIGS[2]
    weak = argparse.Namespace(batch=None, scaling="weak", precision="auto")
    assert bench.batch_plan(weak, w, 8) == (8 * 4096, 4096)
    assert bench.workload_config(weak, w, 8)["scaling"] == "weak"
    strong = argparse.Namespace(batch=None, scaling="strong", precision="auto")
    assert bench.batch_plan(strong, w, 8) == (4096, 512)
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'ap.add_argument("--scaling", default="weak"' in src
