"""Generate the golden fixtures from the UNMODIFIED reference.

Run in the build container (the reference exists only there):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \
        python tests/golden/make_golden.py

It imports ``fps_sft`` 0.1.0 from ``/root/reference/pkg/src`` and records what
the reference's own functions return on seeded inputs:

* ``runs.npz``      -- ``fps_sft(make_dense_source(cube, shape), FpsSftConfig(...))``
                       (driver.py:121-212) on complex64 cubes: iterations,
                       samples, termination, recovered set, iteration log.
* ``ops.npz``       -- per-function pins: ``line_indices`` / ``decoding_offsets``
                       (lines.py:36-64), ``dft_forward(extract_line(...))``
                       (transform.py:17, lines.py:49), ``decode_spectra``
                       (decoder.py:127-169), ``project_onto_bins``
                       (decoder.py:172-191), ``bins_of_frequencies``
                       (numtheory.py:139-153), ``sample_slope`` schedule replay
                       (numtheory.py:95-110, driver.py:142-143).

Small cubes are stored verbatim.  Large cubes (the config-scale instances)
are stored as their generator recipe plus the SHA-256 of the complex64 cube
bytes; ``tests/golden/fixtures.py`` rebuilds them with
``paper_1711_11407_b200.workloads`` and checks the hash before use.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from fps_sft.core import CubeShape, SparseSpectrum, make_dense_source, make_synthetic_source  # noqa: E402
from fps_sft.decoder import decode_spectra, project_onto_bins  # noqa: E402
from fps_sft.driver import FpsSftConfig, fps_sft  # noqa: E402
from fps_sft.lines import LineParams, decoding_offsets, extract_line, line_indices  # noqa: E402
from fps_sft.numtheory import bins_of_frequencies, sample_slope  # noqa: E402
from fps_sft.transform import dft_forward  # noqa: E402

sys.path.insert(0, HERE)
from fixtures import cube_from_recipe, sha  # noqa: E402

PROFILES = {
    "P64": {},
    "P32": dict(mag_tol=1e-4, verify_tol=1e-4, residual_stop=1e-6),
    "PN": dict(mag_tol=0.3, verify_tol=0.5, round_tol=0.3),
}
INLINE_MAX = 1 << 13  # cubes up to this many elements are stored verbatim


def run_cases():
    cases = []
    cases.append(dict(name="dc_8x8", recipe=dict(kind="spectrum", dims=[8, 8], freqs=[[0, 0]],
                                                 amps_re=[3.0], amps_im=[0.0]),
                      cfg=dict(max_iterations=10, seed=5), profile="P64"))
    dl = [[2, 2], [2, 5], [5, 2], [5, 5]]
    cases.append(dict(name="deadlock_8x8", recipe=dict(kind="spectrum", dims=[8, 8], freqs=dl,
                                                       amps_re=[1.0] * 4, amps_im=[0.0] * 4),
                      cfg=dict(max_iterations=32, stall_limit=8, seed=11), profile="P64"))
    for s in range(8):
        for prof in ("P64", "P32"):
            cases.append(dict(name=f"g16x12_k16_s{s}_{prof}",
                              recipe=dict(kind="reference_generate", dims=[16, 12], k=16, seed=s),
                              cfg=dict(max_iterations=30, stall_limit=10, seed=s + 1000),
                              profile=prof))
    cases.append(dict(name="g16x16_k40_max1",
                      recipe=dict(kind="reference_generate", dims=[16, 16], k=40, seed=6),
                      cfg=dict(max_iterations=1, seed=6), profile="P64"))
    cases.append(dict(name="g16x16_k12_certificate",
                      recipe=dict(kind="reference_generate", dims=[16, 16], k=12, seed=8),
                      cfg=dict(max_iterations=20, seed=9), profile="P32"))
    for dims, k, seed in (([4, 6, 5], 7, 1), ([6, 4, 3], 5, 2), ([8, 8, 8], 12, 3),
                          ([12, 18], 9, 4), ([10, 15], 6, 5), ([32], 3, 6), ([9, 12], 8, 7),
                          ([5, 7], 4, 8), ([16, 16, 16], 30, 9)):
        cases.append(dict(name=f"rand_{'x'.join(map(str, dims))}_k{k}",
                          recipe=dict(kind="random", dims=dims, k=k, seed=seed),
                          cfg=dict(max_iterations=20, stall_limit=6, seed=seed + 50),
                          profile="P32"))
    for dims, k, seed in (([32, 32], 30, 21), ([16, 16, 16], 20, 22)):
        cases.append(dict(name=f"noisy_{'x'.join(map(str, dims))}_k{k}",
                          recipe=dict(kind="random", dims=dims, k=k, seed=seed, noise=0.01),
                          cfg=dict(max_iterations=40, seed=seed + 7), profile="PN"))
    # config-scale instances (one or a few each), default T_max
    cases.append(dict(name="cfg1", recipe=dict(kind="workload", config=1, dims=[256, 256], k=20,
                                                index=0), cfg=dict(seed=7), profile="P32"))
    for i in range(3):
        cases.append(dict(name=f"cfg2_i{i}", recipe=dict(kind="workload", config=2,
                                                          dims=[256, 256], k=100, index=i),
                          cfg=dict(seed=2), profile="P32"))
    cases.append(dict(name="cfg3_i0", recipe=dict(kind="workload", config=3, dims=[64, 64, 64],
                                                   k=200, index=0),
                      cfg=dict(seed=3, max_iterations=200), profile="PN"))
    cases.append(dict(name="cfg4_i0", recipe=dict(kind="workload", config=4, dims=[1024, 2048],
                                                   k=1000, index=0), cfg=dict(seed=4), profile="P32"))
    cases.append(dict(name="cfg5_i0", recipe=dict(kind="workload", config=5, dims=[512, 512],
                                                   k=500, index=0), cfg=dict(seed=5), profile="PN"))
    return cases


def main():
    arrays = {}
    meta = {"runs": [], "reference": "fps-sft 0.1.0 (/root/reference/pkg)",
            "numpy": np.__version__}
    for case in run_cases():
        r = case["recipe"]
        cube = cube_from_recipe(r)
        dims = tuple(r["dims"])
        shape = CubeShape(dims)
        cfg = FpsSftConfig(**case["cfg"], **PROFILES[case["profile"]])
        rep = fps_sft(make_dense_source(cube, shape), cfg)
        n = case["name"]
        freqs = rep.recovered.freq_array.reshape(-1, len(dims))
        arrays[f"{n}/freqs"] = freqs
        arrays[f"{n}/amps"] = rep.recovered.amp_array
        log = rep.iteration_log
        arrays[f"{n}/log_alpha"] = np.asarray([s.alpha for s in log], np.int64)
        arrays[f"{n}/log_tau"] = np.asarray([s.tau for s in log], np.int64)
        arrays[f"{n}/log_counts"] = np.asarray([(s.candidates, s.accepted, s.rejected)
                                                for s in log], np.int64)
        if cube.size <= INLINE_MAX:
            arrays[f"{n}/cube"] = cube
        entry = dict(case, sha256=sha(cube), iterations_run=rep.iterations_run,
                     samples_used=rep.samples_used, terminated_by=rep.terminated_by,
                     k_recovered=rep.recovered.k)
        meta["runs"].append(entry)
        print(f"{n:28s} it={rep.iterations_run:3d} k={rep.recovered.k:4d} {rep.terminated_by}",
              flush=True)
    # baseline_sft (driver.py:219-314), the row/column comparison algorithm
    from fps_sft.driver import baseline_sft
    meta["baseline"] = []
    for name, recipe, cfg in (
            ("bl_single", dict(kind="spectrum", dims=[8, 8], freqs=[[2, 3]], amps_re=[1.5],
                               amps_im=[-0.5]), dict(max_iterations=10)),
            ("bl_deadlock", dict(kind="spectrum", dims=[8, 8], freqs=[[2, 2], [2, 5], [5, 2], [5, 5]], amps_re=[1.0] * 4,
                                 amps_im=[0.0] * 4), dict(max_iterations=30)),
            ("bl_uniform32", dict(kind="reference_generate", dims=[32, 32], k=8, seed=5),
             dict(max_iterations=30)),
            ("bl_uniform64", dict(kind="reference_generate", dims=[64, 64], k=40, seed=9),
             dict(max_iterations=40)),
            ("bl_uniform256", dict(kind="reference_generate", dims=[256, 256], k=128, seed=3),
             dict(max_iterations=60))):
        cube = cube_from_recipe(recipe)
        dims = tuple(recipe["dims"])
        rep = baseline_sft(make_dense_source(cube, CubeShape(dims)),
                           FpsSftConfig(**cfg, **PROFILES["P32"]))
        arrays[f"{name}/freqs"] = rep.recovered.freq_array.reshape(-1, 2)
        arrays[f"{name}/amps"] = rep.recovered.amp_array
        arrays[f"{name}/log_counts"] = np.asarray([(s.candidates, s.accepted, s.rejected)
                                                   for s in rep.iteration_log], np.int64)
        if cube.size <= INLINE_MAX:
            arrays[f"{name}/cube"] = cube
        meta["baseline"].append(dict(name=name, recipe=recipe, cfg=cfg, profile="P32",
                                     sha256=sha(cube), iterations_run=rep.iterations_run,
                                     samples_used=rep.samples_used,
                                     terminated_by=rep.terminated_by))
        print(f"{name:28s} it={rep.iterations_run:3d} k={rep.recovered.k:4d} {rep.terminated_by}")
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **arrays)

    # ---------------- per-function pins ----------------
    ops = {}
    rng = np.random.default_rng(20260101)
    op_meta = {"line": [], "decode": [], "project": [], "schedule": []}
    shapes = [(4, 6), (8, 8), (16, 12), (12, 18), (6, 4, 3), (4, 4, 4), (32,), (256, 256),
              (64, 64, 64), (1024, 2048), (512, 512), (3, 4, 5, 6)]
    for si, dims in enumerate(shapes):
        shape = CubeShape(dims)
        L = shape.line_len
        for j in range(2):
            alpha = sample_slope(shape, rng)
            tau = tuple(int(v) for v in rng.integers(0, shape.dims_array))
            key = f"line{si}_{j}"
            ops[f"{key}/idx"] = line_indices(LineParams(alpha, tau, L), shape)
            ops[f"{key}/offsets"] = np.asarray(decoding_offsets(tau, shape), np.int64)
            if shape.n_total <= (1 << 16):
                cube = (rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(
                    np.complex64)
                src = make_dense_source(cube, shape)
                ops[f"{key}/spectra"] = np.stack(
                    [dft_forward(extract_line(src, LineParams(alpha, off, L)))
                     for off in decoding_offsets(tau, shape)])
                ops[f"{key}/cube"] = cube
            op_meta["line"].append(dict(key=key, dims=list(dims), alpha=list(alpha),
                                        tau=list(tau)))
    # decode_spectra on exact line spectra of sparse mixtures (some colliding)
    for di, dims in enumerate([(8, 8), (16, 12), (12, 18), (6, 4, 3), (64, 64), (9, 10)]):
        shape = CubeShape(dims)
        L = shape.line_len
        for j in range(3):
            k = [2, max(3, L // 2), L][j]
            k = min(k, shape.n_total)
            flat = rng.choice(shape.n_total, size=k, replace=False)
            entries = {tuple(int(v) for v in np.unravel_index(int(f), dims)):
                       complex(rng.uniform(0.5, 2.0) * np.exp(2j * np.pi * rng.random()))
                       for f in flat}
            spec = SparseSpectrum(shape, entries)
            alpha = sample_slope(shape, rng)
            tau = tuple(int(v) for v in rng.integers(0, shape.dims_array))
            src = make_synthetic_source(spec)
            spectra = np.stack([dft_forward(extract_line(src, LineParams(alpha, off, L)))
                                for off in decoding_offsets(tau, shape)])
            key = f"dec{di}_{j}"
            ops[f"{key}/spectra"] = spectra
            for pname in ("P64", "P32"):
                kw = {k2: v for k2, v in PROFILES[pname].items() if k2 != "residual_stop"}
                acc, nc = decode_spectra(spectra, tau, shape, **kw)
                ops[f"{key}/{pname}/bins"] = np.asarray([b for b, _ in acc], np.int64)
                ops[f"{key}/{pname}/freqs"] = np.asarray([s.freq for _, s in acc],
                                                         np.int64).reshape(-1, len(dims))
                ops[f"{key}/{pname}/amps"] = np.asarray([s.amp for _, s in acc], np.complex128)
                ops[f"{key}/{pname}/ncand"] = np.asarray(nc)
            op_meta["decode"].append(dict(key=key, dims=list(dims), alpha=list(alpha),
                                          tau=list(tau)))
    # project_onto_bins / bins_of_frequencies
    for pi, dims in enumerate([(8, 8), (16, 12), (6, 4, 3), (256, 256), (1024, 2048)]):
        shape = CubeShape(dims)
        k = 50
        freqs = np.stack([rng.integers(0, n, k) for n in dims], axis=-1).astype(np.int64)
        amps = rng.standard_normal(k) + 1j * rng.standard_normal(k)
        alpha = sample_slope(shape, rng)
        tau = tuple(int(v) for v in rng.integers(0, shape.dims_array))
        key = f"proj{pi}"
        ops[f"{key}/freqs"] = freqs
        ops[f"{key}/amps"] = amps
        ops[f"{key}/out"] = project_onto_bins(freqs, amps, alpha, tau, shape)
        ops[f"{key}/bins"] = bins_of_frequencies(freqs, alpha, shape)
        op_meta["project"].append(dict(key=key, dims=list(dims), alpha=list(alpha),
                                       tau=list(tau)))
    # schedule replay: the (alpha, tau) stream fps_sft draws (driver.py:131,142-143)
    for qi, (dims, seed, T) in enumerate([((256, 256), 2, 85), ((64, 64, 64), 3, 200),
                                          ((1024, 2048), 4, 64), ((512, 512), 5, 170),
                                          ((16, 12), 1000, 30), ((4, 6, 5), 52, 20),
                                          ((2, 2), 0, 4), ((1, 7), 3, 5)]):
        shape = CubeShape(dims)
        g = np.random.default_rng(seed)
        sched = []
        for _ in range(T):
            a = sample_slope(shape, g)
            t = tuple(int(v) for v in g.integers(0, shape.dims_array))
            sched.append((a, t))
        ops[f"sched{qi}"] = np.asarray(sched, np.int64)
        op_meta["schedule"].append(dict(key=f"sched{qi}", dims=list(dims), seed=seed, T=T))
    # sweep generator pins: run_sweep's trial seeds (oracle.py:215-227) and
    # generate() spectra for uniform and clustered placements (oracle.py:88-139)
    from fps_sft.oracle import GeneratorSpec, _trial_seeds, generate
    op_meta["sweep"] = []
    ops["trial_seeds"] = np.asarray(_trial_seeds(505, 8), dtype=np.uint64)
    for gi, (dims, k, placement, csize, seed) in enumerate(
            [((256, 256), 1280, "uniform", None, 11), ((32, 32), 9, "clustered", 9, 12),
             ((64, 48), 50, "clustered", 25, 13), ((16, 12), 16, "uniform", None, 14)]):
        truth, _ = generate(GeneratorSpec(shape=CubeShape(dims), k=k, placement=placement,
                                          cluster_size=csize, seed=seed))
        ops[f"gen{gi}/freqs"] = truth.freq_array
        ops[f"gen{gi}/amps"] = truth.amp_array
        op_meta["sweep"].append(dict(key=f"gen{gi}", dims=list(dims), k=k, placement=placement,
                                     cluster_size=csize, seed=seed))
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **ops)
    meta["ops"] = op_meta
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
