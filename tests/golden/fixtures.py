"""Loader for the golden fixtures written by ``make_golden.py`` (outputs of
the unmodified reference).  Import-safe on the GPU box: it needs only numpy
and ``paper_1711_11407_b200.workloads`` (to rebuild large cubes, verified by
SHA-256)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from paper_1711_11407_b200 import workloads as W

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(cube: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(cube, np.complex64).tobytes()).hexdigest()


def cube_from_recipe(r: dict) -> np.ndarray:
    """Rebuild a fixture cube (complex64) from its recipe."""
    dims = tuple(r["dims"])
    if r["kind"] == "workload":
        w = W.CONFIGS[r["config"]]
        w = W.Workload(w.name, dims, 1, r["k"], w.placement, w.magnitude, w.noise_var,
                       w.profile, w.seed)
        rng = W.instance_rngs(w.seed, 1, r["index"])[0]
        return W.make_instance(w, rng)[2]
    if r["kind"] == "reference_generate":
        f, a = W.reference_generate(dims, r["k"], r["seed"])
        return W.synthesize_np(dims, f, a).astype(np.complex64)
    if r["kind"] == "spectrum":
        return W.synthesize_np(dims, np.asarray(r["freqs"]), np.asarray(r["amps_re"]) +
                               1j * np.asarray(r["amps_im"])).astype(np.complex64)
    if r["kind"] == "random":
        rng = np.random.default_rng(r["seed"])
        k = r["k"]
        flat = rng.choice(int(np.prod(dims)), size=k, replace=False)
        f = np.stack(np.unravel_index(flat, dims), axis=-1)
        a = rng.uniform(0.5, 2.0, k) * np.exp(2j * np.pi * rng.random(k))
        cube = W.synthesize_np(dims, f, a)
        if r.get("noise", 0) > 0:
            s = np.sqrt(r["noise"] / 2)
            cube = cube + s * (rng.standard_normal(dims) + 1j * rng.standard_normal(dims))
        return cube.astype(np.complex64)
    raise ValueError(r["kind"])



PROFILES = {
    "P64": {},
    "P32": dict(mag_tol=1e-4, verify_tol=1e-4, residual_stop=1e-6),
    "PN": dict(mag_tol=0.3, verify_tol=0.5, round_tol=0.3),
}


def meta() -> dict:
    with open(os.path.join(HERE, "golden.json")) as fh:
        return json.load(fh)


_NPZ = {}


def npz(name: str):
    if name not in _NPZ:
        _NPZ[name] = dict(np.load(os.path.join(HERE, name)))
    return _NPZ[name]


def run_cube(entry: dict) -> np.ndarray:
    """The exact complex64 cube the reference ran on for a ``runs`` entry."""
    arrays = npz("runs.npz")
    key = f"{entry['name']}/cube"
    cube = arrays[key] if key in arrays else cube_from_recipe(entry["recipe"])
    if sha(cube) != entry["sha256"]:
        raise AssertionError(f"fixture cube for {entry['name']} does not reproduce")
    return cube


def run_expected(entry: dict) -> dict:
    a = npz("runs.npz")
    n = entry["name"]
    return dict(freqs=a[f"{n}/freqs"], amps=a[f"{n}/amps"], log_alpha=a[f"{n}/log_alpha"],
                log_tau=a[f"{n}/log_tau"], log_counts=a[f"{n}/log_counts"],
                iterations_run=entry["iterations_run"], samples_used=entry["samples_used"],
                terminated_by=entry["terminated_by"])
