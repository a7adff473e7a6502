"""``recover`` from the reference's command line (``fps_sft/cli.py:117-171``),
run on the GPU path: ``python -m paper_1711_11407_b200 recover ...``.

Same flags, outputs and exit codes as the reference's subcommand: a ground
truth spectrum is read (``--input``, the reference's text format) or drawn
(``--shape --k --placement``, the reference's generator and seed split), the
lazy source is materialised on the device, ``fps_sft`` recovers it, and
``recovered_spectrum.txt``, ``report.json`` and ``manifest.json`` are written
to ``--out``; exit 0 when the recovery matches the truth, 2 when it does not,
1 on input errors.  Differences: the cube is complex64 (the device layout), so
the match uses ``--rtol`` (default 1e-5) instead of the reference's exact
complex128 1e-8; ``--precision`` picks the arithmetic (float64 by default,
with the reference's default tolerances); ``--algo`` names the GPU entry
points.  The other subcommands (sweep, image, selftest) are reachable from
Python (``sweep.run_sweep``, ``imaging.reconstruct_sparse_image``).
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import sys
from pathlib import Path

import numpy as np

from . import __version__
from .core import CubeShape, SparseSpectrum, make_synthetic_source, spectra_match
from .driver import PROFILES, FpsSftConfig, RecoveryReport
from .spectrum_io import load_spectrum, save_spectrum
from .sweep import PLACEMENTS, generate_spectrum


def parse_shape(text: str) -> CubeShape:
    try:
        return CubeShape(int(part) for part in text.lower().split("x"))
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"bad shape {text!r}: {exc}") from None


def default_seed() -> int:
    env = os.environ.get("FPS_SFT_SEED")
    if env is not None:
        try:
            return int(env)
        except ValueError:
            raise SystemExit(f"FPS_SFT_SEED must be an integer, got {env!r}") from None
    return 0


def split_seed(seed: int) -> tuple[int, int]:
    """(generator seed, algorithm seed), as the reference derives them."""
    gen_ss, algo_ss = np.random.SeedSequence(seed).spawn(2)
    return (int(gen_ss.generate_state(1, dtype=np.uint64)[0]),
            int(algo_ss.generate_state(1, dtype=np.uint64)[0]))


def report_dict(report: RecoveryReport) -> dict:
    return {
        "iterations_run": report.iterations_run,
        "samples_used": report.samples_used,
        "percent_samples": report.percent_samples(),
        "k_recovered": report.recovered.k,
        "terminated_by": report.terminated_by,
        "iteration_log": [
            {"iteration": s.iteration, "alpha": list(s.alpha), "tau": list(s.tau),
             "candidates": s.candidates, "accepted": s.accepted, "rejected": s.rejected}
            for s in report.iteration_log
        ],
    }


def write_manifest(out_dir: Path, subcommand: str, resolved: dict, seed: int) -> None:
    manifest = {
        "subcommand": subcommand,
        "config": resolved,
        "seed": seed,
        "version": __version__,
        "created_utc": datetime.datetime.now(datetime.timezone.utc).isoformat(),
        "argv": sys.argv[1:],
    }
    (out_dir / "manifest.json").write_text(json.dumps(manifest, indent=2) + "\n")


def algo_config(args, seed: int) -> FpsSftConfig:
    kwargs = dict(PROFILES[args.profile]) if args.profile else {}
    kwargs["seed"] = seed
    if args.tmax:
        kwargs["max_iterations"] = args.tmax
    if args.stall:
        kwargs["stall_limit"] = args.stall
    return FpsSftConfig(**kwargs)


def truth_spectrum(args, gen_seed: int) -> SparseSpectrum:
    if args.input:
        truth = load_spectrum(args.input)
        if args.shape and args.shape.dims != truth.shape.dims:
            raise SystemExit(f"--shape {args.shape.dims} conflicts with input file shape "
                             f"{truth.shape.dims}")
        return truth
    if not args.shape or not args.k:
        raise SystemExit("recover needs either --input or both --shape and --k")
    placement, cluster = PLACEMENTS[args.placement]
    freqs, amps = generate_spectrum(args.shape, args.k, gen_seed, placement, cluster)
    return SparseSpectrum(args.shape, {tuple(int(v) for v in f): complex(a)
                                       for f, a in zip(freqs, amps)})


def cmd_recover(args) -> int:
    from . import ALGORITHMS

    out_dir = Path(args.out)
    out_dir.mkdir(parents=True, exist_ok=True)
    seed = args.seed if args.seed is not None else default_seed()
    gen_seed, algo_seed = split_seed(seed)
    truth = truth_spectrum(args, gen_seed)
    shape = truth.shape
    config = algo_config(args, algo_seed)
    runner = ALGORITHMS[args.algo]
    report = runner(make_synthetic_source(truth), config, precision=args.precision)
    success = spectra_match(report.recovered, truth, rtol=args.rtol)

    save_spectrum(report.recovered, out_dir / "recovered_spectrum.txt")
    payload = report_dict(report)
    payload.update(shape=list(shape.dims), k_true=truth.k, success=success, algo=args.algo,
                   precision=args.precision)
    (out_dir / "report.json").write_text(json.dumps(payload, indent=2) + "\n")
    write_manifest(out_dir, "recover",
                   {"algo": args.algo, "shape": list(shape.dims), "k": truth.k,
                    "placement": args.placement if not args.input else None,
                    "input": args.input, "tmax": config.max_iterations,
                    "stall": config.stall_limit, "precision": args.precision,
                    "profile": args.profile}, seed)
    print(f"recovered {report.recovered.k}/{truth.k} sinusoids in {report.iterations_run} "
          f"iterations ({report.samples_used} samples); "
          f"{'perfect' if success else 'incomplete'}")
    return 0 if success else 2


def build_parser() -> argparse.ArgumentParser:
    from . import ALGORITHMS

    parser = argparse.ArgumentParser(prog="fps-sft-b200",
                                     description="FPS-SFT recovery on the B200 path")
    parser.add_argument("--version", action="version", version=__version__)
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("recover", help="recover a sparse spectrum from a synthetic source")
    p.add_argument("--shape", type=parse_shape, default=None, help="cube shape, e.g. 256x256")
    p.add_argument("--k", type=int, default=None, help="number of sinusoids to generate")
    p.add_argument("--placement", choices=sorted(PLACEMENTS), default="uniform")
    p.add_argument("--input", default=None, help="spectrum file to use as ground truth")
    p.add_argument("--algo", choices=sorted(ALGORITHMS), default="fps-b200")
    p.add_argument("--precision", choices=["fp32", "fp64"], default="fp64")
    p.add_argument("--profile", choices=sorted(PROFILES), default=None,
                   help="tolerance profile (default: the reference's defaults)")
    p.add_argument("--rtol", type=float, default=1e-5, help="amplitude match tolerance")
    p.add_argument("--seed", type=int, default=None, help="RNG seed (default: FPS_SFT_SEED or 0)")
    p.add_argument("--tmax", type=int, default=None, help="iteration cap")
    p.add_argument("--stall", type=int, default=None, help="stall limit")
    p.add_argument("--out", default="out", help="output directory")
    p.set_defaults(func=cmd_recover)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
