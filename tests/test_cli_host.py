"""The ``recover`` command-line mirror (reference cli.py:117-171) on the host:
seed split and generated ground truth pinned to the unmodified reference
(tests/golden/cli.json, made by tests/golden/make_cli_golden.py), argument
errors, the lazy source's exact-phase samples."""
import json
import os

import numpy as np
import pytest

from paper_1711_11407_b200 import CubeShape, make_synthetic_source
from paper_1711_11407_b200 import cli
from paper_1711_11407_b200 import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cli.json")))


@pytest.mark.parametrize("seed", sorted(GOLD["split"], key=int))
def test_seed_split_matches_reference(seed):
    assert list(cli.split_seed(int(seed))) == GOLD["split"][seed]


@pytest.mark.parametrize("case", GOLD["truth"], ids=lambda c: c["placement"])
def test_generated_truth_matches_reference(case):
    args = cli.build_parser().parse_args(
        ["recover", "--shape", "x".join(map(str, case["shape"])), "--k", str(case["k"]),
         "--placement", case["placement"], "--seed", str(case["seed"])])
    gen_seed, _ = cli.split_seed(case["seed"])
    truth = cli.truth_spectrum(args, gen_seed)
    assert [list(f) for f in truth.entries] == case["freqs"]
    got = np.asarray([[a.real, a.imag] for a in truth.entries.values()])
    np.testing.assert_array_equal(got, np.asarray(case["amps"]))


def test_recover_needs_a_truth(tmp_path):
    args = cli.build_parser().parse_args(["recover", "--out", str(tmp_path)])
    with pytest.raises(SystemExit):
        cli.truth_spectrum(args, 0)
    with pytest.raises(SystemExit):
        cli.build_parser().parse_args(["recover", "--shape", "3y4"])


def test_synthetic_source_samples_exactly(rng):
    case = GOLD["truth"][1]
    shape = CubeShape(case["shape"])
    args = cli.build_parser().parse_args(
        ["recover", "--shape", "x".join(map(str, case["shape"])), "--k", str(case["k"]),
         "--placement", case["placement"], "--seed", str(case["seed"])])
    truth = cli.truth_spectrum(args, cli.split_seed(case["seed"])[0])
    src = make_synthetic_source(truth)
    dense = W.synthesize_np(shape.dims, truth.freq_array, truth.amp_array)
    idx = np.stack([rng.integers(0, d, 50) for d in shape.dims], axis=1)
    np.testing.assert_allclose(src.sample_many(idx), dense[tuple(idx.T)], atol=1e-12)
    assert abs(src.sample(tuple(idx[0])) - dense[tuple(idx[0])]) < 1e-12
