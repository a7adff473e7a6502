"""Pin the CPU oracle (oracle/fps_oracle.py) to the reference.

Two kinds of evidence: (1) the golden fixtures under tests/golden, which are
outputs of the unmodified reference (tests/golden/make_golden.py), and (2) the
inline known-answer values of the reference's own tests (cited per test).
"""

import numpy as np
import pytest

import fixtures as G
from oracle import fps_oracle as O

RUNS = G.meta()["runs"]
OPS = G.meta()["ops"]


def _profile(entry):
    kw = dict(G.PROFILES[entry["profile"]])
    cfg = dict(entry["cfg"])
    seed = cfg.pop("seed", 0)
    return O.Profile(**cfg, **kw), seed


@pytest.mark.parametrize("entry", RUNS, ids=[r["name"] for r in RUNS])
def test_oracle_reproduces_reference_runs(entry):
    cube = G.run_cube(entry)
    prof, seed = _profile(entry)
    rep = O.recover(cube, cube.shape, prof, seed=seed)
    exp = G.run_expected(entry)
    assert rep.iterations_run == exp["iterations_run"]
    assert rep.samples_used == exp["samples_used"]
    assert rep.terminated_by == exp["terminated_by"]
    np.testing.assert_array_equal(rep.freqs, exp["freqs"])
    np.testing.assert_allclose(rep.amps, exp["amps"], rtol=0, atol=1e-12)
    assert [tuple(x[0]) for x in rep.log] == [tuple(a) for a in exp["log_alpha"]]
    assert [tuple(x[1]) for x in rep.log] == [tuple(t) for t in exp["log_tau"]]
    assert [tuple(x[2:]) for x in rep.log] == [tuple(c) for c in exp["log_counts"]]


@pytest.mark.parametrize("entry", OPS["schedule"], ids=[e["key"] for e in OPS["schedule"]])
def test_schedule_replay(entry):
    got = O.replay_schedule(entry["dims"], entry["seed"], entry["T"])
    np.testing.assert_array_equal(got, G.npz("ops.npz")[entry["key"]])


@pytest.mark.parametrize("entry", OPS["line"], ids=[e["key"] for e in OPS["line"]])
def test_lines_and_spectra(entry):
    ops = G.npz("ops.npz")
    k = entry["key"]
    np.testing.assert_array_equal(O.line_coords(entry["alpha"], entry["tau"], entry["dims"]),
                                  ops[f"{k}/idx"])
    np.testing.assert_array_equal(np.asarray(O.stepped_offsets(entry["tau"], entry["dims"])),
                                  ops[f"{k}/offsets"])
    if f"{k}/spectra" in ops:
        got = O.line_spectra(ops[f"{k}/cube"], entry["alpha"], entry["tau"], entry["dims"])
        np.testing.assert_array_equal(got, ops[f"{k}/spectra"])


@pytest.mark.parametrize("entry", OPS["decode"], ids=[e["key"] for e in OPS["decode"]])
@pytest.mark.parametrize("pname", ["P64", "P32"])
def test_classifier(entry, pname):
    ops = G.npz("ops.npz")
    k = entry["key"]
    prof = O.Profile(**G.PROFILES[pname])
    bins, m, amp, nc = O.classify(ops[f"{k}/spectra"], entry["tau"], entry["dims"], prof,
                                  prof.energy_floor_abs)
    assert nc == int(ops[f"{k}/{pname}/ncand"])
    np.testing.assert_array_equal(bins, ops[f"{k}/{pname}/bins"])
    np.testing.assert_array_equal(m, ops[f"{k}/{pname}/freqs"])
    np.testing.assert_array_equal(amp, ops[f"{k}/{pname}/amps"])


@pytest.mark.parametrize("entry", OPS["project"], ids=[e["key"] for e in OPS["project"]])
def test_projection(entry):
    ops = G.npz("ops.npz")
    k = entry["key"]
    np.testing.assert_array_equal(O.bins_of(ops[f"{k}/freqs"], entry["alpha"], entry["dims"]),
                                  ops[f"{k}/bins"])
    got = O.project(ops[f"{k}/freqs"], ops[f"{k}/amps"], entry["alpha"], entry["tau"],
                    entry["dims"])
    np.testing.assert_array_equal(got, ops[f"{k}/out"])


# ---- inline known answers from the reference's own tests ----

def test_diagonal_line_4x6():  # pkg/tests/test_lines.py:18-24
    got = [tuple(r) for r in O.line_coords((1, 1), (0, 0), (4, 6))]
    assert got == [(0, 0), (1, 1), (2, 2), (3, 3), (0, 4), (1, 5),
                   (2, 0), (3, 1), (0, 2), (1, 3), (2, 4), (3, 5)]


def test_offsets_goldens():  # pkg/tests/test_lines.py:90-103
    assert O.stepped_offsets((0, 0), (8, 8)) == [(0, 0), (1, 0), (0, 1)]
    assert O.stepped_offsets((7, 7), (8, 8)) == [(7, 7), (0, 7), (7, 0)]
    assert O.stepped_offsets((1, 2, 3), (4, 4, 4)) == [(1, 2, 3), (2, 2, 3), (1, 3, 3), (1, 2, 0)]


@pytest.mark.parametrize("alpha,ok", [((1, 1), True), ((1, 5), True), ((3, 1), True),
                                      ((2, 1), False), ((1, 3), False), ((2, 3), False)])
def test_slope_validity_4x6(alpha, ok):  # pkg/tests/test_numtheory.py:46-54
    assert O.slope_ok(alpha, (4, 6)) == ok


def test_bin_map_goldens():  # pkg/tests/test_numtheory.py:137-139
    assert int(O.bins_of([[1, 0]], (1, 1), (4, 6))[0]) == 3
    assert int(O.bins_of([[2, 3]], (1, 1), (8, 8))[0]) == 5


def test_decode_golden_8x8():  # pkg/tests/test_decoder.py:57-63
    spectra = np.zeros((3, 8), complex)
    spectra[:, 5] = [1, np.exp(1j * np.pi / 2), np.exp(3j * np.pi / 4)]
    bins, m, amp, nc = O.classify(spectra, (0, 0), (8, 8), O.P64, 1e-12)
    assert list(bins) == [5] and tuple(m[0]) == (2, 3) and abs(amp[0] - 1) < 1e-12


def test_dc_single_iteration():  # pkg/tests/test_driver.py:42-47
    cube = O.synthesize((8, 8), [[0, 0]], [3.0])
    rep = O.recover(cube, (8, 8), O.Profile(max_iterations=10), seed=5)
    assert rep.iterations_run == 1 and rep.terminated_by == "residual_clean"
    assert rep.entries() == {(0, 0): pytest.approx(3 + 0j)}


def test_default_t_max():  # pkg/tests/test_driver.py:36-38
    assert O.default_t_max((256, 256)) == 85 and O.default_t_max((2, 2)) == 1
