"""Imaging duality path, host side (no GPU): the restated phantom and the
sparsity levels are pinned to the reference's own pixels (SHA-256 in
tests/golden/imaging.json, written by make_imaging_golden.py from the
unmodified reference, imaging.py:56-101)."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_1711_11407_b200 import imaging as I

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "imaging.json")))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("key", sorted(GOLD["phantom"]))
def test_phantom_bit_identical_to_reference(key):
    dims, seed = key.split("_s")
    d = tuple(int(v) for v in dims.split("x"))
    assert _sha(I.synthetic_phantom(d, int(seed)).pixels) == GOLD["phantom"][key]


def test_sparsity_levels_match_reference():
    ph = I.synthetic_phantom((512, 576), 1)
    for row in GOLD["duality_512x576"]:
        thr = I.threshold_for_fraction(ph, row["target"])
        assert thr == row["threshold"]
        sp = I.sparsify(ph, thr)
        assert _sha(sp.pixels) == row["sparse_sha"]
        assert int(np.count_nonzero(sp.pixels)) == row["k"]
        assert I.nonzero_fraction(sp) == row["fraction"]


def test_image_validation():  # imaging.py:35-47
    with pytest.raises(ValueError):
        I.GrayImage(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        I.GrayImage(np.full((2, 2), 1.5))
    with pytest.raises(ValueError):
        I.sparsify(I.GrayImage(np.zeros((2, 2))), 2.0)
    with pytest.raises(ValueError):
        I.threshold_for_fraction(I.GrayImage(np.zeros((2, 2))), 0.0)


def test_stepped_offsets():  # lines.py:55-64
    from paper_1711_11407_b200.large import stepped_offsets
    assert stepped_offsets((3, 7), (4, 8)) == [(3, 7), (0, 7), (3, 0)]
