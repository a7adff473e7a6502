"""Spectrum text format (reference core.py:280-333; tests mirror
pkg/tests/test_core.py:160-206): exact round trip including float bits,
comments and blank lines, and parse errors that carry file:line context."""

import numpy as np
import pytest

from paper_1711_11407_b200.core import CubeShape, SparseSpectrum
from paper_1711_11407_b200.spectrum_io import load_spectrum, save_spectrum


@pytest.mark.parametrize("dims", [(7,), (4, 6), (3, 5, 2), (2, 2, 2, 3)])
def test_round_trip_is_bit_exact(tmp_path, dims):
    rng = np.random.default_rng(len(dims))
    shape = CubeShape(dims)
    k = min(6, shape.n_total)
    flat = rng.choice(shape.n_total, size=k, replace=False)
    vals = rng.standard_normal((k, 2)) * 10.0 ** rng.integers(-300, 300, (k, 2))
    entries = {tuple(int(v) for v in np.unravel_index(f, dims)): complex(re, im)
               for f, (re, im) in zip(flat, vals)}
    spec = SparseSpectrum(shape, entries)
    path = tmp_path / "spec.txt"
    save_spectrum(spec, path)
    loaded = load_spectrum(path)
    assert loaded.shape.dims == spec.shape.dims
    assert loaded.entries == spec.entries


def test_comments_and_blank_lines(tmp_path):
    path = tmp_path / "spec.txt"
    path.write_text("# a comment\n\n# shape 4 6\n# another\n1 2 0.5 -0.25\n")
    assert load_spectrum(path).entries == {(1, 2): 0.5 - 0.25j}


@pytest.mark.parametrize("content,message", [
    ("1 2 0.5 0.5\n", "before '# shape'"),
    ("# shape 4 6\n1 2 0.5\n", "expected 4 fields"),
    ("# shape 4 6\n9 2 0.5 0.5\n", "out of range"),
    ("# shape 4 6\n1 2 0 0\n", "zero amplitude"),
    ("# shape 4 6\n1 2 0.5 0.5\n1 2 1 1\n", "duplicate"),
    ("# shape\n", "bad shape header"),
    ("# shape 4 6\n# shape 4 6\n", "duplicate shape header"),
    ("# just a comment\n", "missing '# shape'"),
    ("# shape 4 6\n1 x 0.5 0.5\n", "spec.txt:2"),
])
def test_parse_errors_carry_context(tmp_path, content, message):
    path = tmp_path / "spec.txt"
    path.write_text(content)
    with pytest.raises(ValueError, match=message):
        load_spectrum(path)


def test_matches_reference_file_byte_for_byte(tmp_path):
    """tests/golden/spectrum_ref.txt was written by the reference's own
    save_spectrum (make_io_golden.py)."""
    import os

    gold = os.path.join(os.path.dirname(__file__), "golden", "spectrum_ref.txt")
    spec = load_spectrum(gold)
    ref = np.load(os.path.join(os.path.dirname(__file__), "golden", "spectrum_ref.npz"))
    assert spec.entries == {tuple(int(v) for v in f): complex(a)
                            for f, a in zip(ref["freqs"], ref["amps"])}
    out = tmp_path / "again.txt"
    save_spectrum(spec, out)
    assert out.read_bytes() == open(gold, "rb").read()
