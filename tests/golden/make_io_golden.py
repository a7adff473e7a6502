"""Golden spectrum text file written by the UNMODIFIED reference's
``save_spectrum`` (core.py:286-291), for the byte-level format pin in
tests/test_spectrum_io.py.  Run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py
"""
import os

import numpy as np
from fps_sft.core import CubeShape, SparseSpectrum, save_spectrum

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(2024)
shape = CubeShape((16, 12, 5))
flat = rng.choice(shape.n_total, size=25, replace=False)
vals = rng.standard_normal((25, 2)) * 10.0 ** rng.integers(-20, 20, (25, 2))
entries = {tuple(int(v) for v in np.unravel_index(f, shape.dims)): complex(re, im)
           for f, (re, im) in zip(flat, vals)}
save_spectrum(SparseSpectrum(shape, entries), os.path.join(HERE, "spectrum_ref.txt"))
np.savez(os.path.join(HERE, "spectrum_ref.npz"),
         freqs=np.asarray(list(entries.keys())), amps=np.asarray(list(entries.values())))
