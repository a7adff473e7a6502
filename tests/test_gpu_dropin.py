"""The drop-in proven through the reference itself: the unmodified reference
package (installed into baseline/_ref by ``pip install --target``; these
tests skip when it is absent) dispatches to the B200 path through its own
``ALGORITHMS`` registry (``pkg/src/fps_sft/oracle.py:33,152-160``), hands it
its own source objects (``DenseSource``, ``core.py:220-238``;
``SyntheticSource``, ``core.py:176-217``) and config class, and gets results
equal to what its own ``fps_sft`` returns on the same source and config.
"""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1711_11407_b200 as P  # noqa: E402
from paper_1711_11407_b200 import workloads as W  # noqa: E402

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline",
                   "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "fps_sft")):
        pytest.skip("the reference is not installed in baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import fps_sft
    finally:
        sys.path.remove(REF)
    assert os.path.abspath(fps_sft.__file__).startswith(REF)
    return fps_sft


P32 = dict(mag_tol=1e-4, verify_tol=1e-4, residual_stop=1e-6)


def _same_report(got, want, rtol):
    assert got.iterations_run == want.iterations_run
    assert got.samples_used == want.samples_used
    assert got.terminated_by == want.terminated_by
    assert list(got.recovered.entries) == list(want.recovered.entries)
    for f, a in want.recovered.entries.items():
        assert abs(got.recovered.entries[f] - a) <= rtol * abs(a), f
    assert [(s.alpha, s.tau, s.candidates, s.accepted, s.rejected) for s in got.iteration_log] \
        == [(s.alpha, s.tau, s.candidates, s.accepted, s.rejected) for s in want.iteration_log]


@pytest.mark.parametrize("dims,k,seed", [((64, 48), 12, 3), ((256, 256), 100, 8),
                                         ((32, 32, 16), 20, 4)])
def test_reference_dense_source_and_config(ref, dims, k, seed):
    """The reference's own ``make_dense_source`` object and ``FpsSftConfig``
    instance into ``b200.fps_sft``: the same report as the reference's
    ``fps_sft`` on that very object (support, iterations, samples, log)."""
    f, a = W.reference_generate(dims, k, seed)
    cube = W.synthesize_np(dims, f, a).astype(np.complex64)
    src = ref.make_dense_source(cube, ref.CubeShape(dims))
    cfg = ref.FpsSftConfig(seed=seed + 11, **P32)
    want = ref.fps_sft(src, cfg)
    _same_report(P.fps_sft(src, cfg), want, 1e-4)
    _same_report(P.fps_sft(src, cfg, precision="fp64"), want, 1e-9)


def test_reference_run_trial_dispatches_to_b200(ref):
    """``ALGORITHMS["fps-b200"] = b200.fps_sft`` and the reference's
    ``run_trial`` (generate -> lazy SyntheticSource -> ALGORITHMS[algo] ->
    spectra_match): success at the north-star tolerance, like its own."""
    ref.oracle.ALGORITHMS["fps-b200"] = P.fps_sft
    try:
        for seed in range(4):
            spec = ref.oracle.GeneratorSpec(shape=ref.CubeShape((128, 96)), k=40, seed=seed)
            cfg = ref.FpsSftConfig(seed=100 + seed, **P32)
            got = ref.oracle.run_trial("fps-b200", spec, cfg, match_rtol=1e-4)
            own = ref.oracle.run_trial("fps", spec, cfg, match_rtol=1e-4)
            assert got.success and own.success
            assert got.samples_used == got.iterations * 3 * 384
    finally:
        ref.oracle.ALGORITHMS.pop("fps-b200", None)
