"""B200-native FPS-SFT: the projection-slice sparse Fourier transform
recovery loop (arXiv 1711.11407) as hand-written sm_100a CUDA behind a C ABI.

Drop-in for the reference package's ``fps_sft`` path: same names and
meanings as ``fps_sft.core`` / ``fps_sft.driver`` for the types the loop
consumes and produces, plus batched and per-step device entry points.
"""

from .core import (CubeShape, DenseSource, FreqIndex, SignalSource, Sinusoid, SparseSpectrum,
                   SyntheticSource, make_dense_source, make_synthetic_source, spectra_match)
from .driver import (PROFILES, BatchResult, BatchRunner, FpsSftConfig, IterationStats,
                     RecoveryReport, default_max_iterations, fps_sft, fps_sft_batch, interleave,
                     materialize, max_k_cap)
from .baseline import baseline_sft
from .imaging import GrayImage, reconstruct_sparse_image, synthetic_phantom
from .large import fps_sft_large
from .schedule import (bins_of_frequencies, is_valid_slope, sample_slope, schedule_from_seed,
                       valid_slopes)

__version__ = "0.1.0"

ALGORITHMS = {"fps-b200": fps_sft, "baseline-b200": baseline_sft}

__all__ = ["ALGORITHMS", "BatchResult", "BatchRunner", "CubeShape", "DenseSource",
           "FpsSftConfig", "FreqIndex", "GrayImage", "IterationStats", "PROFILES",
           "RecoveryReport", "fps_sft_large", "reconstruct_sparse_image", "synthetic_phantom",
           "SignalSource", "Sinusoid", "SyntheticSource", "SparseSpectrum", "baseline_sft", "bins_of_frequencies",
           "default_max_iterations", "fps_sft", "fps_sft_batch", "interleave", "is_valid_slope",
           "make_dense_source", "make_synthetic_source", "materialize", "max_k_cap", "sample_slope",
           "schedule_from_seed", "spectra_match", "valid_slopes"]
