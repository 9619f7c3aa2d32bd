"""B200-native DPar2 hot path (arXiv 2203.12798): stage-1 randomized-SVD
compression of every irregular slice and the compressed-space ALS, as
hand-written sm_100a CUDA kernels behind a C ABI (libdpar2_b200.so).

The public surface mirrors the reference package's hot-path API
(P/__init__.py:19-32): ``fit_dpar2``, ``compress``, ``IrregularTensor``,
``SolverOptions``, ``FitTrace``, ``Parafac2Factors``, ``fitness`` and the
kernel-level functions.  See DESIGN.md.
"""
from .errors import (ArchiveFormatError, DecompositionError, DegenerateInputError, NonFiniteInputError,
                     NumericFailure, RankTooLargeError, ShapeMismatchError)
from .factors import FitTrace, Parafac2Factors, SliceViews, SolverOptions, initial_factors, push_col_norms
from .linalg import RsvdParams, derived_seed
from .scheduler import PartitionPlan, greedy_partition, resolve_threads

__version__ = "0.1.0"

from .tensor import IrregularTensor  # noqa: E402
from .compress import CompressedTensor, compress, reconstruct_slice, set_fp32_products  # noqa: E402
from .solver import (Rotations, convergence_metric, fit_dpar2, mttkrp_mode1, mttkrp_mode2,  # noqa: E402
                     mttkrp_mode3, rotated_cores, update_factors, update_rotations)
from .analysis import fitness  # noqa: E402
from .archive import fit_compressed, load_archive, load_compressed, save_archive, save_compressed  # noqa: E402

_LAZY = ["IrregularTensor", "CompressedTensor", "compress", "reconstruct_slice", "fit_dpar2", "update_rotations",
         "rotated_cores", "mttkrp_mode1", "mttkrp_mode2", "mttkrp_mode3", "update_factors", "convergence_metric",
         "fitness", "Rotations", "load_archive", "save_archive", "load_compressed", "save_compressed",
         "fit_compressed", "set_fp32_products"]

__all__ = sorted(list(_LAZY) + [
    "ArchiveFormatError", "DecompositionError", "DegenerateInputError", "NonFiniteInputError", "NumericFailure", "RankTooLargeError",
    "ShapeMismatchError", "FitTrace", "Parafac2Factors", "SliceViews", "SolverOptions", "initial_factors", "push_col_norms",
    "RsvdParams", "derived_seed", "PartitionPlan", "greedy_partition", "resolve_threads"])
