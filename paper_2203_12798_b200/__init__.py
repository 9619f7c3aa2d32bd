"""B200-native DPar2 hot path (arXiv 2203.12798): stage-1 randomized-SVD
compression of every irregular slice and the compressed-space ALS, as
hand-written sm_100a CUDA kernels behind a C ABI (libdpar2_b200.so).

The public surface mirrors the reference package's hot-path API
(P/__init__.py:19-32): ``fit_dpar2``, ``compress``, ``IrregularTensor``,
``SolverOptions``, ``FitTrace``, ``Parafac2Factors``, ``fitness`` and the
kernel-level functions.  See DESIGN.md.
"""
from .errors import (DecompositionError, DegenerateInputError, NonFiniteInputError, NumericFailure,
                     RankTooLargeError, ShapeMismatchError)
from .factors import FitTrace, Parafac2Factors, SolverOptions, initial_factors, push_col_norms
from .linalg import RsvdParams, derived_seed
from .scheduler import PartitionPlan, greedy_partition, resolve_threads

__version__ = "0.1.0"

_LAZY = {
    "IrregularTensor": "tensor", "CompressedTensor": "compress", "compress": "compress",
    "reconstruct_slice": "compress", "fit_dpar2": "solver", "update_rotations": "solver",
    "rotated_cores": "solver", "mttkrp_mode1": "solver", "mttkrp_mode2": "solver", "mttkrp_mode3": "solver",
    "update_factors": "solver", "convergence_metric": "solver", "fitness": "analysis",
    "fit_dpar2_distributed": "distributed",
}


def __getattr__(name):  # torch-dependent modules load on first use
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f"{__name__}.{mod}"), name)


__all__ = sorted(list(_LAZY) + [
    "DecompositionError", "DegenerateInputError", "NonFiniteInputError", "NumericFailure", "RankTooLargeError",
    "ShapeMismatchError", "FitTrace", "Parafac2Factors", "SolverOptions", "initial_factors", "push_col_norms",
    "RsvdParams", "derived_seed", "PartitionPlan", "greedy_partition", "resolve_threads"])
