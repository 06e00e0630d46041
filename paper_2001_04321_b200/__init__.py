"""B200-native HER-AHALS hot path for dense nonnegative CP (arXiv 2001.04321).

The package is a thin Python mirror of the reference toolkit's solver API
(``her_run``, ``ao_run``, ``AoConfig``, ``HerParams``, ``generate``,
``random_init``, the ``ObjectiveProvider`` surface) over the C ABI of
``libntf_b200.so`` (include/ntf_b200.h), whose kernels are hand-written for
sm_100a. Importing the package requires the built shared library.
"""
from . import _lib

_lib.lib()  # fail loudly when the CUDA extension is not built

from .api import (  # noqa: E402,F401
    RUN_DIMTREE, RUN_DIRECT, RUN_GENERIC, RUN_NO_GRAPH, RUN_NO_OVERLAP, AoConfig, Context, CudaError, GpuDenseProvider, HerIterationInfo, HerParams, HerState, InnerStop,
    InvalidArgument, KruskalModel, LogicError, NcclError, NnlsSolver, ObjectiveProvider, RunTrace, Session,
    SyntheticSpec, TraceRecord, UnsupportedError, ahals_solve, ao_run, default_context, device_count,
    factor_error, generate, her_run, load_tensor, pinned_empty, mttkrp_bytes, mttkrp_flops, nnls_solver_from_name, ntft_info,
    random_init, save_tensor, TuckerFormat, TuckerProvider, ttm, hosvd_compress, expand,
    slab_range, solve_nnls, stream_seed, update_betas,
)

__all__ = [n for n in dir() if not n.startswith("_")]
