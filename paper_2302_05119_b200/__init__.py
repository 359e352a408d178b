"""concpd_b200 — B200-native CoNCPD-APG / lraCoNCPD-APG hot path.

Drop-in replacement for the solver surface of the reference package
``concpd`` (arXiv 2302.05119; `pkg/src/concpd/__init__.py:1-43`): the same
names, signatures, result types and error behaviour, computed by
hand-written sm_100a kernels behind a C ABI (include/concpd_b200.h).
Importing fails loudly if the native library has not been built.
"""

from . import _lib  # noqa: F401  (loads libconcpd_b200.so or raises ImportError)
from .cpd_als import AlsOptions, AlsResult, cpd_als
from .kruskal import (
    CoupledFactorSet,
    KruskalTensor,
    ddiag_to_tensor,
    normalize_columns,
    reconstruct,
    tensor_to_ddiag,
)
from .solver import (
    CoupledProblem,
    SolveResult,
    SolverOptions,
    TraceRow,
    core_gradient,
    core_linear_term,
    core_linear_terms_tc,
    core_linear_term_lra,
    extrapolation_weight,
    factor_gradient,
    factor_linear_term,
    factor_linear_term_lra,
    init_factors,
    lipschitz_core,
    lipschitz_factor,
    objective,
    solve,
    t_next,
)
from .tensor_ops import (
    factors_khatri_rao,
    hadamard_gram,
    khatri_rao,
    matricize,
    refold,
    spectral_norm,
    unvectorize,
    vectorize,
)

__version__ = "0.1.0"
