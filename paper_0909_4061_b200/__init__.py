"""B200-native randomized range finder / randomized SVD (Halko-Martinsson-Tropp).

A drop-in for the hot path of the reference package ``lowrank``: the passes
over A (Gaussian sketch A Omega, subspace iteration with re-orthonormalization,
the projection Q*A, the SRFT sketch), the orthonormalization, the small SVD
and the posterior error estimator -- with the reference's function names,
signatures, validation, pass counters and sign conventions.  All arithmetic
runs in hand-written sm_100a CUDA kernels (liblowrank_b200.so, C ABI in
include/lowrank_b200.h); there is no CPU fallback.

    import paper_0909_4061_b200 as lr
    basis = lr.subspace_iteration_range(A, ell=110, q=2, seed=2)
    f = lr.direct_svd(A, basis.Q)
"""

from . import config
from ._lib import ConvergenceError, LibraryMissing, NotPSDError
from .core import (CudaDenseOperator, DenseOperator, MatVecOperator, OperatorCounters, SmallSVD,
                   as_operator, orthonormalize_double_gs, small_eig_hermitian, small_svd)
from .factor import (NystromFactors, PartialEig, PartialSVD, direct_eig_hermitian, direct_svd,
                     eig_nystrom, randomized_svd, truncate_rank)
from .rangefinder import (RangeBasis, adaptive_range_finder, adaptive_range_finder_blocked,
                          fast_range_finder, posterior_error_estimate, power_iteration_range,
                          randomized_range_finder, subspace_iteration_range)
from .sketch import (GsrftOperator, SketchSpec, SrftOperator, dft, gaussian_matrix, gsrft_apply,
                     gsrft_operator, rng_for, srft_apply, srft_operator)
from .sparse import CudaCsrOperator

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")]
