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
from .factor import (InterpolativeDecomp, NystromFactors, PartialEig, PartialSVD, SampleBundle,
                     column_id, direct_eig_hermitian, direct_svd, eig_nystrom, eig_one_pass,
                     eig_via_row_extraction, randomized_svd, row_id, sample_bundle,
                     svd_via_row_extraction,
                     sample_bundle_two_sided, stage_a, svd_one_pass_general, svd_single_pass,
                     truncate_rank)
from .io import (MatrixFormatError, RowBlockStream, StreamError, accumulate_two_sided_samples,
                 in_memory_sample_bundle, read_matrix_binary, stream_row_blocks,
                 streamed_sample_bundle, write_matrix_binary)
from .rangefinder import (RangeBasis, adaptive_range_finder, adaptive_range_finder_blocked,
                          fast_range_finder, posterior_error_estimate, power_iteration_range,
                          randomized_range_finder, subspace_iteration_range)
from .sketch import (GsrftOperator, SketchSpec, SrftOperator, dense_sketch_matrix, dft,
                     gaussian_matrix, gsrft_apply, gsrft_operator, op_count, reset_op_count,
                     rng_for, sketch_apply, srft_apply, srft_operator)
from .sparse import CudaCsrOperator

__version__ = "0.1.0"

__all__ = [name for name in dir() if not name.startswith("_")]
