"""Numerical defaults of the hot path (reference config.py:9,19,22-23,26)."""

# Gram-Schmidt drop tolerance relative to ||Y||_F (orthonormalize_double_gs).
GS_DROP_TOL = 1e-10

# Fixed-rank sketches default to k + DEFAULT_OVERSAMPLE samples.
DEFAULT_OVERSAMPLE = 5

# Posterior error estimator: probe count and inflation factor.
DEFAULT_PROBES = 10
DEFAULT_ALPHA = 10.0

# Probe batch of the blocked adaptive range finder.
ADAPTIVE_BLOCK = 8

# Semidefinite tolerance of the PSD Cholesky (pivots in [-PSD_TOL ||B||_2, 0]
# clamp to zero), reference config.py:16.
PSD_TOL = 1e-12

# One-pass SVD solves a dense system over vec(B); refuse above this size
# (reference config.py:30-31).  Condition threshold above which one-pass
# solvers attach a warning (config.py:33-34).
ONE_PASS_DIM_CAP = 250_000
ONE_PASS_COND_WARN = 1e12
