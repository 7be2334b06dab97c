"""Seeded synthetic QP instances shared by the oracle tests, the GPU tests and bench.py.

This package only *generates inputs* (matrices and vectors drawn from seeded numpy
generators, plus the feasible-point bookkeeping b = A x0, c = A^T y0 + z0 - q x0 that the
BASELINE.json config recipes prescribe).  It holds none of the method's arithmetic:
no normal-equation operator, no sketch, no PCG, no IP-PMM step.  Neither `oracle/` nor
the CUDA path is imported from here.
"""
from .configs import (QPInstance, make_config, make_general, make_svm_dual, make_portfolio,  # noqa: F401
                      structured_dense_A, CONFIG_NAMES, gaussian_matrix)
