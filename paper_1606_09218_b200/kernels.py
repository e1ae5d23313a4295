"""``rstensor.kernels`` under its reference name (``kernels.py:1-482``).

The host prologue (sinc quadrature, doubled-grid projection, split, support
radius) lives in :mod:`.quadrature`; this module re-exports it so that
``from rstensor.kernels import project_kernel`` ports by renaming the package.
"""

from .quadrature import *  # noqa: F401,F403
from .quadrature import (DEFAULT_R_RANGE, QuadratureRule, RadialKernel, ReferenceCanonical,  # noqa: F401
                         build_quadrature, effective_support, eval_expansion, project_kernel,
                         split_rank, split_tensor)
