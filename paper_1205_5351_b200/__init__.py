"""paper_1205_5351_b200 — B200-native (sm_100a) batched TILT solver (Ren & Lin, arXiv 1205.5351).

The hot path (warp/Jacobian, orthonormalisation, LADMAP with warm Jacobi SVT, persistent scheduler)
lives in ``csrc/`` and is reached through the C ABI of ``libtilt.so`` (``include/tilt.h``). This
package is the thin binding; ``dist`` adds the multi-GPU sharding. Importing it fails loudly when
the CUDA library has not been built.
"""
from ._abi import (AFFINE, HOMOGRAPHY, CONVERGED, MAX_OUTER, WINDOW_ESCAPE, SINGULAR_GRAM, ZERO_PATCH,  # noqa: F401
                   DIVERGED, BAD_BOX, CONSTRAINTS_NONE, CONSTRAINTS_CENTER_AREA, TiltError, TiltParams, default_params,
                   lib, LIB_PATH, EXPORTS)
from .solver import TiltSolver, REPORT_DTYPE, reports_to_numpy, p_of  # noqa: F401

__all__ = ["TiltSolver", "default_params", "TiltParams", "TiltError", "AFFINE", "HOMOGRAPHY", "REPORT_DTYPE",
           "reports_to_numpy"]
