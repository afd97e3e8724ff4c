"""B200-native hot path of multidimensional SSA (arXiv 1309.5050): 2D-SSA, MSSA and
Shaped 2D-SSA trajectory-operator products, block Lanczos SVD and diagonal
averaging, as hand-written sm_100a CUDA kernels behind a C ABI (include/ssa_b200.h).

This package never imports oracle/ (test infrastructure) and has no CPU fallback:
importing the API requires the built libssa_b200.so.
"""
from .api import Plan, version, launch_count, release_workspace  # noqa: F401
from ._lib import SSAError, SO_PATH  # noqa: F401
