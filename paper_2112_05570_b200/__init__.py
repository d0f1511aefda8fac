"""B200-native batched 2D ray-query engine for the hot path of arXiv 2112.05570
(`mintri`): stackless ray traversal through a constrained (annealed MWT)
triangulation, its start-triangle location, and like-for-like roped kd-tree /
SAH BVH walks -- hand-written sm_100a CUDA behind a C ABI (include/mwt.h).

Importing the package loads libmwt.so; there is no CPU fallback.
"""
from ._lib import MwtError  # noqa: F401  (loads libmwt.so, fails loudly)

__version__ = "0.1.0"
