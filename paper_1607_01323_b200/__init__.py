"""B200-native matrix-free DG operators (arXiv 1607.01323 hot path).

Drop-in for the reference ``dgins`` operator/solver API on the GPU:
``operators`` (SIP Laplace, mass, Helmholtz, projection, convective),
``solvers`` (PCG, Chebyshev, Lanczos, zero-mean projections), ``mesh`` /
``spaces`` (structured boxes), ``parallel`` (x-slab decomposition over
NCCL).  All compute runs in hand-written sm_100a CUDA kernels of the
in-tree ``libdgmf.so`` (C ABI: include/dgmf.h).
"""

__version__ = "0.1.0"

from . import _lib  # noqa: F401
