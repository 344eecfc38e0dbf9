"""B200-native Gauss-Newton Hessian-matvec library for arXiv 1608.03630 (diffeomorphic registration).

The compute path is the CUDA library libdiffreg.so (C ABI: include/diffreg.h); this package is its
thin ctypes binding.  Nothing here falls back to a CPU implementation.
"""
from .diffreg import *  # noqa: F401,F403
from .diffreg import Config, Context, DiffRegError, lib  # noqa: F401
from . import dist  # noqa: F401,E402
