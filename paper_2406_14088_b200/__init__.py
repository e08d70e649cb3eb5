"""B200-native parameter reallocation (ReaL, arXiv 2406.14088).

`rlplan` mirrors the reference planner API; `runtime` executes plans on
B200s through librrealloc.so (sm_100a kernels). Importing this package loads
the shared library and fails loudly if it has not been built.
"""
from . import rlplan  # noqa: F401
from ._lib import LIB_PATH, ValidationError  # noqa: F401

__version__ = "0.1.0"
