"""B200-native RS-tensor pose rescoring (arXiv 2510.26611, Algorithm PLIE + Eq. (22)).

The product is librsdock.so (C ABI in include/rs_dock.h, CUDA kernels for sm_100a);
`rsdock` is its thin ctypes binding."""
from . import rsdock  # noqa: F401
from .rsdock import Protein  # noqa: F401
