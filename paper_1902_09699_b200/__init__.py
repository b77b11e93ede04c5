"""B200-native PARSDMM hot path (arXiv 1902.09699): sm_100a CUDA kernels behind
the C ABI in include/sip.h, with a thin ctypes binding (``sip``)."""
from .sip import EXPORTS, Grid, SipError, grid_for, lib  # noqa: F401
