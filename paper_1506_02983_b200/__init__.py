"""B200-native hot path of ECMG_jcg (arXiv:1506.02983): a C-ABI CUDA library (libecmg.so, sources
in csrc/, header in include/ecmg.h) and its thin ctypes binding (ecmg.py)."""
from . import ecmg  # noqa: F401
from .ecmg import Grid, EcmgError, PROB  # noqa: F401
