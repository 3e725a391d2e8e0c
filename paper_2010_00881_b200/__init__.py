"""B200-native hierarchical p-multigrid for finite cell systems (arXiv 2010.00881).

The compute path is libfcm_mg.so (sm_100a CUDA + C++, C ABI in include/fcm_mg.h);
this package is a thin ctypes layer.  See DESIGN.md."""
from ._lib import EXPORTED, FcmError  # noqa: F401

__all__ = ["EXPORTED", "FcmError"]
