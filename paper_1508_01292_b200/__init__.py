"""B200-native compact CNN cascade face detector hot path (arXiv 1508.01292).

The product is libccnn.so (include/ccnn.h, sm_100a kernels in csrc/); ``ccnn`` is its
ctypes binding.  There is no CPU fallback.
"""
from .ccnn import Detector, CcnnError, load, BOX_DTYPE, CAND_DTYPE  # noqa: F401
