"""B200-native Schwarz waveform relaxation hot path (Besse & Xing,
arXiv:1503.02564): C-ABI library libswr.so (include/swr.h) + ctypes binding."""
from .swr import SWR, SWRError, lib, LIB_PATH  # noqa: F401
