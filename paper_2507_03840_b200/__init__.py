"""B200-native esgnn hot path: CUDA sm_100a kernels behind a C ABI
(include/esg.h, libesg_b200.so); `esg` is the ctypes binding."""
from . import esg  # noqa: F401
