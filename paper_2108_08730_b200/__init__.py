"""B200-native wavelength-adaptive 27-point Helmholtz hot path (arXiv 2108.08730).

The compute lives in `libhz.so` (hand-written sm_100a CUDA behind the C ABI of include/hz.h);
`hz` is its thin ctypes binding.  PyTorch provides device memory, streams and process groups.
"""
from . import hz  # noqa: F401  (raises ImportError when libhz.so is missing: no CPU fallback)
from .hz import *  # noqa: F401,F403
