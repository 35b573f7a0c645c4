"""B200-native partitioned sort (arXiv 1105.6040's scatter / sort / merge path).

Layers:
  include/b200sort.h + csrc/*.cu   C ABI and sm_100a kernels (libb200sort.so)
  _lib.py / device.py              ctypes binding, per-device Context
  sortbench.py                     the reference's entry points (same names/semantics)
  sample_sort.py                   multi-GPU sample sort, one process per GPU
"""
from ._lib import B2SError, LIB_PATH  # noqa: F401
from .errors import ConfigError, DeviceError, ProgrammingError, VerificationError  # noqa: F401

__all__ = ["ConfigError", "DeviceError", "ProgrammingError", "VerificationError", "LIB_PATH"]
