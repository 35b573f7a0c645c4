"""Exception taxonomy of the reference (P/include/sortbench/errors.hpp:10-46),
mapped from the C ABI's status codes (include/b200sort.h)."""
from __future__ import annotations


class ConfigError(ValueError):
    """Invalid configuration or arguments (CLI exit 2, P/tools/sortbench.cpp:379-388)."""


class ProgrammingError(RuntimeError):
    """Internal misuse, e.g. quick_sort's out-of-range segment (P/src/sort_core.cpp:137-142)."""


class VerificationError(RuntimeError):
    """Output that is not the sorted input (P/src/bench.cpp:95-104)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL / out-of-memory failures (std::runtime_error in the shims);
    ``status`` is 2 (out of memory), 3 (CUDA) or 5 (NCCL)."""

    def __init__(self, msg: str, status: int = 3):
        super().__init__(msg)
        self.status = status


def from_status(status: int, msg: str) -> Exception:
    if status == 1:
        return ConfigError(msg)
    if status == 4:
        return ProgrammingError(msg)
    return DeviceError(msg, status)
