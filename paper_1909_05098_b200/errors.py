"""Exception hierarchy of the B200 FED-FEM engine.

The class names, base classes and attributes follow the reference package's
error module (/root/reference/pkg/src/fedheat/errors.py:4-51) so callers can
catch the same types.  The native library reports failures as integer status
codes (see include/fedheat_b200.h, ``FH_ERR_*``); `raise_for_status` turns a
status plus the library's thread-local message into one of these exceptions.
"""

from __future__ import annotations


class FedheatError(Exception):
    """Root of every error raised by this package."""


class MeshFormatError(FedheatError, ValueError):
    """Bad mesh input; ``line`` is the 1-based source line when known."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


class DegenerateElementError(FedheatError, ValueError):
    """An element with non-positive volume / Jacobian determinant."""

    def __init__(self, message: str, element: int | None = None):
        self.element = element
        super().__init__(message if element is None else f"element {element}: {message}")


class ConfigError(FedheatError, ValueError):
    """Invalid configuration value or combination."""


class InstabilityError(FedheatError, RuntimeError):
    """Non-finite or runaway temperature after an explicit step."""

    def __init__(self, message: str, step: int, time: float, node: int | None = None):
        self.step = step
        self.time = time
        self.node = node
        super().__init__(f"step {step} (t={time:.6g} s): {message}")


class ConvergenceError(FedheatError, RuntimeError):
    """An iterative solve did not reach its tolerance."""


class SizeCapError(FedheatError, ValueError):
    """A size-capped helper was asked to exceed its cap."""


class DeviceError(FedheatError, RuntimeError):
    """CUDA / NCCL failure inside the native engine (status FH_ERR_DEVICE)."""


# status codes shared with include/fedheat_b200.h
FH_OK = 0
FH_ERR_CONFIG = 1
FH_ERR_INSTABILITY = 2
FH_ERR_DEVICE = 3
FH_ERR_DEGENERATE = 4
FH_ERR_FORMAT = 5


def raise_for_status(status: int, message: str) -> None:
    if status == FH_OK:
        return
    if status == FH_ERR_CONFIG:
        raise ConfigError(message)
    if status == FH_ERR_DEGENERATE:
        raise DegenerateElementError(message)
    if status == FH_ERR_FORMAT:
        raise MeshFormatError(message)
    if status == FH_ERR_DEVICE:
        raise DeviceError(message)
    raise FedheatError(f"native status {status}: {message}")
