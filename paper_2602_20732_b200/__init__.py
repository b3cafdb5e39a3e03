"""CHESS decode hot path, B200-native (sm_100a CUDA behind a C-ABI).

Drop-in for the reference `pagesel` selector/engine API
(/root/reference/pkg/src/pagesel/__init__.py:43-86): the same public names,
argument meanings and exceptions, computed by hand-written CUDA kernels in
libchess_b200.so.  There is no CPU fallback: every compute entry point goes
through the C-ABI and raises if the library is missing.
"""

from .config import PRESETS, SelectionConfig, preset_config
from .errors import (
    CalibrationError,
    ConfigurationError,
    EmptyContextError,
    OutOfPagesError,
    PageSelError,
)

__all__ = [
    "PRESETS",
    "SelectionConfig",
    "preset_config",
    "CalibrationError",
    "ConfigurationError",
    "EmptyContextError",
    "OutOfPagesError",
    "PageSelError",
]
