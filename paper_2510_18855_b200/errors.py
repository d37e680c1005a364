"""Exception types of the drop-in.

When the reference package (``mismatchlab``) is importable, its own classes are
re-exported so code that already catches ``mismatchlab.errors.NumericError``
(e.g. ``cli.py:367-375``) keeps working unchanged; otherwise identical
definitions (``errors.py:4-13`` of the reference) are provided.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the host environment
    from mismatchlab.errors import ConfigError, NumericError, TickCapError  # type: ignore
except Exception:  # noqa: BLE001

    class ConfigError(ValueError):
        """Invalid or malformed experiment configuration (exit code 2)."""

    class NumericError(RuntimeError):
        """A computation produced non-finite values (exit code 3)."""

    class TickCapError(RuntimeError):
        """The simulator exceeded its tick cap without reaching the budget (exit code 4)."""


__all__ = ["ConfigError", "NumericError", "TickCapError"]
