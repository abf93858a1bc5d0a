"""The ``strategy`` argument of ``Pipeline``, kept for API compatibility.

In the reference it selects serial execution or a thread pool that splits
every stage into row/column blocks
(/root/reference/pkg/src/clutterwhiten/parallel.py:18-85).  Here each frame
is one fused GPU launch whatever the strategy says, so it changes neither
the work nor the results; it is still parsed, validated and reported with
the reference's spellings and error messages (parallel.py:25-40).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["ExecStrategy"]

_MODES = ("serial", "parallel")
_DEFAULT_POOL = 4  # workers of a bare "parallel"


@dataclass(frozen=True)
class ExecStrategy:
    """A mode (``serial`` | ``parallel``) and, for ``parallel``, a worker
    count of at least one."""

    mode: str = "serial"
    workers: int = 1

    def __post_init__(self):
        if self.mode not in _MODES:
            raise ValueError(f"strategy mode must be serial|parallel, got {self.mode!r}")
        if self.mode == "parallel" and self.workers < 1:
            raise ValueError(f"parallel strategy needs workers >= 1, got {self.workers}")

    @classmethod
    def parse(cls, text: str) -> "ExecStrategy":
        """Accepts ``serial``, ``parallel`` and ``parallel:N``."""
        mode, colon, count = text.partition(":")
        if not colon and mode in _MODES:
            return cls(mode, _DEFAULT_POOL if mode == "parallel" else 1)
        if colon and mode == "parallel":
            return cls(mode, int(count))
        raise ValueError(f"unknown strategy {text!r}")

    @property
    def name(self) -> str:
        """The spelling ``parse`` accepts back."""
        return f"parallel:{self.workers}" if self.mode == "parallel" else "serial"
