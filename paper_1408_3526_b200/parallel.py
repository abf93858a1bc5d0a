"""Execution-strategy argument kept for API compatibility.

The reference parallelises with row/column fork-join on a thread pool
(/root/reference/pkg/src/clutterwhiten/parallel.py:18-85).  Here every
frame is one fused GPU launch, so the strategy never changes the work or
the results; ``Pipeline`` still accepts and reports it, with the same
parsing and error messages (parallel.py:25-40).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["ExecStrategy"]


@dataclass(frozen=True)
class ExecStrategy:
    """``serial`` or ``parallel`` with ``workers >= 1``."""

    mode: str = "serial"
    workers: int = 1

    def __post_init__(self):
        if self.mode not in ("serial", "parallel"):
            raise ValueError(f"strategy mode must be serial|parallel, got {self.mode!r}")
        if self.mode == "parallel" and self.workers < 1:
            raise ValueError(f"parallel strategy needs workers >= 1, got {self.workers}")

    @classmethod
    def parse(cls, text: str) -> "ExecStrategy":
        """``"serial"``, ``"parallel"`` (4 workers) or ``"parallel:N"``."""
        if text == "serial":
            return cls()
        if text == "parallel":
            return cls("parallel", 4)
        head, sep, tail = text.partition(":")
        if head == "parallel" and sep:
            return cls("parallel", int(tail))
        raise ValueError(f"unknown strategy {text!r}")

    @property
    def name(self) -> str:
        return self.mode if self.mode == "serial" else f"parallel:{self.workers}"
