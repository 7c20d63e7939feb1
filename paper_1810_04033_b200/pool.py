"""Device "pool": the GPU stand-in for the reference WorkerPool.

The reference requires a worker pool for every non-serial strategy
(strategies.py:538-539) and drives each colour with
`WorkerPool.parallel_for` (taskrt.py:455-491).  On the GPU one kernel grid
replaces the pool, so `DevicePool` only carries the device and stream the
sweeps are issued on, plus the attributes the strategy layer reads
(`size`, `tracing`).  `Schedule` is accepted and ignored: colouring results do
not depend on it (reference tests/test_strategies.py:155-164).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["DevicePool", "WorkerPool", "Schedule"]


@dataclass(frozen=True)
class Schedule:
    """Loop schedule of the reference parallel_for (taskrt.py:56-82)."""

    kind: str = "static"
    chunk: int = 1

    def __post_init__(self):
        if self.kind not in ("static", "dynamic"):
            raise ValueError(f"schedule must be 'static' or 'dynamic', got {self.kind!r}")
        if self.chunk < 1:
            raise ValueError("chunk must be >= 1")

    @classmethod
    def parse(cls, text: str) -> "Schedule":
        if text == "static":
            return cls("static")
        if text.startswith("dynamic"):
            _, _, rest = text.partition(":")
            return cls("dynamic", int(rest) if rest else 1)
        raise ValueError(f"cannot parse schedule {text!r}")

    def describe(self) -> str:
        return "static" if self.kind == "static" else f"dynamic:{self.chunk}"


class DevicePool:
    """One CUDA device (and the torch current stream on it)."""

    def __init__(self, size: int = 1, device=None, steal_seed=None, stall_timeout: float = 10.0):
        if size < 1:
            raise ValueError("pool size must be >= 1")
        self.size = size          # kept for API compatibility; the grid ignores it
        self.device = device
        self.tracing = False      # per-cell tracing does not exist on the GPU path
        self.closed = False

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.shutdown()

    def shutdown(self):
        self.closed = True


WorkerPool = DevicePool
