"""Report types shared by the GPU executor and the simulator model.

Same schema as the reference simulator's (``swapgraph/sim.py:43-113``), so a
measured run and a modelled run of one schedule can be compared field by
field: the executor fills ``peak_device_bytes`` from the device pool's
high-water mark, ``peak_host_bytes`` from the pinned pool,
``transfer_time_total`` from copy-engine busy time and
``transfer_wait_total`` from compute-stream stalls on swap-in events.
Times are seconds.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Any


class DeadlockError(RuntimeError):
    """Reachable ops can never run (e.g. a control edge from a blocked op)."""


@dataclass(frozen=True)
class SimConfig:
    """Capacity and link model (sim.py:47-71).  The measured ``simulate``
    (simulate.py) enforces ``device_capacity_bytes`` as its pool budget and maps
    ``overlap_transfers`` onto separate or shared copy streams; the bandwidths
    are not modelled there (the host link is real)."""

    device_capacity_bytes: int = 16 * 2**30
    host_to_device_bandwidth: float = float(80 * 2**30)
    device_to_host_bandwidth: float = float(80 * 2**30)
    overlap_transfers: bool = True
    serial_engine: bool = False

    def __post_init__(self):
        if self.device_capacity_bytes <= 0:
            raise ValueError("device_capacity_bytes must be positive")
        if not self.host_to_device_bandwidth > 0:
            raise ValueError("host_to_device_bandwidth must be positive")
        if not self.device_to_host_bandwidth > 0:
            raise ValueError("device_to_host_bandwidth must be positive")

    @classmethod
    def serial_oracle(cls, device_capacity_bytes: int = 16 * 2**30) -> "SimConfig":
        """One engine, instantaneous transfers."""
        return cls(device_capacity_bytes=device_capacity_bytes,
                   host_to_device_bandwidth=math.inf, device_to_host_bandwidth=math.inf,
                   serial_engine=True)


@dataclass(frozen=True)
class TraceEvent:
    time: float
    event: str  # start | finish | xfer_start | xfer_finish | alloc | free
    node: int | None = None
    tensor: int | None = None
    bytes: int = 0
    device: str | None = None


@dataclass
class SimReport:
    peak_device_bytes: int
    peak_host_bytes: int
    makespan: float
    transfer_time_total: float
    transfer_wait_total: float
    oom: bool
    event_trace: list[TraceEvent] = field(default_factory=list)

    def to_dict(self) -> dict[str, Any]:
        d = {k: getattr(self, k) for k in ("peak_device_bytes", "peak_host_bytes", "makespan",
                                           "transfer_time_total", "transfer_wait_total", "oom")}
        d["event_trace"] = [dict(time=e.time, event=e.event, node=e.node, tensor=e.tensor,
                                 bytes=e.bytes, device=e.device) for e in self.event_trace]
        return d
