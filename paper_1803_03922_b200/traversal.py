"""Direction-rule constants and scalar helpers (mirror of delegate_bfs.traversal).

The per-level kernels themselves (previsit/visit_forward/visit_backward,
traversal.py:58-139) run on the GPU inside libdbfs
(csrc/bfs_device.cuh); the direction decision is evaluated on device with
the same exact-integer / correctly-rounded arithmetic as
``estimate_backward_workload`` and ``decide_direction`` here
(traversal.py:142-163), which are kept for API compatibility.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

UNREACHED = -1
FORWARD = "forward"
BACKWARD = "backward"
DO_KINDS = ("dd", "dn", "nd")
DEFAULT_FACTOR0 = {"dd": 0.5, "dn": 0.05, "nd": 1e-7}
DEFAULT_FACTOR1 = {"dd": 0.0, "dn": 0.0, "nd": 0.0}


@dataclass
class DirectionState:
    kind: str
    factor0: float
    factor1: float
    direction: str = FORWARD
    allow_switch_back: bool = True


@dataclass
class WorkloadEstimate:
    fv: float = 0.0
    u_size: float = 0.0
    q: float = 0.0
    s: float = 0.0

    @property
    def bv(self) -> float:
        return estimate_backward_workload(self.u_size, self.q, self.s)

    def merge(self, other: "WorkloadEstimate") -> None:
        self.fv += other.fv
        self.u_size += other.u_size
        self.q += other.q
        self.s += other.s


def estimate_backward_workload(u_size: float, q: float, s: float) -> float:
    """|U| * (q + s) / q; infinite with no frontier (traversal.py:142-148)."""
    if q < 0 or s < 0:
        raise ValueError("q and s must be nonnegative")
    if q == 0:
        return math.inf
    return u_size * (q + s) / q


def decide_direction(est: WorkloadEstimate, ds: DirectionState) -> str:
    """Hysteresis rule (traversal.py:151-163)."""
    if ds.kind not in DO_KINDS:
        raise ValueError(f"direction optimization undefined for kind {ds.kind!r}")
    bv = est.bv
    if ds.direction == FORWARD:
        if math.isfinite(bv) and est.fv > ds.factor0 * bv:
            ds.direction = BACKWARD
    else:
        if ds.allow_switch_back and est.fv < ds.factor1 * bv:
            ds.direction = FORWARD
    return ds.direction
