"""Communication types (mirror of delegate_bfs.comm).

The collectives run inside libdbfs: in-process workers exchange through
device memory, one-worker-per-process runs use NCCL over NVLink
(csrc/dist.cu).  ``CommStats`` keeps the reference's analytic accounting
(comm.py:39-72): mask bytes 2*d*p_rank/8 per dirty iteration, 4 bytes per
normal record.
"""

from __future__ import annotations

from dataclasses import dataclass, field


class RoutingError(ValueError):
    """A record was addressed to a worker that does not own the vertex."""


class StructuralError(ValueError):
    """Mask length mismatch between workers."""


@dataclass
class CommStats:
    mask_bytes: list = field(default_factory=list)
    normal_bytes: list = field(default_factory=list)
    message_count: list = field(default_factory=list)
    pair_count: list = field(default_factory=list)
    wire_bytes: int = 0  # bytes actually moved (8-byte records with parents, masks)
    measured_time_s: float = 0.0  # NCCL level loop: measured exchange time (0: fused into the peer kernel)

    @property
    def total_mask_bytes(self) -> float:
        return sum(self.mask_bytes)

    @property
    def total_normal_bytes(self) -> int:
        return sum(self.normal_bytes)

    @property
    def total_messages(self) -> int:
        return sum(self.message_count)

    @property
    def s_prime(self) -> int:
        return sum(1 for b in self.mask_bytes if b > 0)

    def to_dict(self) -> dict:
        return {
            "mask_bytes": self.mask_bytes,
            "normal_bytes": self.normal_bytes,
            "message_count": self.message_count,
            "pair_count": self.pair_count,
            "total_mask_bytes": self.total_mask_bytes,
            "total_normal_bytes": self.total_normal_bytes,
            "s_prime": self.s_prime,
        }
