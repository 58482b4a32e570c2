"""Transfer-channel vocabulary of the reference (transfer.py), host side.

On B200 the channel is real: tickets are CUDA events on the cache's copy
stream and the fetch is the K5 zero-copy gather (csrc/select.cu).  What stays
on the host is the protocol -- a ticket issued at (step, layer) must be awaited
exactly once at (step+1, layer) -- and the latency arithmetic used by the
report rows.  Same names, argument meaning and error behaviour as
``transfer.py:31-115``.
"""
from __future__ import annotations

from dataclasses import dataclass

__all__ = ["ProtocolError", "ChannelModel", "PrefetchTicket", "transfer_time",
           "step_latency", "TicketBook"]


class ProtocolError(RuntimeError):
    """Raised when the issue/await ticket contract is violated (transfer.py:31-32)."""


@dataclass(frozen=True)
class ChannelModel:
    """transfer.py:35-47 (modelled link; the device path measures the real one)."""
    bandwidth: float = 16e9
    scatter_penalty: float = 5.0
    fixed_overhead: float = 0.0

    def __post_init__(self) -> None:
        if self.bandwidth <= 0:
            raise ValueError("bandwidth must be positive")
        if self.scatter_penalty < 1:
            raise ValueError("scatter_penalty must be >= 1")
        if self.fixed_overhead < 0:
            raise ValueError("fixed_overhead must be >= 0")


@dataclass(frozen=True)
class PrefetchTicket:
    """transfer.py:50-55.  ``positions`` is per (seq, unit) on the device path."""
    step: int
    layer: int
    positions: tuple
    num_bytes: int


def transfer_time(num_bytes: float, model: ChannelModel, contiguous: bool) -> float:
    """transfer.py:58-63."""
    if num_bytes < 0:
        raise ValueError("num_bytes must be >= 0")
    factor = 1.0 if contiguous else model.scatter_penalty
    return model.fixed_overhead + num_bytes / model.bandwidth * factor


def step_latency(compute_s: float, transfer_s: float, overlapped: bool) -> float:
    """transfer.py:66-71."""
    if compute_s < 0 or transfer_s < 0:
        raise ValueError("latencies must be >= 0")
    return max(compute_s, transfer_s) if overlapped else compute_s + transfer_s


class TicketBook:
    """Host mirror of the (step, layer) ticket contract of SimulatedChannel
    (transfer.py:84-100): duplicate issue or a missing await raises
    ProtocolError.  The C library enforces the same rule per layer; this
    book lets callers (and CPU tests) check it without a device."""

    def __init__(self) -> None:
        self._pending: dict[tuple[int, int], PrefetchTicket] = {}

    def issue(self, ticket: PrefetchTicket) -> None:
        key = (ticket.step, ticket.layer)
        if key in self._pending:
            raise ProtocolError(f"duplicate ticket for step {ticket.step} layer {ticket.layer}")
        self._pending[key] = ticket

    def await_layer(self, step: int, layer: int) -> PrefetchTicket:
        key = (step - 1, layer)
        if key not in self._pending:
            raise ProtocolError(f"no ticket was issued at step {step - 1} for layer {layer}")
        return self._pending.pop(key)

    def pending(self) -> list:
        return sorted(self._pending)
