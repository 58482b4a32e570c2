"""B200-native SpeCache decode hot path (arXiv 2503.16163).

Drop-in for the reference's cache + per-layer decode step
(/root/reference/pkg/src/speckv: kvcache.TwoTierCache, engine's decode-layer
body, transfer's ticket protocol), with the compute in hand-written sm_100a
CUDA (csrc/ -> libspecache.so, C ABI in include/specache.h).
"""
from .budget import FULL_PRECISION_BITS, CacheBudget, frontier, memory_ratio
from .transfer import (ChannelModel, PrefetchTicket, ProtocolError, TicketBook,
                       step_latency, transfer_time)

__version__ = "0.1.0"

__all__ = [
    "CacheBudget", "memory_ratio", "frontier", "FULL_PRECISION_BITS",
    "ChannelModel", "PrefetchTicket", "ProtocolError", "TicketBook", "step_latency",
    "transfer_time", "DeviceTwoTierCache", "SpeculativeLayerDecoder", "StepMetrics",
    "LayerResult", "select_topk",
]


def __getattr__(name):
    # device-facing classes load libspecache.so lazily (and loudly)
    if name == "DeviceTwoTierCache":
        from .cache import DeviceTwoTierCache
        return DeviceTwoTierCache
    if name in ("SpeculativeLayerDecoder", "StepMetrics", "LayerResult", "select_topk"):
        from . import decode
        return getattr(decode, name)
    raise AttributeError(name)
