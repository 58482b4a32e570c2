"""CPU-only: the C-ABI library loads and exports every symbol the public
header declares; host-side logic (budget, ticket protocol, latency model)
matches the reference's behaviour.  No compute calls (no GPU here)."""
import ctypes
import math

import pytest

from paper_2503_16163_b200 import (CacheBudget, ChannelModel, PrefetchTicket, ProtocolError,
                                   TicketBook, frontier, memory_ratio, step_latency, transfer_time)
from paper_2503_16163_b200 import _lib


def test_library_exports_every_header_symbol():
    syms = _lib.header_symbols()
    assert len(syms) >= 20
    handle = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in syms if not hasattr(handle, s)]
    assert not missing, missing
    assert set(syms) == set(_lib._SIGS), set(syms) ^ set(_lib._SIGS)
    assert _lib.lib().spc_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_loudly():
    from paper_2503_16163_b200 import DeviceTwoTierCache
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises((RuntimeError, MemoryError)):
        DeviceTwoTierCache(1, 2, 8, CacheBudget())


def test_budget_validation_and_ratio():
    with pytest.raises(ValueError):
        CacheBudget(bits=3)
    with pytest.raises(ValueError):
        CacheBudget(residual=0)
    b = CacheBudget(bits=2, group_size=32, residual=64, prefetch_k=64, context_length=4096)
    assert b.ratio() == memory_ratio(2, 32, 4096, 128) == 0.22
    assert memory_ratio(2, 32, 10**12, 0) == 0.19      # half-up, not bankers
    assert memory_ratio(16, math.inf, 10**12, 0) == 1.00
    for length, bits, g, ratio in [(32768, 2, 32, 0.19), (32768, 1, 64, 0.10), (8192, 1, 32, 0.14)]:
        assert memory_ratio(bits, g, length, 128) == ratio


def test_frontier():
    assert frontier(96, 64, 32) == 32 and frontier(95, 64, 32) == 0
    assert frontier(32768, 64, 32) == 32704


def test_ticket_protocol():
    book = TicketBook()
    with pytest.raises(ProtocolError):
        book.await_layer(1, 0)
    book.issue(PrefetchTicket(0, 0, (1, 3), 64))
    with pytest.raises(ProtocolError):
        book.issue(PrefetchTicket(0, 0, (), 0))
    assert book.await_layer(1, 0).positions == (1, 3)
    with pytest.raises(ProtocolError):
        book.await_layer(1, 0)


def test_latency_model():
    m = ChannelModel(bandwidth=1e6, scatter_penalty=5.0)
    assert transfer_time(1000, m, True) == pytest.approx(1e-3)
    assert transfer_time(1000, m, False) == pytest.approx(5e-3)
    assert step_latency(3.0, 2.0, True) == 3.0 and step_latency(3.0, 2.0, False) == 5.0
    with pytest.raises(ValueError):
        ChannelModel(bandwidth=0)
    with pytest.raises(ValueError):
        transfer_time(-1, m, True)
