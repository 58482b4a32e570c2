"""the reference's token loop (generate, engine.py:342-386)
driven end to end on the device cache via DeviceSpeculativeDecoder, against
reference runs recorded with the same bf16 hot-path boundary
(tests/golden/gen_golden.py:gen_adapter)."""
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _model(z):
    cfg = SimpleNamespace(**{k[4:]: int(z[k]) for k in z.files if k.startswith("cfg_") and k != "cfg_rope_base"})
    cfg.rope_base = float(z["cfg_rope_base"])
    layers = [SimpleNamespace(**{n: z[f"w_{i}_{n}"] for n in
                                 ("wq", "wk", "wv", "wo", "attn_norm", "ffn_norm", "w1", "w2")})
              for i in range(cfg.layers)]
    w = SimpleNamespace(embedding=z["w_embedding"], layers=layers, final_norm=z["w_final_norm"],
                        head=z["w_head"])
    return cfg, w


@pytest.mark.parametrize("tag", ["b2", "b1", "b16_exact"])
def test_generate_matches_reference_token_stream(tag):
    from paper_2503_16163_b200 import CacheBudget, ChannelModel
    from paper_2503_16163_b200.adapter import generate
    z = golden(f"adapter_{tag}.npz")
    cfg, w = _model(z)
    budget = CacheBudget(bits=int(z["bits"]), group_size=int(z["g"]), residual=int(z["r"]),
                         prefetch_k=int(z["k"]), context_length=int(z["L"]))
    res = generate(cfg, w, z["prompt"].tolist(), int(z["steps"]), budget,
                   ChannelModel(bandwidth=1e6), compute_time_per_step=1e-3)
    assert res.tokens == z["tokens"].tolist()
    for got, exp in zip(res.logits, z["logits"]):
        np.testing.assert_allclose(got, exp, rtol=2e-3, atol=2e-3)
    np.testing.assert_allclose([m.pinned_mass for m in res.metrics], z["pinned_mass"], rtol=1e-3, atol=1e-5)
    assert [m.new_pins for m in res.metrics] == z["new_pins"].tolist()
    assert [m.bytes_fetched for m in res.metrics] == z["bytes"].tolist()
    assert [m.speculative_hit for m in res.metrics] == z["hit"].tolist()
    np.testing.assert_allclose([r["overlapped_s"] for r in res.latency_rows], z["overlapped"], rtol=1e-12)
    if tag == "b16_exact":  # exact fallback (test_acceptance.py:108-123): same tokens as the full cache
        assert res.tokens == z["base_tokens"].tolist()


def test_phase_rules():
    from paper_2503_16163_b200 import CacheBudget, ProtocolError
    from paper_2503_16163_b200.adapter import DeviceSpeculativeDecoder
    z = golden("adapter_b2.npz")
    cfg, w = _model(z)
    dec = DeviceSpeculativeDecoder(cfg, w, CacheBudget(bits=16, group_size=4, residual=8,
                                                       prefetch_k=1024, context_length=1024))
    with pytest.raises(ProtocolError):
        dec.predecode()
    with pytest.raises(ProtocolError):
        dec.decode_step()
    dec.prefill([1, 2, 3])
    with pytest.raises(ProtocolError):
        dec.prefill([1, 2, 3])
    with pytest.raises(ProtocolError):
        dec.decode_step()
    dec.predecode()
    with pytest.raises(ProtocolError):
        dec.predecode()
    dec.close()
