"""SURVEY 8(f) row 4 on the B200, through the C ABI (csrc/hitrate.cu):

* spc_topk_hitrate / spc_eviction_hitrate are bit-identical to the
  reference's hitrate.py on its own golden sequences (flat, peaky, tied,
  sparse and one-position rows; k from 0 to beyond the row length);
* a 32k-position trace (real context length) from spc_full_attend on
  synthetic peaky keys: rows sum to 1, top-k dominates eviction, both grow
  with k, k >= n gives the full mass, and sampled rows equal the oracle;
* spc_full_attend against a torch fp32 attention (1e-6);
* hitrate_experiment on the device equals the reference report
  (tests/golden/hitrate_report.json) to 1e-6 -- the attention is fp32 on a
  different summation order, the curves are then exact.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from oracle import hitrate as O

pytestmark = pytest.mark.gpu


def _golden_sequences():
    d = golden("hitrate_rows.npz")
    out = []
    for i in range(int(d["nseq"])):
        lens = d[f"lens_{i}"]
        rows = np.split(d[f"rows_{i}"], np.cumsum(lens)[:-1])
        out.append((rows, d[f"topk_{i}"], d[f"evict_{i}"]))
    return d["ks"], out


def test_device_rates_bit_exact_vs_reference():
    from paper_2503_16163_b200 import hitrate as H
    ks, seqs = _golden_sequences()
    for rows, topk, evict in seqs:
        tr = H.AttentionTrace([[rows]])
        tr.validate(1e-5)
        for j, k in enumerate(ks):
            np.testing.assert_array_equal(tr.topk_hitrates(int(k))[0], topk[j])
            np.testing.assert_array_equal(tr.eviction_hitrates(int(k))[0], evict[j])
        np.testing.assert_array_equal(H.topk_hitrate(rows, 3), topk[list(ks).index(3)])
        np.testing.assert_array_equal(H.eviction_hitrate(rows, 5), evict[list(ks).index(5)])


def test_validate_rejects_unnormalised_rows():
    from paper_2503_16163_b200 import hitrate as H
    tr = H.AttentionTrace([[[np.array([0.5, 0.4], np.float32)]]])
    with pytest.raises(ValueError):
        tr.validate()


def test_full_attend_matches_torch_fp32():
    import torch
    from paper_2503_16163_b200 import _lib
    rng = np.random.default_rng(3)
    Hq, Hkv, d, n = 8, 2, 128, 777
    q = torch.as_tensor(rng.standard_normal((Hq, d)), dtype=torch.float32, device="cuda")
    K = torch.as_tensor(rng.standard_normal((n, Hkv, d)), dtype=torch.float32, device="cuda")
    V = torch.as_tensor(rng.standard_normal((n, Hkv, d)), dtype=torch.float32, device="cuda")
    out = torch.empty((Hq, d), dtype=torch.float32, device="cuda")
    probs = torch.zeros((Hq, 1000), dtype=torch.float32, device="cuda")
    scale = float(np.float32(d ** -0.5))
    _lib.check(_lib.lib().spc_full_attend(q.data_ptr(), K.data_ptr(), V.data_ptr(), n, Hq, Hkv, d, scale,
                                          out.data_ptr(), probs.data_ptr(), 1000,
                                          torch.cuda.current_stream().cuda_stream))
    torch.backends.cuda.matmul.allow_tf32 = False
    for h in range(Hq):
        hk = h // (Hq // Hkv)
        s = (q[h].double() @ K[:, hk].double().T) * scale
        p = torch.softmax(s, dim=-1)
        np.testing.assert_allclose(probs[h, :n].double().cpu().numpy(), p.cpu().numpy(), rtol=2e-5, atol=1e-9)
        np.testing.assert_allclose(out[h].double().cpu().numpy(), (p @ V[:, hk].double()).cpu().numpy(),
                                   rtol=1e-4, atol=1e-5)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().spc_full_attend(q.data_ptr(), K.data_ptr(), V.data_ptr(), 0, Hq, Hkv, d, scale,
                                              out.data_ptr(), probs.data_ptr(), 1000, 0))


def test_real_length_trace_properties():
    """32k-position rows (C2's context) from the device attention on peaky
    synthetic keys, 4 steps x 8 heads; curves checked by property and, on a
    sample of rows, against the oracle."""
    import torch
    from paper_2503_16163_b200 import _lib
    from paper_2503_16163_b200.hitrate import AttentionTrace
    rng = np.random.default_rng(7)
    Hq, Hkv, d, n0, steps = 8, 2, 128, 32768, 4
    L = n0 + steps
    K = rng.standard_normal((L, Hkv, d)).astype(np.float32)
    V = rng.standard_normal((L, Hkv, d)).astype(np.float32)
    q0 = rng.standard_normal((Hq, d)).astype(np.float32)
    needles = rng.choice(n0, 64, replace=False)
    for h in range(Hkv):
        K[needles, h] += 0.5 * q0[h * (Hq // Hkv)]
    Kd, Vd = torch.as_tensor(K, device="cuda"), torch.as_tensor(V, device="cuda")
    data = torch.zeros((Hq, steps, L), dtype=torch.float32, device="cuda")
    out = torch.empty((Hq, d), dtype=torch.float32, device="cuda")
    scale = float(np.float32(d ** -0.5))
    lens = []
    for t in range(steps):
        q = q0 + 0.3 * rng.standard_normal((Hq, d)).astype(np.float32)
        qd = torch.as_tensor(q, device="cuda")
        rows = data[:, t]
        _lib.check(_lib.lib().spc_full_attend(qd.data_ptr(), Kd.data_ptr(), Vd.data_ptr(), n0 + t + 1, Hq, Hkv, d,
                                              scale, out.data_ptr(), rows.data_ptr(), rows.stride(0),
                                              torch.cuda.current_stream().cuda_stream))
        lens.append(n0 + t + 1)
    tr = AttentionTrace(data=data, lens=lens)
    tr.validate(1e-5)
    prev_tk = None
    for k in (0, 16, 64, 256, 1024, 4096, L):
        tk, ev = tr.topk_hitrates(k), tr.eviction_hitrates(k)
        assert (ev <= tk + 1e-12).all()
        if prev_tk is not None:
            assert (tk >= prev_tk - 1e-12).all()
        prev_tk = tk
        if k in (64, 1024, L):   # L: the global-memory bitonic path (take > 16384)
            host = data[0].cpu().numpy()
            rows = [host[t, :lens[t]] for t in range(steps)]
            np.testing.assert_array_equal(tk[0], O.topk_hitrate(rows, k))
            np.testing.assert_array_equal(ev[0], O.eviction_hitrate(rows, k))
    np.testing.assert_allclose(tr.topk_hitrates(L), 1.0, atol=1e-5)
    # the q heads the needles were planted along (one per kv head) concentrate their mass
    tk64 = tr.topk_hitrates(64)
    assert tk64[[0, Hq // Hkv]].mean() > 0.3 > 3 * tk64[[1, 2, 3]].mean()


def test_hitrate_experiment_matches_reference_report():
    from paper_2503_16163_b200.hitrate import hitrate_experiment
    with open(os.path.join(GOLDEN, "hitrate_report.json")) as fh:
        ref = json.load(fh)
    wpath = os.path.join(GOLDEN, "report_toy.spkc")
    cwd = os.getcwd()
    os.chdir(GOLDEN)
    try:
        rep = hitrate_experiment(weights_path="report_toy.spkc", max_len=4096, **ref["args"])
    finally:
        os.chdir(cwd)
    r = ref["report"]
    assert rep["experiment"] == "hitrate" and rep["config"] == r["config"]
    assert [(x["k"], x["query_step"]) for x in rep["rows"]] == [(x["k"], x["query_step"]) for x in r["rows"]]
    for a, b in zip(rep["rows"], r["rows"]):
        assert a["topk_rate"] == pytest.approx(b["topk_rate"], abs=1e-6)
        assert a["eviction_rate"] == pytest.approx(b["eviction_rate"], abs=1e-6)
    for key in ("topk_mean", "eviction_mean"):
        np.testing.assert_allclose(rep["summary"][key], r["summary"][key], atol=1e-6)
    assert os.path.exists(wpath)


def test_cli_hitrate_json_and_csv(tmp_path):
    from click.testing import CliRunner
    from paper_2503_16163_b200.cli import main
    w = os.path.join(GOLDEN, "report_toy.spkc")
    r = CliRunner().invoke(main, ["hitrate", w, "--steps", "4", "--prompt-len", "8", "--k-sweep", "2,8"])
    assert r.exit_code == 0, r.output
    rep = json.loads(r.output)
    assert rep["experiment"] == "hitrate" and len(rep["rows"]) == 8
    assert all(x["eviction_rate"] <= x["topk_rate"] + 1e-9 for x in rep["rows"])
    out = tmp_path / "h.csv"
    r = CliRunner().invoke(main, ["hitrate", w, "--steps", "3", "--prompt-len", "8", "--csv", "--out", str(out)])
    assert r.exit_code == 0, r.output
    assert out.read_text().splitlines()[0] == "k,query_step,topk_rate,eviction_rate"
