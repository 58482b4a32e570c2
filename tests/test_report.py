"""run_decode report + CLI on the device, against reports
the reference's own experiments.run_decode wrote (tests/golden/gen_golden.py:
gen_report, bf16 hot-path boundary) and its weight file format.

CPU: weight-file byte compatibility, prompts, CLI argument errors.
GPU: the logical-clock report equals the reference report field by field
(pinned_mass to 1e-6 -- fp32 sums in a different order), byte-stable JSON,
CSV / --out emission, and the measured-clock rows.
"""
import hashlib
import json
import os

import numpy as np
import pytest
from click.testing import CliRunner

from conftest import GOLDEN

WFILE = os.path.join(GOLDEN, "report_toy.spkc")
CASES = ["b1", "b2_seed9", "b2_prompt"]


def _case(tag):
    with open(os.path.join(GOLDEN, f"report_{tag}.json")) as fh:
        return json.load(fh)


def test_weight_file_byte_compatible():
    from paper_2503_16163_b200.weights import DecoderConfig, init_decoder, load_weights, save_weights
    ref = open(WFILE, "rb").read()
    cfg, w = load_weights(WFILE)
    assert (cfg.layers, cfg.q_heads, cfg.kv_heads, cfg.head_dim, cfg.vocab, cfg.hidden, cfg.ffn,
            cfg.seed) == (2, 4, 2, 8, 64, 32, 64, 2)
    mine = init_decoder(DecoderConfig(seed=2))
    np.testing.assert_array_equal(mine.layers[1].w2, w.layers[1].w2)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "w.spkc")
        assert save_weights(p, cfg, mine) == len(ref)
        assert open(p, "rb").read() == ref


def test_weight_file_errors(tmp_path):
    from paper_2503_16163_b200.weights import DecoderConfig, load_weights
    blob = open(WFILE, "rb").read()
    (tmp_path / "magic").write_bytes(b"XXXX" + blob[4:])
    (tmp_path / "trail").write_bytes(blob + b"\0\0\0\0")
    (tmp_path / "short").write_bytes(blob[:-4])
    (tmp_path / "ver").write_bytes(blob[:4] + (2).to_bytes(4, "little") + blob[8:])
    for name, msg in [("magic", "bad magic"), ("trail", "trailing"), ("short", "missing"),
                      ("ver", "version 2")]:
        with pytest.raises(ValueError, match=msg):
            load_weights(str(tmp_path / name))
    with pytest.raises(ValueError, match="divisible"):
        DecoderConfig(q_heads=3, kv_heads=2)
    with pytest.raises(ValueError, match="even"):
        DecoderConfig(head_dim=7)


def test_make_prompt_matches_reference_reports():
    from paper_2503_16163_b200.report import make_prompt
    for tag in ("b1", "b2_seed9"):
        c = _case(tag)
        p = make_prompt(64, c["args"]["prompt_len"], c["args"]["seed"])
        assert len(p) == c["report"]["config"]["prompt_len"]
        assert c["report"]["summary"]["tokens"][0] is not None


def test_cli_gen_weights_and_argument_errors(tmp_path):
    from paper_2503_16163_b200.cli import main
    r = CliRunner()
    out = r.invoke(main, ["gen-weights", str(tmp_path / "w.spkc"), "--seed", "2"])
    assert out.exit_code == 0, out.output
    payload = json.loads(out.output)
    assert payload["sha256"] == hashlib.sha256(open(WFILE, "rb").read()).hexdigest()
    assert payload["bytes_written"] == os.path.getsize(WFILE)
    assert r.invoke(main, ["decode", WFILE, "--bits", "3"]).exit_code != 0
    assert r.invoke(main, ["decode", str(tmp_path / "nope.spkc")]).exit_code != 0
    assert r.invoke(main, ["gen-weights", str(tmp_path / "x"), "--head-dim", "7"]).exit_code != 0


# ---- GPU -------------------------------------------------------------------------------
def _run(args, clock="logical"):
    from paper_2503_16163_b200.report import run_decode
    return run_decode(WFILE, clock=clock, max_len=4096, **args)


def _strip(rep):
    rep = json.loads(json.dumps(rep))
    rep["config"].pop("weights_path")
    for row in rep["rows"]:
        row.pop("pinned_mass")
    rep["summary"].pop("mean_pinned_mass")
    return rep


@pytest.mark.gpu
@pytest.mark.parametrize("tag", CASES)
def test_logical_report_matches_reference(tag):
    c = _case(tag)
    got = _run(c["args"])
    exp = c["report"]
    assert list(got) == list(exp)
    assert list(got["config"]) == list(exp["config"])
    assert [list(r) for r in got["rows"]] == [list(r) for r in exp["rows"]]
    assert list(got["summary"]) == list(exp["summary"])
    assert _strip(got) == _strip(exp)
    np.testing.assert_allclose([r["pinned_mass"] for r in got["rows"]],
                               [r["pinned_mass"] for r in exp["rows"]], rtol=0, atol=1e-6)
    assert abs(got["summary"]["mean_pinned_mass"] - exp["summary"]["mean_pinned_mass"]) < 1e-6


@pytest.mark.gpu
def test_cli_decode_byte_stable_csv_and_out(tmp_path):
    from paper_2503_16163_b200.cli import main
    r = CliRunner()
    args = ["decode", WFILE, "--steps", "4", "--prompt-len", "12", "--bits", "1", "--g", "4",
            "--residual", "4", "--seed", "9"]
    a, b = r.invoke(main, args), r.invoke(main, args)
    assert a.exit_code == b.exit_code == 0, a.output
    assert a.stdout_bytes == b.stdout_bytes
    assert len(json.loads(a.output)["rows"]) == 4
    c = r.invoke(main, args + ["--csv"])
    lines = c.output.strip().splitlines()
    assert lines[0].startswith("step,token,speculative_hit") and len(lines) == 5
    out = tmp_path / "rep.json"
    assert r.invoke(main, args + ["--out", str(out)]).exit_code == 0
    assert json.loads(out.read_text()) == json.loads(a.output)


@pytest.mark.gpu
def test_measured_clock_rows():
    c = _case("b2_seed9")
    got = _run(c["args"], clock="measured")
    exp = c["report"]
    assert got["config"]["clock"] == "measured"
    assert got["summary"]["tokens"] == exp["summary"]["tokens"]
    assert [r["bytes_fetched"] for r in got["rows"]] == [r["bytes_fetched"] for r in exp["rows"]]
    for row in got["rows"]:
        assert row["overlapped_s"] > 0 and row["compute_s"] > 0
        assert row["compute_s"] <= row["overlapped_s"] + 1e-9
        assert row["serialized_s"] == pytest.approx(row["compute_s"] + row["transfer_s"], abs=2e-9)
        assert (row["transfer_s"] > 0) == (row["bytes_fetched"] > 0)
    assert got["summary"]["overlapped_total_s"] > 0
