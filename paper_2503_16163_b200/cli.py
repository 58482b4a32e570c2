"""`python -m paper_2503_16163_b200 {gen-weights,decode,hitrate}`.

The reference's `speckv gen-weights` / `speckv decode` UX (src/speckv/cli.py:
71-120: same options, defaults, JSON/CSV/--out emission) running in-process on
the B200; the reference's FastAPI service and remote `--server` mode are out
of scope (control plane).  `decode --clock measured` reports
CUDA-event step timings instead of the logical transfer clock.
"""
from __future__ import annotations

import csv
import hashlib
import io
import json
import sys

import click


def _emit(report: dict, as_csv: bool, out: str | None) -> None:
    """cli.py:36-51: the full report as indented JSON, or the rows as CSV."""
    if as_csv:
        buf = io.StringIO()
        rows = report.get("rows", [])
        if rows:
            w = csv.DictWriter(buf, fieldnames=list(rows[0].keys()))
            w.writeheader()
            w.writerows(rows)
        text = buf.getvalue()
    else:
        text = json.dumps(report, indent=2) + "\n"
    if out:
        with open(out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


@click.group()
def main():
    """SpeCache two-tier KV decode on the B200."""


@main.command("gen-weights")
@click.argument("path")
@click.option("--seed", default=0, type=int)
@click.option("--layers", default=2, type=int)
@click.option("--q-heads", default=4, type=int)
@click.option("--kv-heads", default=2, type=int)
@click.option("--head-dim", default=8, type=int)
@click.option("--vocab", default=64, type=int)
@click.option("--hidden", default=32, type=int)
@click.option("--ffn", default=64, type=int)
def gen_weights(path, seed, layers, q_heads, kv_heads, head_dim, vocab, hidden, ffn):
    """Generate a seeded weight file (api.py:87-100 response fields)."""
    from .weights import DecoderConfig, init_decoder, save_weights
    try:
        cfg = DecoderConfig(layers=layers, q_heads=q_heads, kv_heads=kv_heads, head_dim=head_dim,
                            vocab=vocab, hidden=hidden, ffn=ffn, seed=seed)
        n = save_weights(path, cfg, init_decoder(cfg))
    except (ValueError, OSError) as exc:
        raise click.ClickException(str(exc))
    with open(path, "rb") as fh:
        digest = hashlib.sha256(fh.read()).hexdigest()
    sys.stdout.write(json.dumps({"path": path, "bytes_written": n, "sha256": digest}, indent=2) + "\n")


@main.command()
@click.argument("weights_path")
@click.option("--prompt", default=None, help="Comma-separated token ids.")
@click.option("--prompt-len", default=32, type=int)
@click.option("--steps", default=32, type=int)
@click.option("--bits", default="2", type=click.Choice(["1", "2", "4", "16"]))
@click.option("--g", "group_size", default=32, type=int)
@click.option("--k", default=64, type=int)
@click.option("--residual", default=64, type=int)
@click.option("--bandwidth", default=16e9, type=float)
@click.option("--alpha", default=5.0, type=float)
@click.option("--overhead", default=0.0, type=float)
@click.option("--compute-s", default=0.0, type=float)
@click.option("--mode", default="sim", type=click.Choice(["sim", "thread"]))
@click.option("--seed", default=0, type=int)
@click.option("--max-len", default=4096, type=int)
@click.option("--clock", default="logical", type=click.Choice(["logical", "measured"]),
              help="logical: the reference's transfer model; measured: CUDA-event step timings.")
@click.option("--device", default=0, type=int)
@click.option("--json", "as_json", flag_value=True, default=True, help="Full report as JSON (default).")
@click.option("--csv", "as_csv", is_flag=True, default=False, help="Report rows as CSV.")
@click.option("--out", default=None, help="Write output to a file.")
def decode(weights_path, prompt, prompt_len, steps, bits, group_size, k, residual, bandwidth, alpha,
           overhead, compute_s, mode, seed, max_len, clock, device, as_json, as_csv, out):
    """Run a speculative two-tier decode and report per-step metrics."""
    from .report import run_decode
    from .transfer import ProtocolError
    ids = [int(t) for t in prompt.split(",")] if prompt else None
    try:
        report = run_decode(weights_path, ids, prompt_len, steps, int(bits), group_size, k, residual,
                            bandwidth, alpha, overhead, compute_s, mode, seed, max_len=max_len,
                            clock=clock, device=device)
    except (ValueError, OSError, ProtocolError) as exc:
        raise click.ClickException(str(exc))
    _emit(report, as_csv, out)


@main.command()
@click.argument("weights_path")
@click.option("--prompt", default=None, help="Comma-separated token ids.")
@click.option("--prompt-len", default=32, type=int)
@click.option("--steps", default=32, type=int)
@click.option("--k-sweep", default="1,4,16,64", help="Comma-separated k values.")
@click.option("--seed", default=0, type=int)
@click.option("--max-len", default=4096, type=int)
@click.option("--device", default=0, type=int)
@click.option("--json", "as_json", flag_value=True, default=True, help="Full report as JSON (default).")
@click.option("--csv", "as_csv", is_flag=True, default=False, help="Report rows as CSV.")
@click.option("--out", default=None, help="Write output to a file.")
def hitrate(weights_path, prompt, prompt_len, steps, k_sweep, seed, max_len, device, as_json, as_csv, out):
    """Top-k vs greedy-eviction hit-rate curves from a traced decode (cli.py:128-146)."""
    from .hitrate import hitrate_experiment
    ids = [int(t) for t in prompt.split(",")] if prompt else None
    try:
        report = hitrate_experiment(weights_path, ids, prompt_len, steps, [int(v) for v in k_sweep.split(",")],
                                    seed, max_len=max_len, device=device)
    except (ValueError, OSError) as exc:
        raise click.ClickException(str(exc))
    _emit(report, as_csv, out)


if __name__ == "__main__":
    main()
