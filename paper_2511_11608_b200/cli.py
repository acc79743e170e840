"""Command-line drop-in for the reference CLI's codec commands.

    python -m paper_2511_11608_b200 gen|encode|decode|stats [options]

Same subcommands, options, defaults, output text / JSON and exit codes as the reference
(cli.py:1-37, :61-250): 0 success, 2 usage/config, 3 I/O, 4 file format.  The codec work
runs on the GPU: `.tns` files are loaded into device memory (pinned host staging), encoded
/ decoded by libsif.so, and written back.  Planner and simulator commands (plan, plan-ar,
search, simulate) are outside the codec path and not provided; `calibrate`
writes a measured DeviceTimeModel JSON for the reference planner's --timemodel option.
"""

from __future__ import annotations

import json
import sys

import click
import numpy as np

EXIT_OK = 0
EXIT_USAGE = 2
EXIT_IO = 3
EXIT_FORMAT = 4


def _fail(code: int, message: str):
    click.echo(f"error: {message}", err=True)
    sys.exit(code)


def _run(fn):
    """cli.py:46-58 exception -> exit code mapping."""
    from .errors import ConfigError, SlicerError, StreamFormatError, TensorFormatError

    try:
        fn()
    except (TensorFormatError, StreamFormatError) as exc:
        _fail(EXIT_FORMAT, str(exc))
    except ConfigError as exc:
        _fail(EXIT_USAGE, str(exc))
    except OSError as exc:
        _fail(EXIT_IO, str(exc))
    except SlicerError as exc:
        _fail(EXIT_USAGE, str(exc))


@click.group()
def main():
    """Split-computing feature codec (B200 CUDA implementation)."""


@main.command()
@click.option("--rows", type=int, required=True)
@click.option("--cols", type=int, required=True)
@click.option("--seed", type=int, default=0, show_default=True)
@click.option("--dist", type=click.Choice(["uniform", "gaussian"]), default="uniform")
@click.option("--out", "out_path", required=True, type=click.Path(dir_okay=False))
def gen(rows, cols, seed, dist, out_path):
    """Generate a deterministic fixture tensor (.tns)."""

    def go():
        from .tensor import random_tensor, save_tensor

        t = random_tensor(rows, cols, seed, dist)
        save_tensor(t, out_path)
        click.echo(f"wrote {rows}x{cols} {dist} tensor (seed {seed}) to {out_path}")

    _run(go)


def _parse_q_list(text):
    from .errors import ConfigError

    try:
        return tuple(int(p) for p in text.split(","))
    except ValueError:
        raise ConfigError(f"bad Q list {text!r}; expected comma-separated integers")


def _block_rows(blocks):
    out, idx = [], {"plus": 0, "minus": 0}
    for b in blocks:
        out.append({"plane": b["plane"], "index": idx[b["plane"]], "nnz": b["nnz"], "q": b["q"]})
        idx[b["plane"]] += 1
    return out


@main.command("encode")
@click.option("--in", "in_path", required=True, type=click.Path(exists=True, dir_okay=False))
@click.option("--out", "out_path", required=True, type=click.Path(dir_okay=False))
@click.option("--sparsity", "-s", type=float, required=True)
@click.option("--lambda", "lam", type=float, default=0.0, show_default=True)
@click.option("--blocks", default="1,1", show_default=True, help="M+,M- block counts")
@click.option("--qbit", type=int, default=8, show_default=True)
@click.option("--delta", type=float, default=None, help="ABQ distortion budget")
@click.option("--fixed-q", default=None, help="comma-separated Q vector (disables ABQ)")
@click.option("--seed", type=int, default=0, show_default=True)
@click.option("--json", "as_json", is_flag=True)
def encode_cmd(in_path, out_path, sparsity, lam, blocks, qbit, delta, fixed_q, seed, as_json):
    """Compress a .tns tensor into a .sif bitstream."""

    def go():
        from .codec import MODE_ABQ, MODE_FIXED, CodecConfig, broadcast_q, encode
        from .errors import ConfigError
        from .tensor import load_tensor

        m = _parse_q_list(blocks)
        if len(m) != 2:
            raise ConfigError("--blocks expects 'M+,M-'")
        m_plus, m_minus = m
        if fixed_q is not None:
            cfg = CodecConfig(s=sparsity, lam=lam, m_plus=m_plus, m_minus=m_minus, q_bit=qbit,
                              delta=0.0 if delta is None else delta, mode=MODE_FIXED,
                              fixed_q=broadcast_q(_parse_q_list(fixed_q), m_plus, m_minus))
        else:
            cfg = CodecConfig(s=sparsity, lam=lam, m_plus=m_plus, m_minus=m_minus, q_bit=qbit,
                              delta=0.01 if delta is None else delta, mode=MODE_ABQ)
        x = load_tensor(in_path)
        p = encode(x, cfg, seed)
        data = bytes(p)
        with open(out_path, "wb") as f:
            f.write(data)
        bits = p.payload_bits
        size = x.shape[0] * x.shape[1]
        info = {"payload_bits": bits, "bits_per_element": bits / size, "blocks": _block_rows(p.blocks())}
        if as_json:
            click.echo(json.dumps(info, indent=2))
        else:
            click.echo(f"payload: {bits} bits ({bits / size:.3f} bits/element)")
            for b in info["blocks"]:
                click.echo(f"  {b['plane']} block {b['index']}: nnz={b['nnz']} q={b['q']}")

    _run(go)


@main.command("decode")
@click.option("--in", "in_path", required=True, type=click.Path(exists=True, dir_okay=False))
@click.option("--out", "out_path", required=True, type=click.Path(dir_okay=False))
@click.option("--ref", "ref_path", default=None, type=click.Path(exists=True, dir_okay=False))
@click.option("--json", "as_json", is_flag=True)
def decode_cmd(in_path, out_path, ref_path, as_json):
    """Reconstruct a tensor from a .sif bitstream."""

    def go():
        from .codec import decode, deserialize
        from .errors import ConfigError
        from .tensor import load_tensor, save_tensor

        with open(in_path, "rb") as f:
            p = deserialize(f.read())
        y = decode(p)
        save_tensor(y, out_path)
        rows, cols = int(y.shape[0]), int(y.shape[1])
        info = {"rows": rows, "cols": cols}
        if ref_path:
            ref = load_tensor(ref_path)
            if tuple(ref.shape) != (rows, cols):
                raise ConfigError("--ref tensor shape does not match decoded tensor")
            # report-only statistics, reduced on the host in the reference's order
            err = np.abs(ref.cpu().numpy().reshape(-1).astype(np.float64) -
                         y.cpu().numpy().reshape(-1).astype(np.float64))
            info["max_abs_error"] = float(err.max())
            info["mean_abs_error"] = float(err.mean())
        if as_json:
            click.echo(json.dumps(info, indent=2))
        else:
            msg = f"decoded {rows}x{cols} tensor to {out_path}"
            if ref_path:
                msg += f" (max err {info['max_abs_error']:.6g}, mean err {info['mean_abs_error']:.6g})"
            click.echo(msg)

    _run(go)


@main.command("stats")
@click.option("--in", "in_path", required=True, type=click.Path(exists=True, dir_okay=False))
@click.option("--json", "as_json", is_flag=True)
def stats_cmd(in_path, as_json):
    """Payload statistics of a .sif bitstream."""

    def go():
        from .stats import stats

        with open(in_path, "rb") as f:
            info = stats(f.read())
        if as_json:
            click.echo(json.dumps(info, indent=2))
        else:
            rows, cols = info["shape"]
            click.echo(f"{rows}x{cols}, nnz {info['nonzeros']} (sparsity {info['actual_sparsity']:.3f})")
            click.echo(f"exact {info['payload_bits_exact']} bits, upper bound {info['payload_bits_upper_bound']} bits, "
                       f"{info['bits_per_element']:.3f} bits/element")
            for b in info["blocks"]:
                click.echo(f"  {b['plane']} block {b['index']}: nnz={b['nnz']} q={b['q']} "
                           f"o={b['scale']:.6g} v_min={b['v_min']:.6g}")

    _run(go)


@main.command("calibrate")
@click.option("--rows", type=int, default=1024, show_default=True)
@click.option("--cols", type=int, default=196, show_default=True)
@click.option("--batch", type=int, default=64, show_default=True)
@click.option("--kind", type=click.Choice(["resnet", "llm"]), default="resnet", show_default=True)
@click.option("--out", "out_path", required=True, type=click.Path(dir_okay=False))
@click.option("--json", "as_json", is_flag=True)
def calibrate_cmd(rows, cols, batch, kind, out_path, as_json):
    """Measure a DeviceTimeModel (profiles.py schema) for the planner's --timemodel."""

    def go():
        from .timemodel import calibrate

        m = calibrate(rows=rows, cols=cols, batch=batch, kind=0 if kind == "resnet" else 1)
        m.save(out_path)
        if as_json:
            click.echo(json.dumps(m.to_dict(), indent=2))
        else:
            click.echo(f"wrote time model ({rows}x{cols} x{batch} {kind}) to {out_path}")

    _run(go)


if __name__ == "__main__":
    main()
