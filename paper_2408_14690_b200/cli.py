"""GPU backend for the reference CLI's ``bench`` subcommand (cli.py:272-290,
parser cli.py:362-370): same flags, same TSV columns

    sparsity  median_ns  min_ns  dense_median_ns  speedup  weight_bytes

(cells formatted like cli.py:86-89, ``%.9g`` for floats), the same optional
``--out`` file plus ``<out>.manifest.json`` (cli.py:59-71), and the same exit
codes for invalid arguments (ValueError -> 2, OSError -> 3, cli.py:375-387).
Timing is the device sweep of :func:`kernel.bench_gemv` (CUDA events,
oracle-checked reps); ``--dtype bf16`` streams bf16 rows.

    python -m paper_2408_14690_b200.cli bench --rows 4096 --cols 14336
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

EXIT_OK, EXIT_INVALID, EXIT_IO = 0, 2, 3


def _fmt_cell(c) -> str:
    if isinstance(c, float):
        return f"{c:.9g}"
    return str(c)


def _emit_table(headers, rows, out: str | None) -> None:
    text = "\n".join(["\t".join(headers)] + ["\t".join(_fmt_cell(c) for c in r) for r in rows]) + "\n"
    if out:
        Path(out).write_text(text)
    else:
        sys.stdout.write(text)


def _csv_floats(text: str) -> list[float]:
    try:
        return [float(tok) for tok in text.split(",") if tok.strip() != ""]
    except ValueError:
        raise ValueError(f"expected a comma-separated list of numbers, got {text!r}") from None


def _write_manifest(target: Path, command: str, seed: int, params: dict, outputs: list[str]) -> None:
    from . import __version__
    manifest = {"tool": "actsparse", "version": __version__, "backend": "teal_b200", "subcommand": command,
                "seed": seed, "parameters": params, "inputs": [], "outputs": outputs,
                "created_unix": time.time()}
    target.write_text(json.dumps(manifest, indent=2, sort_keys=True) + "\n")


def cmd_bench(args) -> int:
    from .kernel import bench_gemv
    from .tensor import RngStream
    bpe = 2 if args.dtype == "bf16" else 4
    result = bench_gemv(args.rows, args.cols, _csv_floats(args.sparsities), args.reps, args.warmup,
                        RngStream(args.seed), bytes_per_element=bpe)
    rows = [(pt.sparsity, pt.median_ns, pt.min_ns, result.dense_median_ns,
             result.dense_median_ns / pt.median_ns, pt.traffic.weight_bytes_sparse) for pt in result.points]
    _emit_table(("sparsity", "median_ns", "min_ns", "dense_median_ns", "speedup", "weight_bytes"), rows, args.out)
    if args.out:
        _write_manifest(Path(args.out + ".manifest.json"), "bench", args.seed,
                        {"rows": args.rows, "cols": args.cols, "sparsities": args.sparsities,
                         "reps": args.reps, "warmup": args.warmup, "dtype": args.dtype}, [args.out])
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="teal_b200", description="B200 backend of the actsparse CLI")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bench", help="sparse GEMV latency/traffic benchmark (GPU)")
    p.add_argument("--seed", type=int, default=0, help="random seed (default 0)")
    p.add_argument("--format", choices=("tsv",), default="tsv", help="table format (default tsv)")
    p.add_argument("--rows", type=int, default=4096)
    p.add_argument("--cols", type=int, default=14336)
    p.add_argument("--sparsities", default="0,0.25,0.5,0.9")
    p.add_argument("--reps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--dtype", choices=("f32", "bf16"), default="f32",
                   help="weight element type streamed (the reference is fp32)")
    p.add_argument("--out")
    p.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INVALID
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
