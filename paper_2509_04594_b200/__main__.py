"""``python -m paper_2509_04594_b200 run ...`` — the reference's ``tilebench run``
(/root/reference/pkg/src/tilebench/cli.py:61-138) for the GPU backends, with
kernel-only device seconds.

Same flags (``--backends --sizes --trials --seed --tile --warmup --verify
--out``), same records CSV + ``.meta.json`` sidecar (records.py:24-66), same
exit codes (0 ok, 1 trial failure with a ``# aborted:`` marker, 2 bad
configuration; cli.py:110-135), so ``tilebench analyze --in <out>`` consumes
the GPU rows unchanged. ``--verify`` compares the last trial of each pair with
the host CPU product (numpy's BLAS; ``--verify-with cublas``: cuBLAS DGEMM on
the device) against the reference's max_abs_rel_diff bar.
"""
from __future__ import annotations

import argparse
import sys

from .backends import BackendRegistry, TileConfig, cublas_multiply
from .errors import InvalidConfigError, TilebenchError, TrialError
from .harness import RunConfig, RunMetadata, run_trials, write_records


def _csv_ints(text: str) -> tuple[int, ...]:
    try:
        return tuple(int(x) for x in text.split(",") if x.strip())
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers, got {text!r}") from None


def _csv_names(text: str) -> tuple[str, ...]:
    return tuple(x.strip() for x in text.split(",") if x.strip())


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="python -m paper_2509_04594_b200", description=__doc__.splitlines()[0])
    sub = parser.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="execute device-timed trials and write a records CSV")
    run.add_argument("--backends", type=_csv_names, default=("gpu-tiled",), help="comma-separated backend names")
    run.add_argument("--sizes", type=_csv_ints, required=True, help="comma-separated matrix sizes")
    run.add_argument("--trials", type=int, default=30)
    run.add_argument("--seed", type=int, default=0)
    run.add_argument("--tile", type=int, default=32)
    run.add_argument("--warmup", type=int, default=1)
    run.add_argument("--verify", action="store_true", help="check the last product of each pair after timing")
    run.add_argument("--verify-with", choices=("cpu", "cublas"), default="cpu",
                     help="--verify reference: the host CPU product (numpy / BLAS, like the reference's CPU "
                          "oracle check, harness.py:237-243) or cuBLAS DGEMM on the device")
    run.add_argument("--out", required=True, help="records CSV path")
    run.set_defaults(fn=cmd_run)
    return parser


def _host_product(a, b):
    """The CPU product of the trial's own operands (numpy's BLAS on the host):
    an independent reference for ``--verify``, as the reference checks against
    its CPU oracle; not this package's GPU code."""
    import numpy as np

    return np.matmul(np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64))


def cmd_run(args) -> int:
    registry = BackendRegistry()
    config = RunConfig(backends=args.backends, sizes=args.sizes, trials=args.trials, warmup=args.warmup,
                       seed=args.seed, tile=TileConfig(args.tile), verify=args.verify)
    try:
        config.validate(registry)
    except TilebenchError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    records = []

    def progress(name, n, trial, total):
        print(f"{name} n={n} trial {trial + 1}/{total}", file=sys.stderr)

    try:
        verifier = None
        if args.verify:
            verifier = cublas_multiply if args.verify_with == "cublas" else _host_product
        records, meta = run_trials(config, registry, progress=progress, on_record=records.append,
                                   verifier=verifier)
    except TrialError as exc:
        meta = RunMetadata.capture(config, {"clock": "cuda-events kernel-only"})
        write_records(args.out, records, meta, aborted=str(exc))
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except InvalidConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    write_records(args.out, records, meta)
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
