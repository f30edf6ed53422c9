"""``compute`` front end on the GPU path.

    python -m paper_2509_01654_b200 compute data/fr.words --match 1 --mismatch -1 --gap -2 --out data/fr

takes the reference's ``phonsim compute`` arguments (cli.py:75-85), prints the same four lines
(cli.py:184-190), writes the same ``.nwedges`` + manifest files and uses the same exit codes
(cli.py:13: 0 success, 1 usage error, 2 data error, 3 I/O error).  ``--workers`` is accepted and
ignored; ``--device`` picks the GPU, ``--devices 0,1,...`` shares the edge range between several.
``--scheme FILE`` (aligner.py:195-239) with per-pair overrides resolved against ``--inventory`` -- or, as in the
reference (cli.py:167-174), the ``.inventory`` file next to a ``.words`` file -- runs on the packed kernel's
table-driven cell.  Every other ``phonsim`` sub-command works on the finished store and stays with the reference.
"""
from __future__ import annotations

import argparse
import sys

from .engine import compute_all_pairs, preflight_range_check
from .host_types import DEFAULT_CHUNK_SIZE, ComputePlan, DataError, ScoringScheme
import os

from .store import PipelinedEdgeStoreWriter, load_inventory, load_scheme_file, load_words

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_IO = 0, 1, 2, 3


class UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):          # argparse would exit(2): route through the reference's codes
        raise UsageError(message)


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="paper_2509_01654_b200", description="B200 all-pairs Needleman-Wunsch scoring")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("compute", help="score all word pairs into an edge store")
    p.add_argument("words_file", help=".words file from `phonsim ingest`")
    p.add_argument("--match", type=int, default=1)
    p.add_argument("--mismatch", type=int, default=-1)
    p.add_argument("--gap", type=int, default=-1)
    p.add_argument("--scheme", default=None, help="scheme file (match/mismatch/gap + per-pair overrides); overrides --match/--mismatch/--gap")
    p.add_argument("--inventory", default=None, help="inventory sidecar for scheme-file overrides (default: <words_file stem>.inventory)")
    p.add_argument("--workers", type=int, default=1, help="accepted for compatibility, ignored")
    p.add_argument("--chunk-size", type=int, default=DEFAULT_CHUNK_SIZE)
    p.add_argument("--device", type=int, default=0, help="CUDA device index")
    p.add_argument("--devices", default=None, help="comma-separated CUDA device indices to share the work (default: --device)")
    p.add_argument("--out", required=True, help="output prefix for the edge store")
    p.set_defaults(func=cmd_compute)
    return parser


def cmd_compute(args) -> int:
    if args.workers < 1:
        raise UsageError("workers must be positive")
    if args.chunk_size < 1:
        raise UsageError("chunk-size must be positive")
    try:
        devices = [int(d) for d in args.devices.split(",")] if args.devices else [args.device]
    except ValueError:
        raise UsageError("devices must be a comma-separated list of integers") from None
    words = load_words(args.words_file)
    if args.scheme:
        inventory_path = args.inventory
        if inventory_path is None and args.words_file.endswith(".words"):
            guess = args.words_file[: -len(".words")] + ".inventory"
            if os.path.exists(guess):
                inventory_path = guess
        scheme = load_scheme_file(args.scheme, load_inventory(inventory_path) if inventory_path else None)
    else:
        scheme = ScoringScheme(args.match, args.mismatch, args.gap)
    preflight_range_check(words, scheme)            # fail before any output file exists (cli.py:177)
    plan = ComputePlan(n=len(words), chunk_size=args.chunk_size, worker_count=args.workers, scheme=scheme)
    writer = PipelinedEdgeStoreWriter(args.out, words, scheme)
    stats = compute_all_pairs(words, scheme, writer, plan, devices=devices)
    manifest = writer.finalize()
    print(f"computed {stats.edges_written} edges in {stats.wall_time:.2f} s")
    print(f"scores: min {stats.min_score}, max {stats.max_score}, mean {stats.mean_score:.4f}")
    print(f"payload digest {manifest.payload_digest}")
    print(f"wrote {writer.payload_path}")
    return EXIT_OK


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
        return args.func(args)
    except UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except DataError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_DATA
    except ValueError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except (OSError, RuntimeError, MemoryError) as exc:      # I/O and CUDA / device failures
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
