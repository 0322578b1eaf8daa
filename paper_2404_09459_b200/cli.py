"""Command line of the drop-in (reference ``rgsv/cli.py``):
the same subcommands, flags, output formats and exit codes, routed to the
device path.

    python -m paper_2404_09459_b200 gsv     --g1 A.mtx --g2 B.mtx [options]
    python -m paper_2404_09459_b200 compare --g1 A.mtx --g2 B.mtx [options]
    python -m paper_2404_09459_b200 extract --input A.mtx [options]
    python -m paper_2404_09459_b200 bounds  --g1 A.mtx --g2 B.mtx [--k K --oversample P]
    python -m paper_2404_09459_b200 synth   --m M --p P --n N --field real --out-dir DIR
    python -m paper_2404_09459_b200 bench   (--g1 A --g2 B | --m M --p P --n N --field real)

Routing (cli.py:88-176): ``gsv`` -> ``compute_gsv``, ``compare`` ->
``compare``, ``extract`` -> ``extract_basis``, ``bounds`` -> the direct
spectrum, the randomized ``engine._run_pipeline`` bases, the projected pair
Q_i Q_i^T G_i (two DMMA GEMMs per matrix, on the device) and the
certificates of ``bounds.py``. ``--seed`` defaults to ``RGSV_SEED`` and then
0 (cli.py:39-44). One flag is added: ``--power-iters`` (the q of
``ExtractionConfig``; 0, the reference's behaviour, by default).

``synth`` (cli.py:113-132) writes g1.mtx, g2.mtx and the true spectrum of a
``synthetic.synth_gmp`` pair; ``bench`` (cli.py:135-155) runs the timing
harness of this package's ``bench`` module and prints the per-method medians.
Both keep the reference's ``--field`` default ("complex"), which the device
path rejects with a ``validation`` error: pass ``--field real``.
"""

from __future__ import annotations

import argparse
import dataclasses
import os
import sys

from . import io
from .errors import GsvError, ValidationError

# errors.py categories -> process exit codes (cli.py:27-36)
EXIT_CODES = {"parse": 3, "dimension": 4, "validation": 5, "rank": 6, "numerical": 7,
              "infeasible": 8, "degenerate": 9, "recovery": 10}
EXIT_IO = 11


def _seed_of(args) -> int:
    if args.seed is not None:
        return args.seed
    raw = os.environ.get("RGSV_SEED", "0")
    try:
        return int(raw)
    except ValueError:
        raise ValidationError(f"RGSV_SEED must be an integer, got {raw!r}") from None


def _extraction(args):
    from .rangefinder import ExtractionConfig

    return ExtractionConfig(tol=args.tol, blocksize=args.blocksize, seed=_seed_of(args),
                            max_cols=args.max_cols, trim_tol=args.trim_tol,
                            power_iters=args.power_iters)


def _options(args):
    from .engine import GsvOptions

    return GsvOptions(extraction=_extraction(args), classify_tol=args.classify_tol,
                      method=args.method)


def _pair(args):
    from .engine import GmpPair

    return GmpPair(io.read_matrix(args.g1), io.read_matrix(args.g2))


def _run_gsv(args) -> int:
    from .engine import compute_gsv

    io.write_report(compute_gsv(_pair(args), _options(args)), args.output, args.format)
    return 0


def _run_compare(args) -> int:
    from .analysis import compare

    io.write_report(compare(_pair(args), _options(args)), args.output, args.format)
    return 0


def _run_extract(args) -> int:
    from .rangefinder import extract_basis

    io.write_report(extract_basis(io.read_matrix(args.input), _extraction(args)), args.output,
                    args.format)
    return 0


def _run_bounds(args) -> int:
    """cli.py:158-176: certificate of the randomized pipeline against the
    direct spectrum, E = perturbation_bound(pair, projected pair)."""
    from . import engine
    from .bounds import perturbation_bound, projector_bound, quantity_error_bounds
    from .engine import DIRECT, RANDOMIZED, GmpPair, compute_gsv
    from .rangefinder import projected

    pair = _pair(args)
    opts = _options(args)
    direct = compute_gsv(pair, dataclasses.replace(opts, method=DIRECT))
    pl = engine._run_pipeline(pair, dataclasses.replace(opts, method=RANDOMIZED))
    pair_proj = GmpPair(projected(pair.g1, pl.q1), projected(pair.g2, pl.q2))
    e_script = perturbation_bound(pair, pair_proj)
    cert = quantity_error_bounds(direct, e_script, eta=pair.stack_norm2 ** 2)
    io.write_report(cert, args.output, args.format)
    if args.k is not None:
        for which in ("first", "second"):
            bound = projector_bound(pair, direct, args.k, args.oversample, which)
            print(f"projector_bound[{which}] (k={args.k}, oversample={args.oversample}): "
                  f"{bound:.6e}", file=sys.stderr)
    return 0


def _run_synth(args) -> int:
    from pathlib import Path

    from .synthetic import SynthSpec, synth_gmp

    spec = SynthSpec(m=args.m, p=args.p, n=args.n, rank_frac=args.rank_frac,
                     seed=_seed_of(args), field=args.field)
    result = synth_gmp(spec)
    out = Path(args.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    io.write_matrix(out / "g1.mtx", result.pair.g1.t.cpu().numpy())
    io.write_matrix(out / "g2.mtx", result.pair.g2.t.cpu().numpy())
    ext = "json" if args.format == "json" else "csv"
    io.write_report(result.true_spectrum, out / f"truth.{ext}", args.format)
    print(f"wrote {out}/g1.mtx {out}/g2.mtx {out}/truth.{ext} "
          f"(condition_r={result.condition_r:.6g})", file=sys.stderr)
    return 0


def _run_bench(args) -> int:
    from .bench import RunConfig, median_seconds, run_bench
    from .synthetic import SynthSpec

    synth = None
    sizes = (args.m, args.p, args.n)
    if any(v is not None for v in sizes):
        if any(v is None for v in sizes):
            raise ValidationError("--m, --p and --n must be given together")
        synth = SynthSpec(m=args.m, p=args.p, n=args.n, rank_frac=args.rank_frac,
                          seed=_seed_of(args), field=args.field)
    cfg = RunConfig(g1_path=args.g1, g2_path=args.g2, synth=synth, options=_options(args),
                    output=args.output, format=args.format, repetitions=args.reps)
    records = run_bench(cfg)
    io.write_report(records, cfg.output, cfg.format)
    for method, sec in sorted(median_seconds(records).items()):
        print(f"median {method}: {sec:.6f} s", file=sys.stderr)
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="rgsv",
        description="Generalized singular values of a matrix pair by randomized basis "
                    "extraction on a B200, with comparative-analysis quantities and error "
                    "certificates (drop-in for the reference rgsv command line).")
    sub = parser.add_subparsers(dest="command", required=True)

    def pair_inputs(p):
        p.add_argument("--g1", required=True, help="first matrix file (Matrix Market or CSV)")
        p.add_argument("--g2", required=True, help="second matrix file")

    def extraction_flags(p):
        p.add_argument("--tol", type=float, default=None,
                       help="absolute basis-extraction residual target (default 1e-10*||G||_F)")
        p.add_argument("--blocksize", type=int, default=100)
        p.add_argument("--seed", type=int, default=None,
                       help="base seed (default: RGSV_SEED env var, then 0)")
        p.add_argument("--max-cols", type=int, default=None)
        p.add_argument("--trim-tol", type=float, default=1e-12)
        p.add_argument("--power-iters", type=int, default=0,
                       help="power iterations of a fixed-width sketch (extension; default 0)")

    def gsv_flags(p):
        p.add_argument("--method", choices=["randomized", "direct"], default="randomized")
        extraction_flags(p)
        p.add_argument("--classify-tol", type=float, default=1e-10)

    def output_flags(p):
        p.add_argument("-o", "--output", default=None, help="output file (default stdout)")
        p.add_argument("--format", choices=["csv", "json"], default="csv")

    p = sub.add_parser("gsv", help="compute the GSV spectrum of a pair")
    pair_inputs(p), gsv_flags(p), output_flags(p)
    p.set_defaults(func=_run_gsv)

    p = sub.add_parser("compare", help="full comparative-analysis report")
    pair_inputs(p), gsv_flags(p), output_flags(p)
    p.set_defaults(func=_run_compare)

    p = sub.add_parser("extract", help="basis extraction residual history")
    p.add_argument("--input", required=True, help="matrix file")
    extraction_flags(p), output_flags(p)
    p.set_defaults(func=_run_extract)

    p = sub.add_parser("bounds", help="error certificates for a pair")
    pair_inputs(p)
    p.add_argument("--k", type=int, default=None, help="sketch target rank")
    p.add_argument("--oversample", type=int, default=5)
    gsv_flags(p), output_flags(p)
    p.set_defaults(func=_run_bounds)

    p = sub.add_parser("synth", help="generate a synthetic pair with known spectrum")
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--p", type=int, required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--rank-frac", type=float, default=0.6)
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--field", choices=["real", "complex"], default="complex")
    p.add_argument("--out-dir", required=True)
    p.add_argument("--format", choices=["csv", "json"], default="csv")
    p.set_defaults(func=_run_synth)

    p = sub.add_parser("bench", help="time randomized vs direct")
    p.add_argument("--g1", default=None)
    p.add_argument("--g2", default=None)
    p.add_argument("--m", type=int, default=None)
    p.add_argument("--p", type=int, default=None)
    p.add_argument("--n", type=int, default=None)
    p.add_argument("--rank-frac", type=float, default=0.6)
    p.add_argument("--field", choices=["real", "complex"], default="complex")
    p.add_argument("--reps", type=int, default=1)
    gsv_flags(p), output_flags(p)
    p.set_defaults(func=_run_bench)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except GsvError as exc:
        print(f"error: category={exc.category}: {exc}", file=sys.stderr)
        return EXIT_CODES.get(exc.category, 1)
    except OSError as exc:
        print(f"error: category=io: {exc}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
