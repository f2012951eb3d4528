"""Command-line front end, as the reference's (/root/reference/pkg/src/hjsvd/
cli.py): ``gen``, ``factor``, ``hsvd``, ``eig`` and ``bench`` with the same
files (GJH1 bundles, CSV manifests and RunRecord rows), arguments and exit
codes, plus the B200 flags --mode, --block-cols and --shards.

    python -m paper_1008_1371_b200.cli gen --n 512 --seed 1 --out BUNDLE
    python -m paper_1008_1371_b200.cli eig --in BUNDLE --out RESULT [--mode block]

gen/factor run the GPU factory (factory.py: double-double generator and
Bunch-Parlett, bit-identical to the reference's).  The strategy lab
(check-strategy) is outside this package's scope.
"""

import argparse
import os
import sys
import time
from dataclasses import dataclass, fields

import numpy as np

from .errors import DefinitenessLostError, NumericalSingularityError, ShapeError
from .factory import SpectrumSpec, bunch_parlett_factor, generate_factor_pair
from .linalg import SignatureVector, orthonormality_distance
from .matio import read_csv_matrix, read_gjh, write_csv_matrix, write_gjh
from .solver import SolverConfig, border, drive, recover_V, strip_bordered

EXIT_OK = 0
EXIT_FAIL = 1
EXIT_USAGE = 2
EXIT_IO = 3
EXIT_SINGULAR = 4
EXIT_DEFINITENESS = 5
EXIT_NONCONVERGENCE = 6


@dataclass
class RunRecord:
    """One solver run, one CSV row (cli.py:36-59)."""

    n: int
    r: int
    p: int
    sweeps: int
    stop_reason: str
    wall_time: float
    max_rel_eig_err: float
    dU: float
    rotations: int
    skips: int
    sorting_enabled: bool

    @classmethod
    def header(cls):
        return ",".join(f.name for f in fields(cls))

    def row(self):
        return ",".join(f"{getattr(self, f.name):.17g}"
                        if isinstance(getattr(self, f.name), float)
                        else str(getattr(self, f.name)) for f in fields(self))


def write_records(path, records):
    with open(path, "w") as fh:
        fh.write(RunRecord.header() + "\n")
        for rec in records:
            fh.write(rec.row() + "\n")


def read_bundle(path):
    """(G, J, lambda_true or None) of a bundle directory (cli.py:85-90)."""
    G, p = read_gjh(os.path.join(path, "G.gjh"))
    J = SignatureVector.from_p(G.shape[1], p)
    lam_path = os.path.join(path, "lambda_true.csv")
    lam = read_csv_matrix(lam_path).ravel() if os.path.exists(lam_path) else None
    return G, J, lam


def write_bundle(out, bundle):
    """Bundle directory of a generated instance (cli.py:72-82)."""
    os.makedirs(out, exist_ok=True)
    spec = bundle.spec
    p = bundle.factor.J.p
    write_gjh(os.path.join(out, "M.gjh"), bundle.M, p)
    write_gjh(os.path.join(out, "G.gjh"), bundle.factor.G, p)
    write_csv_matrix(os.path.join(out, "lambda_true.csv"), bundle.lambda_true[np.newaxis, :])
    with open(os.path.join(out, "manifest.csv"), "w") as fh:
        fh.write("seed,n,a,p\n")
        fh.write(f"{spec.seed},{spec.n},{spec.a:.17g},{p}\n")


def cmd_gen(args):
    """cli.py:92-98: generate a test bundle (GPU factory)."""
    spec = SpectrumSpec(args.n, args.a, args.seed, args.pos_count)
    bundle = generate_factor_pair(spec)
    write_bundle(args.out, bundle)
    print(f"gen: wrote bundle to {args.out} (n={spec.n}, a={spec.a}, "
          f"seed={spec.seed}, p={bundle.factor.J.p})")
    return EXIT_OK


def cmd_factor(args):
    """cli.py:101-106: factor a symmetric GJH1 matrix (GPU Bunch-Parlett)."""
    M, _ = read_gjh(args.infile)
    pair = bunch_parlett_factor(M)
    write_gjh(args.out, pair.G, pair.J.p)
    print(f"factor: wrote {args.out} (n={M.shape[0]}, p={pair.J.p})")
    return EXIT_OK


def cmd_bench(args):
    """cli.py:198-222: sweep/time/error table across orders, inertias and
    sorting, on GPU-generated bundles (plus --mode)."""
    orders = [int(x) for x in args.orders.split(",")]
    records = []
    for n in orders:
        if n % 2 != 0:
            raise ShapeError("bench orders must be even")
        for p in (0, max(1, n // 16), n // 2):
            bundle = generate_factor_pair(SpectrumSpec(n, args.a, args.seed, pos_count=p))
            for sort in (True, False):
                cfg = SolverConfig(workers=args.workers, sort=sort, mode=args.mode)
                for _ in range(args.repeats):
                    t0 = time.perf_counter()
                    result = drive(bundle.factor.G, bundle.factor.J, cfg)
                    wall = time.perf_counter() - t0
                    lt = np.sort(bundle.lambda_true)
                    err = float(np.max(np.abs(np.sort(result.lam) - lt) / np.abs(lt)))
                    records.append(RunRecord(n, n, p, result.sweeps_used, result.stop_reason,
                                             wall, err, orthonormality_distance(result.U),
                                             result.rotations, result.skips, sort))
    write_records(args.out, records)
    print(f"bench: wrote {len(records)} rows to {args.out}")
    return EXIT_OK


def solver_config(args):
    return SolverConfig(max_sweeps=args.max_sweeps,
                        accumulate_v=not args.no_accumulate_v,
                        workers=args.workers, schedule=args.schedule,
                        sort=not args.no_sort, mode=args.mode,
                        block_cols=args.block_cols)


def run_solve(args):
    """Solve one bundle and write the result directory (cli.py:118-158)."""
    G, J, lam_true = read_bundle(args.infile)
    n, r = G.shape
    p_orig = J.p
    info = None
    if r % 2 != 0:
        if not args.border:
            raise ShapeError("r is odd; rerun with --border")
        G, J, info = border(G, J, r + 1, max(n + 1, r + 1))
    cfg = solver_config(args)
    t0 = time.perf_counter()
    if args.shards > 1:
        from .sharded import drive_local_shards
        result = drive_local_shards(G, J, cfg, nshards=args.shards)
    else:
        result = drive(G, J, cfg)
    wall = time.perf_counter() - t0
    if info is not None:
        result = strip_bordered(result, info)
    err = float("nan")
    if lam_true is not None:
        lt = np.sort(lam_true)
        err = float(np.max(np.abs(np.sort(result.lam) - lt) / np.abs(lt)))
    dU = orthonormality_distance(result.U)
    rec = RunRecord(n, r, p_orig, result.sweeps_used, result.stop_reason, wall, err,
                    dU, result.rotations, result.skips, cfg.sort)
    os.makedirs(args.out, exist_ok=True)
    write_csv_matrix(os.path.join(args.out, "sigma.csv"), result.sigma[np.newaxis, :])
    write_csv_matrix(os.path.join(args.out, "lambda.csv"), result.lam[np.newaxis, :])
    write_gjh(os.path.join(args.out, "U.gjh"), result.U, p_orig)
    if result.Vinv_t is not None:
        Jout = SignatureVector.from_p(result.Vinv_t.shape[1], p_orig)
        write_gjh(os.path.join(args.out, "V.gjh"), recover_V(result.Vinv_t, Jout), Jout.p)
    write_records(os.path.join(args.out, "record.csv"), [rec])
    print(f"{args.command}: n={n} r={r} sweeps={result.sweeps_used} "
          f"stop={result.stop_reason} wall={wall:.3f}s "
          f"max_rel_eig_err={err:.3e} dU={dU:.3e}")
    return EXIT_NONCONVERGENCE if result.stop_reason == "max_sweeps" else EXIT_OK


def build_parser():
    ap = argparse.ArgumentParser(prog="hsvd-b200",
                                 description="B200 hyperbolic SVD solver (hjsvd drop-in)")
    sub = ap.add_subparsers(dest="command", required=True)
    sp = sub.add_parser("gen", help="generate a test bundle")
    sp.add_argument("--n", type=int, required=True)
    sp.add_argument("--a", type=float, default=20.0)
    sp.add_argument("--seed", type=int, required=True)
    sp.add_argument("--pos-count", dest="pos_count", type=int, default=None)
    sp.add_argument("--out", required=True)
    sp.set_defaults(func=cmd_gen)
    sp = sub.add_parser("factor", help="factor a symmetric GJH1 matrix")
    sp.add_argument("--in", dest="infile", required=True)
    sp.add_argument("--out", required=True)
    sp.set_defaults(func=cmd_factor)
    sp = sub.add_parser("bench", help="sweep/time/error table across configs")
    sp.add_argument("--orders", required=True, help="comma-separated even orders")
    sp.add_argument("--a", type=float, default=20.0)
    sp.add_argument("--seed", type=int, required=True)
    sp.add_argument("--repeats", type=int, default=1)
    sp.add_argument("--workers", type=int, default=1)
    sp.add_argument("--mode", choices=("pointwise", "block"), default="pointwise")
    sp.add_argument("--out", required=True)
    sp.set_defaults(func=cmd_bench)
    for name in ("hsvd", "eig"):
        sp = sub.add_parser(name, help=f"run the {name} solver on a bundle")
        sp.add_argument("--in", dest="infile", required=True)
        sp.add_argument("--out", required=True)
        sp.add_argument("--no-sort", dest="no_sort", action="store_true")
        sp.add_argument("--no-accumulate-v", dest="no_accumulate_v", action="store_true")
        sp.add_argument("--max-sweeps", type=int, default=30)
        sp.add_argument("--workers", type=int, default=1)
        sp.add_argument("--schedule", choices=("modulus", "row-cyclic"), default="modulus")
        sp.add_argument("--border", action="store_true",
                        help="embed odd-r factors by a synthetic +1 column")
        sp.add_argument("--mode", choices=("pointwise", "block"), default="pointwise",
                        help="pointwise: bit-exact with hjsvd; block: FP64 tensor cores")
        sp.add_argument("--block-cols", dest="block_cols", type=int, default=32)
        sp.add_argument("--shards", type=int, default=1,
                        help="block mode: slot shards driven from this process")
        sp.set_defaults(func=run_solve)
    return ap


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ShapeError, NotImplementedError) as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except NumericalSingularityError as exc:
        print(f"numerical singularity: {exc}", file=sys.stderr)
        return EXIT_SINGULAR
    except DefinitenessLostError as exc:
        print(f"definiteness lost: {exc}", file=sys.stderr)
        return EXIT_DEFINITENESS
    except OSError as exc:
        print(f"I/O error: {exc}", file=sys.stderr)
        return EXIT_IO
    except ValueError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
