"""Goldens of the factorization front end, made by running the REAL
reference (hjsvd.factory.bunch_parlett_factor, factory.py:270-282) in the
build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_factor.py

Records SHA-256 digests of G (Fortran order), perm and signs, p and the
number of 2x2 pivots, into tests/golden/factor.json; the inputs are seeded
numpy matrices (tests/golden/factor_inputs.py) or reference-generated
spectra stored in factor_inputs.npz.  Nothing on the GPU box reads
/root/reference.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

import hjsvd  # noqa: E402
from digest import digest  # noqa: E402
from factor_inputs import make_input  # noqa: E402

SPECTRA = [(16, 2), (64, 7), (128, 9)]
GEN = [(16, 21, None), (33, 3, None), (64, 17, 10), (100, 23, None), (128, 1, None),
       (40, 3, 0), (24, 5, 24)]
CASES = [("diag", 2, 0), ("offdiag", 2, 0), ("sym", 5, 1), ("sym", 33, 3), ("sym", 200, 4),
         ("sym", 256, 5), ("smalldiag", 100, 6), ("smalldiag", 257, 8), ("ints", 40, 10),
         ("ints", 96, 11)] + [("spectrum", n, s) for n, s in SPECTRA]


def main():
    arrs = {}
    for n, s in SPECTRA:
        M, lam = hjsvd.generate_symmetric(hjsvd.SpectrumSpec(n, 20.0, s))
        arrs[f"M_{n}_{s}"] = M
        arrs[f"lam_{n}_{s}"] = lam
    np.savez_compressed(os.path.join(HERE, "factor_inputs.npz"), **arrs)
    out = []
    for kind, n, seed in CASES:
        M = make_input(kind, n, seed)
        pair = hjsvd.bunch_parlett_factor(M)
        out.append({
            "kind": kind, "n": int(M.shape[0]), "seed": seed,
            "G": digest(pair.G),
            "perm": hashlib.sha256(np.asarray(pair.perm, "<i8").tobytes()).hexdigest(),
            "signs": hashlib.sha256(np.asarray(pair.J.signs, "i1").tobytes()).hexdigest(),
            "p": int(pair.J.p),
        })
        print(kind, n, seed, out[-1]["p"])
    gen = []
    for n, seed, pos in GEN:
        spec = hjsvd.SpectrumSpec(n, 20.0, seed, pos)
        M, lam = hjsvd.generate_symmetric(spec)
        b = hjsvd.generate_factor_pair(spec)
        gen.append({
            "n": n, "seed": seed, "pos_count": pos, "M": digest(M), "lam": digest(lam),
            "bundle_M": digest(b.M), "G": digest(b.factor.G),
            "perm": hashlib.sha256(np.asarray(b.factor.perm, "<i8").tobytes()).hexdigest(),
            "p": int(b.factor.J.p),
        })
        print("gen", n, seed, pos, gen[-1]["p"])
    # the reference's `gen` bundle files, byte for byte
    import tempfile
    from hjsvd.cli import main as ref_cli
    cli = []
    for n, seed, pos in [(48, 5, None), (30, 2, 7)]:
        with tempfile.TemporaryDirectory() as d:
            args = ["gen", "--n", str(n), "--seed", str(seed), "--out", d]
            if pos is not None:
                args += ["--pos-count", str(pos)]
            assert ref_cli(args) == 0
            files = {f: hashlib.sha256(open(os.path.join(d, f), "rb").read()).hexdigest()
                     for f in sorted(os.listdir(d))}
        cli.append({"n": n, "seed": seed, "pos_count": pos, "files": files})
    with open(os.path.join(HERE, "factor.json"), "w") as f:
        json.dump({"reference": "hjsvd.factory.bunch_parlett_factor (factory.py:270-282); "
                                "generate_symmetric / generate_factor_pair (factory.py:104-114, "
                                "285-297)",
                   "singular": {"kind": "ones", "n": 3}, "cases": out, "gen": gen, "cli_gen": cli},
                  f, indent=1)


if __name__ == "__main__":
    main()
