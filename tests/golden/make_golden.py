"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--big]

It imports hjsvd from /root/reference/pkg/src (read-only) and records, for
seeded inputs that numpy regenerates identically anywhere
(np.random.default_rng(seed).standard_normal), the reference's outputs as
SHA-256 digests of the raw float64 bytes (Fortran order) plus the scalar
results, telemetry and (small cases) the full sigma vectors.  Nothing in the
GPU tests, smoke() or bench.py reads /root/reference; they read these files.

Reference anchors: drive solver.py:179-269; rotation_tc _kernels.py:128-173;
dot_chunked _kernels.py:32-59; stepper strategies.py:41-72;
sort_diagonal solver.py:97-110.
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import hjsvd  # noqa: E402
from hjsvd import _kernels  # noqa: E402

from tests.golden.inputs import make_case_input  # noqa: E402


def digest(a):
    if a is None:
        return None
    a = np.asarray(a, dtype="<f8")
    return hashlib.sha256(a.tobytes(order="F")).hexdigest()


def fhex(x):
    return float(x).hex()


# (name, n, r, p, seed, kind, cfg-overrides)
DRIVE_CASES = [
    ("diag2", 2, 2, 1, 0, "diag21", {}),
    ("shear_def", 2, 2, 2, 0, "shear11", {}),
    ("shear_indef", 2, 2, 1, 0, "shear21", {}),
    ("n8_p4", 8, 8, 4, 6, "gauss", {}),
    ("n16_p7", 16, 16, 7, 5, "gauss", {}),
    ("n16x8_p4", 16, 8, 4, 3, "gauss", {}),
    ("n16_nosort", 16, 16, 6, 4, "gauss", {"sort": False}),
    ("n16_max1", 16, 16, 6, 4, "gauss", {"max_sweeps": 1}),
    ("n16_noskip", 16, 16, 6, 4, "gauss", {"use_rel_orth_skip": False}),
    ("n16_nov", 16, 16, 6, 4, "gauss", {"accumulate_v": False}),
    ("n24_rowcyc", 24, 24, 10, 2, "gauss", {"schedule": "row-cyclic"}),
    ("n24_modulus", 24, 24, 10, 2, "gauss", {}),
    ("n32_p12", 32, 32, 12, 9, "gauss", {}),
    ("n32_chunk7", 32, 32, 12, 9, "gauss", {"chunk": 7}),
    ("n64_p32", 64, 64, 32, 0, "gauss", {}),
    ("n96x64_p20", 96, 64, 20, 3, "gauss", {}),
    ("n100_p50_chunk32", 100, 100, 50, 11, "gauss", {}),
    ("n128_J_I", 128, 128, 128, 1, "gauss", {}),
    ("n128_J_minus", 128, 128, 0, 1, "gauss", {}),
    ("n256_p128", 256, 256, 128, 0, "gauss", {}),
    ("n256_graded", 256, 256, 128, 0, "graded12", {}),
    ("n512_p384", 512, 512, 384, 0, "gauss", {}),
    ("n1000_p500", 1000, 1000, 500, 4, "gauss", {}),
]

BIG_CASES = [
    ("n1024_J_I", 1024, 1024, 1024, 0, "gauss", {"workers": 8}),
    ("n2048_graded", 2048, 2048, 1024, 0, "graded10", {"workers": 8}),
    ("n2048_p1024", 2048, 2048, 1024, 0, "gauss", {"workers": 8}),
]


def run_drive(case):
    name, n, r, p, seed, kind, over = case
    G = make_case_input(n, r, seed, kind)
    J = hjsvd.SignatureVector.from_p(r, p)
    cfg = hjsvd.SolverConfig(**over)
    t0 = time.perf_counter()
    res = hjsvd.drive(G, J, cfg)
    wall = time.perf_counter() - t0
    rec = {
        "name": name, "n": n, "r": r, "p": p, "seed": seed, "kind": kind,
        "cfg": over,
        "sigma": digest(res.sigma), "lam": digest(res.lam),
        "U": digest(res.U), "Vinv_t": digest(res.Vinv_t),
        "sweeps_used": res.sweeps_used, "stop_reason": res.stop_reason,
        "rotations": res.rotations, "skips": res.skips,
        "telemetry": [[int(a), int(b), int(c), fhex(d)]
                      for a, b, c, d in res.telemetry],
        "wall_s_reference": wall,
    }
    if r <= 256:
        rec["sigma_hex"] = [fhex(x) for x in res.sigma]
    # residuals the north star names, for the reference's own result
    Jm = J.signs.astype(float)
    V = hjsvd.recover_V(res.Vinv_t, J) if res.Vinv_t is not None else None
    rec["dU"] = float(np.linalg.norm(np.eye(r) - res.U.T @ res.U))
    if V is not None:
        rec["VtJV"] = float(np.linalg.norm(V.T @ (Jm[:, None] * V) - np.diag(Jm))
                            / np.linalg.norm(V) ** 2)
        recon = (res.U * res.sigma) @ V.T
        rec["recon"] = float(np.linalg.norm(G - recon) / np.linalg.norm(G))
    return rec, res


def rotation_cases():
    rng = np.random.default_rng(1234)
    out = []
    specials = [
        (1.0, 2.0, 0.5, -1), (1.0, 1.0, 0.5, -1), (2.0, 1.0, -0.5, 1),
        (1.0, 2.0, 0.0, -1), (1.0, 1.0, -1.5, 1), (1.0, 1.0, 1e-10, -1),
        (1.0, 3.0, 1e-9, -1), (5.0, 5.0, -5.0 + 1e-12, 1), (1e300, 1e-300, 1.0, -1),
        (4.0, 9.0, 5.999999, 1), (4.0, 9.0, -6.5, 1),
    ]
    for a_ii, a_jj, a_ij, hyp in specials:
        out.append((a_ii, a_jj, a_ij, hyp))
    for _ in range(3000):
        a_ii = 10.0 ** rng.uniform(-8, 8)
        a_jj = 10.0 ** rng.uniform(-8, 8) if rng.random() < 0.5 else a_ii * (1 + rng.uniform(-1e-6, 1e-6))
        rho = rng.uniform(-1, 1) * (10.0 ** rng.uniform(-12, 0))
        a_ij = rho * np.sqrt(a_ii * a_jj)
        hyp = -1 if rng.random() < 0.5 else 1
        out.append((a_ii, a_jj, a_ij, hyp))
    recs = []
    for a_ii, a_jj, a_ij, hyp in out:
        t, c, st = _kernels.rotation_tc(a_ii, a_jj, a_ij, hyp)
        recs.append([fhex(a_ii), fhex(a_jj), fhex(a_ij), int(hyp), fhex(t),
                     fhex(c), int(st)])
    return recs


def dot_cases():
    recs = []
    rng = np.random.default_rng(99)
    for length in [1, 2, 3, 31, 32, 33, 63, 64, 65, 100, 257, 1000, 1024, 4097]:
        for chunk in [1, 2, 7, 32, 33]:
            x = rng.standard_normal(length)
            y = rng.standard_normal(length)
            seedx = None
            v = _kernels.dot_chunked(x, y, chunk)
            recs.append([length, chunk, digest(x), digest(y), fhex(v)])
            del seedx
    return recs


def dot_vectors():
    """Regenerate the exact vectors of dot_cases (same rng stream)."""
    rng = np.random.default_rng(99)
    out = []
    for length in [1, 2, 3, 31, 32, 33, 63, 64, 65, 100, 257, 1000, 1024, 4097]:
        for chunk in [1, 2, 7, 32, 33]:
            x = rng.standard_normal(length)
            y = rng.standard_normal(length)
            out.append((length, chunk, x, y))
    return out


def stepper_cases():
    recs = {}
    for r in [2, 4, 6, 8, 12, 16, 64]:
        S = hjsvd.stepper_init(r)
        seq = []
        for _ in range(3 * r):
            seq.append([list(map(int, S.iblk)), list(map(int, S.jblk))])
            hjsvd.stepper_advance_all(S)
        recs[str(r)] = seq
    return recs


def sort_cases():
    recs = []
    rng = np.random.default_rng(7)
    for r, p in [(4, 2), (3, 3), (10, 4), (33, 10), (64, 0), (64, 64), (257, 100)]:
        d = rng.integers(1, 6, size=r).astype(float)  # many ties
        D = hjsvd.DiagonalPackageVector(d.copy(), np.arange(r, dtype=np.int64),
                                        np.array([1] * p + [-1] * (r - p), np.int64), p)
        hjsvd.sort_diagonal(D)
        recs.append([r, p, list(map(float, d)), list(map(int, D.rho))])
    return recs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also n=1024/2048 cases")
    args = ap.parse_args()
    drives = []
    for case in DRIVE_CASES + (BIG_CASES if args.big else []):
        rec, res = run_drive(case)
        drives.append(rec)
        print(f"{rec['name']}: sweeps={rec['sweeps_used']} {rec['stop_reason']} "
              f"rot={rec['rotations']} wall={rec['wall_s_reference']:.2f}s",
              flush=True)
        if case[1] >= 1024:
            np.save(os.path.join(HERE, f"sigma_{case[0]}.npy"), res.sigma)
    out = {
        "generator": "tests/golden/make_golden.py",
        "reference": "hjsvd 0.1.0 at /root/reference/pkg/src",
        "numpy": np.__version__,
        "drive": drives,
        "rotation": rotation_cases(),
        "dot": dot_cases(),
        "stepper": stepper_cases(),
        "sort": sort_cases(),
    }
    path = os.path.join(HERE, "golden_big.json" if args.big else "golden.json")
    if args.big:
        out = {"generator": out["generator"], "reference": out["reference"],
               "numpy": out["numpy"], "drive": drives[len(DRIVE_CASES):]}
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path)


if __name__ == "__main__":
    main()
