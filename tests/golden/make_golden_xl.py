"""Reference outputs for the BENCHMARKED configurations (BASELINE configs 3
and 5), produced by running the reference's algorithm to completion on the
host CPU.  TEST INFRASTRUCTURE: run in the build container, never on the GPU
box.

    python tests/golden/make_golden_xl.py --workers 6 [--hjsvd]

* The solver is the C oracle (oracle/hsvd_oracle.c), which is pinned bit for
  bit to hjsvd.drive (solver.py:179-269) on every golden in golden.json and
  golden_big.json.  A full hjsvd run at n = 8192 takes hours; the oracle is
  the same IEEE operation sequence, faster.
* With --hjsvd, the stock reference (hjsvd.drive from /root/reference/pkg/src,
  numba) is ALSO run at n = 4096, p = 3072 (config 3), its digests are
  compared with the oracle's, and its wall time is recorded.
* Recorded per case: SHA-256 of sigma / lam / U / V^{-T} (float64, F order),
  sweeps, stop reason, rotations, skips, telemetry, the north-star residuals
  of the reference's own result, the wall time and thread count.  The sigma
  vector is saved as sigma_<name>.npy (lam follows from the input signs).

Writes tests/golden/golden_xl.json.
"""

import argparse
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.golden.inputs import make_case_input  # noqa: E402

XL_CASES = [
    # name, n, r, p, seed, kind
    ("n4096_p3072", 4096, 4096, 3072, 0, "gauss"),   # BASELINE config 3
    ("n8192_p4096", 8192, 8192, 4096, 0, "gauss"),   # BASELINE config 5
]


def digest(a):
    if a is None:
        return None
    a = np.asarray(a, dtype="<f8")
    return hashlib.sha256(a.tobytes(order="F")).hexdigest()


def residuals(G, U, sigma, Vinv_t, signs):
    s = signs.astype(np.float64)
    r = U.shape[1]
    out = {"dU": float(np.linalg.norm(U.T @ U - np.eye(r)))}
    V = s[:, None] * Vinv_t * s[None, :]
    out["VtJV"] = float(np.linalg.norm(V.T @ (s[:, None] * V) - np.diag(s))
                        / np.linalg.norm(V) ** 2)
    out["recon"] = float(np.linalg.norm(G - (U * sigma) @ V.T) / np.linalg.norm(G))
    return out


def record(name, n, r, p, seed, kind, res, wall, workers, solver):
    return {
        "name": name, "n": n, "r": r, "p": p, "seed": seed, "kind": kind,
        "solver": solver, "threads": workers, "wall_s": wall,
        "sigma": digest(res.sigma), "lam": digest(res.lam),
        "U": digest(res.U), "Vinv_t": digest(res.Vinv_t),
        "sweeps_used": int(res.sweeps_used), "stop_reason": res.stop_reason,
        "rotations": int(res.rotations), "skips": int(res.skips),
        "telemetry": [[int(a), int(b), int(c), float(d).hex()]
                      for a, b, c, d in res.telemetry],
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--only", default=None, help="comma-separated case names")
    ap.add_argument("--hjsvd", action="store_true",
                    help="also run stock hjsvd.drive at n=4096 and compare")
    args = ap.parse_args()
    path = os.path.join(HERE, "golden_xl.json")
    out = {"generator": "tests/golden/make_golden_xl.py", "cases": [],
           "host": {"cpu": platform.processor() or platform.machine(),
                    "cores_visible": len(os.sched_getaffinity(0))}}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f)
    done = {c["name"]: c for c in out["cases"]}
    O.build()
    for name, n, r, p, seed, kind in XL_CASES:
        if args.only and name not in args.only.split(","):
            continue
        G = make_case_input(n, r, seed, kind)
        signs = np.array([1] * p + [-1] * (r - p), np.int8)
        t0 = time.perf_counter()
        res = O.drive(G, signs, p, workers=args.workers)
        wall = time.perf_counter() - t0
        rec = record(name, n, r, p, seed, kind, res, wall, args.workers,
                     "oracle/hsvd_oracle.c (bit-exact restatement of hjsvd.drive)")
        print(f"{name}: oracle sweeps={res.sweeps_used} {res.stop_reason} "
              f"rot={res.rotations} skips={res.skips} wall={wall:.1f}s", flush=True)
        rec.update(residuals(G, res.U, res.sigma, res.Vinv_t, signs))
        np.save(os.path.join(HERE, f"sigma_{name}.npy"), res.sigma)
        prev = done.get(name, {})
        if "hjsvd" in prev:
            rec["hjsvd"] = prev["hjsvd"]
        done[name] = rec
        out["cases"] = list(done.values())
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
        del res
    if args.hjsvd:
        sys.path.insert(0, "/root/reference/pkg/src")
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
        import hjsvd
        name, n, r, p, seed, kind = XL_CASES[0]
        G = make_case_input(n, r, seed, kind)
        J = hjsvd.SignatureVector.from_p(r, p)
        # JIT warm-up on a small case so the wall time is the solve's
        hjsvd.drive(make_case_input(64, 64, 0, "gauss"), hjsvd.SignatureVector.from_p(64, 32))
        t0 = time.perf_counter()
        res = hjsvd.drive(G, J, hjsvd.SolverConfig(workers=args.workers))
        wall = time.perf_counter() - t0
        ref = record(name, n, r, p, seed, kind, res, wall, args.workers,
                     "hjsvd.drive (stock reference, numba)")
        orc = done[name]
        same = all(ref[k] == orc[k] for k in ("sigma", "lam", "U", "Vinv_t",
                                              "sweeps_used", "rotations", "skips",
                                              "telemetry"))
        print(f"{name}: hjsvd wall={wall:.1f}s bit-identical to oracle: {same}", flush=True)
        orc["hjsvd"] = {"wall_s": wall, "threads": args.workers,
                        "bit_identical_to_oracle": same}
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
