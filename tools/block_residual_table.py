"""Block mode vs the reference: sigma agreement, residual ratios and sweeps
for every block-mode parity case and the five BASELINE configs.  Prints a
markdown table (committed as profiles/r02_block_residual_ratios.md).

Reference results: the C oracle (bit-exact with hjsvd) run here for the
small cases; tests/golden/golden_big.json / golden_xl.json (reference runs
to completion on the build host) for n >= 1024.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import paper_1008_1371_b200 as H  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.block_metrics import sigma_class_reldiff  # noqa: E402
from tests.golden.inputs import make_case_input  # noqa: E402
from tests.test_gpu_xl import residuals_gpu  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")

SMALL = [
    # n, r, p, seed, kind, b, label
    (64, 64, 32, 0, "gauss", 16, ""),
    (96, 64, 20, 3, "gauss", 16, ""),
    (128, 128, 64, 1, "gauss", 32, ""),
    (128, 128, 128, 1, "gauss", 16, ""),
    (256, 256, 128, 0, "gauss", 32, "config 1"),
    (256, 256, 128, 0, "graded12", 32, ""),
    (256, 256, 0, 5, "gauss", 32, ""),
    (512, 512, 384, 0, "gauss", 32, ""),
    (520, 512, 200, 2, "gauss", 32, ""),
    (1000, 1000, 500, 4, "gauss", 32, "padded"),
    (520, 514, 200, 2, "gauss", 32, "padded"),
    (96, 70, 30, 1, "gauss", 16, "padded"),
]
BIG = [("n1024_J_I", "golden_big.json", "config 2"), ("n2048_graded", "golden_big.json", "config 4"),
       ("n2048_p1024", "golden_big.json", ""), ("n4096_p3072", "golden_xl.json", "config 3"),
       ("n8192_p4096", "golden_xl.json", "config 5 (bench)")]


ROT = os.environ.get("ROT", "fast")


def row(label, n, r, p, kind, b, G, signs, ref_sigma, ref_lam, ref_res, ref_sweeps):
    J = H.SignatureVector(signs, p)
    res = H.drive(G, J, H.SolverConfig(mode="block", block_cols=b, block_rotation=ROT))
    d = sigma_class_reldiff(res.sigma, res.lam, ref_sigma, ref_lam)
    rb = residuals_gpu(G, res.U, res.sigma, res.Vinv_t, signs)
    rat = {k: rb[k] / ref_res[k] for k in rb}
    print(f"| {n}x{r} p={p} {kind} b={b} {label} | {d:.1e} | "
          + " | ".join(f"{rb[k]:.2e} / {ref_res[k]:.2e} = **{rat[k]:.2f}**" for k in ("dU", "VtJV", "recon"))
          + f" | {res.sweeps_used} / {ref_sweeps} |", flush=True)
    return rat


def main():
    print(f"block_rotation = {ROT}\n")
    print("| case | max sigma rel diff (per class) | dU block/ref | VtJV block/ref | recon block/ref | sweeps block/ref |")
    print("|---|---|---|---|---|---|")
    worst = {}
    for n, r, p, seed, kind, b, label in SMALL:
        G = make_case_input(n, r, seed, kind)
        signs = np.array([1] * p + [-1] * (r - p), np.int8)
        ref = O.drive(G, signs, p)
        rr = residuals_gpu(G, ref.U, ref.sigma, ref.Vinv_t, signs)
        rat = row(label, n, r, p, kind, b, G, signs, ref.sigma, ref.lam, rr, ref.sweeps_used)
        for k, v in rat.items():
            worst[k] = max(worst.get(k, 0.0), v)
    for name, fname, label in BIG:
        with open(os.path.join(GOLD, fname)) as f:
            data = json.load(f)
        cs = {c["name"]: c for c in data.get("cases", data.get("drive", []))}
        if name not in cs:
            continue
        c = cs[name]
        G = make_case_input(c["n"], c["r"], c["seed"], c["kind"])
        signs = np.array([1] * c["p"] + [-1] * (c["r"] - c["p"]), np.int8)
        sig = np.load(os.path.join(GOLD, f"sigma_{name}.npy"))
        ref_res = {"dU": c["dU"], "VtJV": c["VtJV"], "recon": c["recon"]}
        rat = row(label, c["n"], c["r"], c["p"], c["kind"], 32, G, signs, sig,
                  sig ** 2 * signs.astype(np.float64), ref_res, c["sweeps_used"])
        for k, v in rat.items():
            worst[k] = max(worst.get(k, 0.0), v)
    print("\nworst ratios: " + ", ".join(f"{k} {v:.2f}" for k, v in worst.items()))


if __name__ == "__main__":
    main()
