"""The README quick-start example (run from the repo root: PYTHONPATH=. python tools/readme_example.py)."""
import numpy as np
import paper_1008_1371_b200 as hjsvd                   # instead of: import hjsvd

G = np.random.default_rng(0).standard_normal((1024, 1024))
J = hjsvd.SignatureVector.from_p(1024, 512)
res = hjsvd.drive(G, J)                                  # bit-identical to hjsvd.drive
res = hjsvd.drive(G, J, hjsvd.SolverConfig(mode="block"))   # FP64 tensor cores
V = hjsvd.recover_V(res.Vinv_t, J)

b = hjsvd.generate_factor_pair(hjsvd.SpectrumSpec(2048, 20.0, seed=1))  # GPU factory
lam = np.sort(hjsvd.drive(b.factor.G, b.factor.J, hjsvd.SolverConfig(mode="block")).lam)
print("max rel eig err", np.max(np.abs(lam - b.lambda_true) / np.abs(b.lambda_true)))
