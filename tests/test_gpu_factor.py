"""GPU: the Bunch-Parlett front end (csrc/hsvd_factor.cu through
hsvd_bp_factor) bit for bit against the reference's goldens
(tests/golden/factor.json), its error behaviour (test_factory.py:103-115),
and the eigen pipeline end to end (test_factory.py:134-139)."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from digest import digest  # noqa: E402
from factor_inputs import make_input  # noqa: E402

import paper_1008_1371_b200 as H  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden", "factor.json")))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c['kind']}-{c['n']}-{c['seed']}")
def test_factor_bit_exact(case):
    M = make_input(case["kind"], case["n"], case["seed"])
    pair = H.bunch_parlett_factor(M)
    assert digest(pair.G) == case["G"]
    assert hashlib.sha256(np.asarray(pair.perm, "<i8").tobytes()).hexdigest() == case["perm"]
    assert hashlib.sha256(np.asarray(pair.J.signs, "i1").tobytes()).hexdigest() == case["signs"]
    assert pair.J.p == case["p"]


def test_factor_known_answers():
    pair = H.bunch_parlett_factor(np.diag([4.0, -1.0]))
    np.testing.assert_array_equal(np.abs(pair.G), np.diag([2.0, 1.0]))
    np.testing.assert_array_equal(pair.J.signs, [1, -1])
    pair = H.bunch_parlett_factor(np.array([[0.0, 1.0], [1.0, 0.0]]))
    s = 1.0 / np.sqrt(2.0)
    np.testing.assert_allclose(np.abs(pair.G), [[s, s], [s, s]], rtol=1e-15)


def test_factor_errors():
    with pytest.raises(H.NumericalSingularityError):
        H.bunch_parlett_factor(np.ones((3, 3)))
    with pytest.raises(ValueError):
        H.bunch_parlett_factor(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(H.ShapeError):
        H.bunch_parlett_factor(np.ones((2, 3)))


def test_factor_residual_large():
    # beyond the golden sizes: M = G J G^T to the reference's tolerance
    n = 1024
    M = make_input("smalldiag", n, 21)
    pair = H.bunch_parlett_factor(M)
    R = pair.G @ np.diag(pair.J.signs.astype(float)) @ pair.G.T
    assert np.linalg.norm(R - M) <= 50.0 * n * H.EPS * np.linalg.norm(M)
    np.testing.assert_array_equal(np.sort(pair.perm), np.arange(n))


@pytest.mark.parametrize("mode", ["pointwise", "block"])
def test_eigen_pipeline_end_to_end(mode):
    npz = np.load(os.path.join(HERE, "golden", "factor_inputs.npz"))
    M, lam = npz["M_128_9"], npz["lam_128_9"]
    cfg = H.SolverConfig(mode=mode, block_cols=16) if mode == "block" else None
    got = H.eigvalsh(M, cfg)
    err = np.max(np.abs(got - lam) / np.abs(lam))
    assert err <= 1e-12


# ---- qr_shorten (test_factory.py:148-177, the reference's tolerances) ------
def test_qr_orthonormal_input():
    Q0 = np.linalg.qr(np.random.default_rng(0).standard_normal((6, 3)))[0]
    R, Q = H.qr_shorten(Q0)
    np.testing.assert_allclose(R, np.eye(3), atol=1e-14)


def test_qr_single_column():
    R, Q = H.qr_shorten(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(R, [[5.0]], rtol=1e-15)
    np.testing.assert_allclose(Q, [[0.6], [0.8]], rtol=1e-15)


@pytest.mark.parametrize("shape", [(40, 12), (300, 100), (2048, 512)])
def test_qr_residual_and_orthogonality(shape):
    n, r = shape
    G = np.random.default_rng(4).standard_normal((n, r))
    R, Q = H.qr_shorten(G)
    assert np.linalg.norm(Q @ R - G) <= 20.0 * n * H.EPS * np.linalg.norm(G)
    assert np.linalg.norm(Q.T @ Q - np.eye(r)) <= n * n * H.EPS
    assert np.all(np.diag(R) > 0.0)
    np.testing.assert_allclose(R, np.triu(R), atol=0)
    # the reference's R to rounding (same algorithm; numpy's BLAS sums differ)
    if n <= 300:
        sys.path.insert(0, os.path.dirname(HERE))
        from oracle.qr_ref import qr_shorten_numpy
        R0, Q0 = qr_shorten_numpy(G)
        np.testing.assert_allclose(R, R0, rtol=0, atol=1e-12 * np.abs(R0).max())


def test_qr_errors():
    with pytest.raises(H.ShapeError):
        H.qr_shorten(np.eye(3))
    G = np.zeros((4, 2))
    G[:, 0] = 1.0
    with pytest.raises(H.RankDeficiencyError):
        H.qr_shorten(G)


def test_qr_then_hsvd_tall():
    # the HSVD of a tall G through its R factor (factory.py:300-305)
    rng = np.random.default_rng(9)
    G = rng.standard_normal((96, 32))
    J = H.SignatureVector.from_p(32, 20)
    R, Q = H.qr_shorten(G)
    a = H.drive(G, J)
    b = H.drive(R, J)
    np.testing.assert_allclose(np.sort(a.lam), np.sort(b.lam), rtol=1e-12)


# ---- generation in double-double (factory.py:79-114, 285-297) --------------
@pytest.mark.parametrize("case", GOLD["gen"], ids=lambda c: f"gen-{c['n']}-{c['seed']}-{c['pos_count']}")
def test_generate_bit_exact(case):
    spec = H.SpectrumSpec(case["n"], 20.0, case["seed"], case["pos_count"])
    M, lam = H.generate_symmetric(spec)
    assert digest(M) == case["M"]
    assert digest(lam) == case["lam"]
    b = H.generate_factor_pair(spec)
    assert digest(b.M) == case["bundle_M"]
    assert digest(b.factor.G) == case["G"]
    assert hashlib.sha256(np.asarray(b.factor.perm, "<i8").tobytes()).hexdigest() == case["perm"]
    assert b.factor.J.p == case["p"]


def test_generate_end_to_end_eigenvalues():
    # test_factory.py:134-139 at the reference's size
    b = H.generate_factor_pair(H.SpectrumSpec(160, 20.0, 1))
    res = H.drive(b.factor.G, b.factor.J)
    err = np.max(np.abs(np.sort(res.lam) - b.lambda_true) / np.abs(b.lambda_true))
    assert err <= 1e-12
    assert b.factor.J.p == np.count_nonzero(b.lambda_true > 0)


def test_generate_identity_q():
    M, lam = H.generate_symmetric(H.SpectrumSpec(6, 20.0, 0), eigenvalues=[3.0, -1.0, 2.0, 5.0, -4.0, 1.0],
                                  identity_q=True)
    np.testing.assert_array_equal(M, np.diag([3.0, -1.0, 2.0, 5.0, -4.0, 1.0]))
    np.testing.assert_array_equal(lam, np.sort([3.0, -1.0, 2.0, 5.0, -4.0, 1.0]))


@pytest.mark.parametrize("n", [256, 2048, 4096])
def test_generate_pow2_path_matches_generic(n):
    # power-of-two n takes the warp-shuffle trees and the mirrored update;
    # the generic shared-memory path (pinned to the reference's goldens) must
    # give the same bits
    import subprocess
    code = ("import sys, hashlib; sys.path.insert(0, '.'); import numpy as np; "
            "import paper_1008_1371_b200 as H; "
            f"M, lam = H.generate_symmetric(H.SpectrumSpec({n}, 20.0, 5)); "
            "print(hashlib.sha256(np.ascontiguousarray(M).tobytes()).hexdigest())")
    root = os.path.dirname(HERE)
    out = {}
    for flag in ("1", "0"):
        env = dict(os.environ, HSVD_GEN_POW2=flag)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-1500:]
        out[flag] = r.stdout.strip().splitlines()[-1]
    assert out["1"] == out["0"]
