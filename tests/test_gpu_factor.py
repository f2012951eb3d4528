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
