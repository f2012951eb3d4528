"""CPU: the factorization oracle (oracle/factor_oracle.c) against the
reference's goldens (tests/golden/factor.json, made by
tests/golden/make_golden_factor.py from hjsvd.factory.bunch_parlett_factor)."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
sys.path.insert(0, os.path.dirname(HERE))

from digest import digest  # noqa: E402
from factor_inputs import make_input  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLD = json.load(open(os.path.join(HERE, "golden", "factor.json")))


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c['kind']}-{c['n']}-{c['seed']}")
def test_oracle_factor_bit_exact(case):
    M = make_input(case["kind"], case["n"], case["seed"])
    G, signs, perm, p = O.bp_factor(M)
    assert digest(G) == case["G"]
    assert hashlib.sha256(np.asarray(perm, "<i8").tobytes()).hexdigest() == case["perm"]
    assert hashlib.sha256(np.asarray(signs, "i1").tobytes()).hexdigest() == case["signs"]
    assert p == case["p"]


def test_oracle_factor_singular():
    with pytest.raises(ArithmeticError):
        O.bp_factor(np.ones((3, 3)))
