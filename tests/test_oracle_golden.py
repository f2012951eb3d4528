"""The CPU oracle (oracle/hsvd_oracle.c) is pinned bit-for-bit to the real
reference through tests/golden/golden.json (made by make_golden.py from
/root/reference).  CPU only."""

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.digest import digest, unhex
from tests.golden.inputs import make_case_input


def _cases(golden, maxn=1000):
    return [c for c in golden["drive"] if c["n"] <= maxn]


def test_oracle_drive_matches_reference(golden):
    for c in _cases(golden):
        G = make_case_input(c["n"], c["r"], c["seed"], c["kind"])
        signs = np.array([1] * c["p"] + [-1] * (c["r"] - c["p"]), np.int8)
        cfg = dict(c["cfg"])
        res = O.drive(G, signs, c["p"], **cfg)
        assert digest(res.sigma) == c["sigma"], c["name"]
        assert digest(res.lam) == c["lam"], c["name"]
        assert digest(res.U) == c["U"], c["name"]
        assert digest(res.Vinv_t) == c["Vinv_t"], c["name"]
        assert res.sweeps_used == c["sweeps_used"], c["name"]
        assert res.stop_reason == c["stop_reason"], c["name"]
        assert res.rotations == c["rotations"] and res.skips == c["skips"]
        tele = [[a, b, d, float(e).hex()] for a, b, d, e in res.telemetry]
        assert tele == c["telemetry"], c["name"]


def test_oracle_worker_count_invisible(golden):
    c = next(c for c in golden["drive"] if c["name"] == "n256_p128")
    G = make_case_input(256, 256, 0, "gauss")
    signs = np.array([1] * 128 + [-1] * 128, np.int8)
    for w in (1, 3, 8):
        res = O.drive(G, signs, 128, workers=w)
        assert digest(res.U) == c["U"]


def test_oracle_rotation_matches_reference(golden):
    for a_ii, a_jj, a_ij, hyp, t, c, st in golden["rotation"]:
        tt, cc, s = O.rotation_tc(unhex(a_ii), unhex(a_jj), unhex(a_ij), hyp)
        assert s == st
        if st == 0:
            assert tt == unhex(t) and cc == unhex(c)


def test_oracle_dot_matches_reference(golden):
    from tests.golden.make_golden_vectors import dot_vectors
    for (length, chunk, x, y), rec in zip(dot_vectors(), golden["dot"]):
        assert rec[0] == length and rec[1] == chunk
        assert digest(x) == rec[2]
        assert O.dot_chunked(x, y, chunk) == unhex(rec[4])


def test_oracle_stepper_matches_reference(golden):
    for r, seq in golden["stepper"].items():
        r = int(r)
        ip, jp, ib, jb = O.stepper_init(r)
        for ib_ref, jb_ref in seq:
            assert list(ib) == ib_ref and list(jb) == jb_ref
            O.advance_stepper(ip, jp, ib, jb, r)


def test_oracle_sort_matches_reference(golden):
    for r, p, d, rho_ref in golden["sort"]:
        d = np.array(d)
        rho = np.arange(r, dtype=np.int64)
        js = np.array([1] * p + [-1] * (r - p), np.int64)
        O.sort_diagonal(d, rho, js, p)
        assert list(rho) == rho_ref


@pytest.mark.parametrize("case", [
    ((1.0, 2.0, 0.5, -1), (np.sqrt(2.0) - 1.0, np.cos(np.pi / 8))),
    ((2.0, 1.0, -0.5, 1), (3.0 - 2.0 * np.sqrt(2.0), None)),
])
def test_oracle_closed_forms(case):
    (a, b, c, h), (t_ref, c_ref) = case
    t, cc, st = O.rotation_tc(a, b, c, h)
    assert st == 0
    np.testing.assert_allclose(t, t_ref, rtol=1e-14)
    if c_ref is not None:
        np.testing.assert_allclose(cc, c_ref, rtol=1e-15)
