"""GPU parity: the pointwise CUDA path against the reference's golden
outputs (bit-exact: SHA-256 of sigma, lam, U, V^{-T}; equal sweeps,
rotations, skips, telemetry).  Calls go through the C ABI via the host
package, exactly the path drive() uses."""

import numpy as np
import torch
import pytest

import paper_1008_1371_b200 as H
from tests.golden.digest import digest, unhex
from tests.golden.inputs import make_case_input

pytestmark = pytest.mark.gpu


def _run(c):
    G = make_case_input(c["n"], c["r"], c["seed"], c["kind"])
    J = H.SignatureVector.from_p(c["r"], c["p"])
    cfg = H.SolverConfig(**c["cfg"])
    return H.drive(G, J, cfg)


def _check(c, res):
    assert digest(res.sigma) == c["sigma"], c["name"]
    assert digest(res.lam) == c["lam"], c["name"]
    assert digest(res.U) == c["U"], c["name"]
    assert digest(res.Vinv_t) == c["Vinv_t"], c["name"]
    assert res.sweeps_used == c["sweeps_used"], c["name"]
    assert res.stop_reason == c["stop_reason"], c["name"]
    assert (res.rotations, res.skips) == (c["rotations"], c["skips"]), c["name"]
    tele = [[a, b, d, float(e).hex()] for a, b, d, e in res.telemetry]
    assert tele == c["telemetry"], c["name"]


def test_drive_bit_exact_small(golden):
    for c in golden["drive"]:
        _check(c, _run(c))


def test_drive_bit_exact_big(golden_big):
    for c in golden_big["drive"]:
        _check(c, _run(c))


def test_drive_without_graph_matches(golden):
    c = next(c for c in golden["drive"] if c["name"] == "n64_p32")
    G = make_case_input(64, 64, 0, "gauss")
    res = H.drive(G, H.SignatureVector.from_p(64, 32), H.SolverConfig(use_graph=False))
    _check(c, res)


def test_drive_device_tensor_input(golden):
    import torch
    c = next(c for c in golden["drive"] if c["name"] == "n96x64_p20")
    G = make_case_input(96, 64, 3, "gauss")
    res = H.drive(torch.from_numpy(G).cuda(), H.SignatureVector.from_p(64, 20))
    assert digest(res.sigma.cpu().numpy()) == c["sigma"]
    assert digest(res.U.cpu().numpy()) == c["U"]
    assert digest(res.Vinv_t.cpu().numpy()) == c["Vinv_t"]


def test_input_not_mutated():
    G = make_case_input(32, 32, 9, "gauss")
    G0 = G.copy()
    H.drive(G, H.SignatureVector.from_p(32, 12))
    assert np.array_equal(G, G0)


def test_cuda_input_not_mutated():
    """A column-major float64 CUDA G (whose transpose is already contiguous)
    must be copied, not overwritten by U (the reference copies G,
    solver.py:188)."""
    G = make_case_input(64, 64, 2, "gauss")
    Gd = torch.from_numpy(np.asfortranarray(G)).cuda()   # strides (1, 64)
    Gd = torch.as_strided(Gd.t().contiguous(), (64, 64), (1, 64))
    G0 = Gd.clone()
    res = H.drive(Gd, H.SignatureVector.from_p(64, 32))
    assert torch.equal(Gd, G0)
    assert res.U.data_ptr() != Gd.data_ptr()
    for mode in ("pointwise", "block"):
        res = H.drive(Gd, H.SignatureVector.from_p(64, 32),
                      H.SolverConfig(mode=mode, block_cols=16))
        assert torch.equal(Gd, G0), mode


def test_rotation_kernel_bit_exact(golden):
    rows = golden["rotation"]
    a = np.array([unhex(r[0]) for r in rows])
    b = np.array([unhex(r[1]) for r in rows])
    c = np.array([unhex(r[2]) for r in rows])
    h = np.array([r[3] for r in rows], np.int64)
    from paper_1008_1371_b200 import _device
    t, cc, bad = _device.rotation_batch(a, b, c, h)
    status = np.array([r[6] for r in rows])
    assert bad == int(np.argmax(status != 0))
    ok = status == 0
    assert np.array_equal(t[ok], np.array([unhex(r[4]) for r in rows])[ok])
    assert np.array_equal(cc[ok], np.array([unhex(r[5]) for r in rows])[ok])


def test_dot_kernel_bit_exact(golden):
    from tests.golden.make_golden_vectors import dot_vectors
    for (length, chunk, x, y), rec in zip(dot_vectors(), golden["dot"]):
        assert H.dot_chunked(x, y, chunk) == unhex(rec[4]), (length, chunk)


def test_sort_kernel_matches(golden):
    for r, p, d, rho_ref in golden["sort"]:
        D = H.DiagonalPackageVector(np.array(d), np.arange(r, dtype=np.int64),
                                    np.array([1] * p + [-1] * (r - p), np.int64), p)
        H.sort_diagonal(D)
        assert list(D.rho) == rho_ref


def test_stepper_kernel_matches(golden):
    for r, seq in golden["stepper"].items():
        S = H.stepper_init(int(r))
        for ib, jb in seq:
            assert list(S.iblk) == ib and list(S.jblk) == jb
            H.stepper_advance_all(S)


def test_jacobi_step_matches_oracle():
    from oracle import oracle as O
    G = make_case_input(48, 40, 1, "gauss")
    J = H.SignatureVector.from_p(40, 15)
    D = H.precompute(G, J)
    dO, _ = O.precompute(G)
    assert np.array_equal(D.d, dO)
    H.sort_diagonal(D)
    rhoO = np.arange(40, dtype=np.int64)
    jsO = J.signs.astype(np.int64)
    O.sort_diagonal(dO, rhoO, jsO, 15)
    assert np.array_equal(D.rho, rhoO)
    S = H.stepper_init(40)
    C = np.zeros(20, np.uint8)
    V = np.asfortranarray(np.eye(40))
    Gg = G.copy(order="F")
    GO, VO, CO = G.copy(order="F"), np.asfortranarray(np.eye(40)), C.copy()
    ip, jp, ib, jb = O.stepper_init(40)
    for _ in range(45):
        st = H.jacobi_step(Gg, V, D, S, C)
        so, stats, _ = O.step_blocks(GO, VO, dO, rhoO, jsO, ib, jb, CO, 0, 20)
        O.advance_stepper(ip, jp, ib, jb, 40)
        assert so == 0
        assert st == (int(stats[0]), int(stats[1]), float(stats[2]))
        assert np.array_equal(Gg, GO) and np.array_equal(V, VO)
        assert np.array_equal(D.d, dO) and np.array_equal(C, CO)
        assert np.array_equal(S.iblk, ib) and np.array_equal(S.jblk, jb)


def test_rank_deficiency_raises():
    G = np.eye(4)
    G[:, 2] = 0.0
    with pytest.raises(H.RankDeficiencyError):
        H.drive(G, H.SignatureVector.from_p(4, 2))
    with pytest.raises(H.RankDeficiencyError):
        H.precompute(G, H.SignatureVector.from_p(4, 2))


def test_definiteness_lost_raises():
    # two identical columns with opposite signs: the hyperbolic pair has
    # |tanh 2phi| = 1 (the reference raises DefinitenessLostError too)
    G = np.asfortranarray(np.array([[1.0, 1.0], [1.0, 1.0]]))
    with pytest.raises(H.DefinitenessLostError) as ei:
        H.drive(G, H.SignatureVector.from_p(2, 1))
    assert (ei.value.block, ei.value.i, ei.value.j) == (0, 0, 1)


def test_shape_errors():
    with pytest.raises(H.ShapeError):
        H.drive(np.eye(3), H.SignatureVector.from_p(3, 3))
    with pytest.raises(H.ShapeError):
        H.drive(np.ones((2, 4)), H.SignatureVector.from_p(4, 4))


@pytest.mark.parametrize("mode", ["pointwise", "block"])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_input_raises(mode, bad):
    """as_factor's finiteness rule (linalg.py:58-65), checked on the device
    by the library (no host scan): numpy and CUDA-tensor inputs alike."""
    G = make_case_input(64, 64, 1, "gauss")
    G[17, 40] = bad
    cfg = H.SolverConfig(mode=mode, block_cols=16)
    with pytest.raises(ValueError, match="non-finite"):
        H.drive(G, H.SignatureVector.from_p(64, 32), cfg)
    with pytest.raises(ValueError, match="non-finite"):
        H.drive(torch.from_numpy(G).cuda(), H.SignatureVector.from_p(64, 32), cfg)
