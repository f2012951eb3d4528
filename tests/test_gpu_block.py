"""Block mode (FP64 tensor-core Gram/update + smem inner rotations) against
the reference: sigma per sign class within 1e-10 relative (north star
tolerance), residuals next to the reference's own, protocol stop, sweep
count within the documented band.  The reference results come from the
oracle (bit-exact with hjsvd, tests/test_oracle_golden.py)."""

import numpy as np
import pytest

import paper_1008_1371_b200 as H
from oracle import oracle as O
from tests.block_metrics import residuals, sigma_class_reldiff
from tests.golden.inputs import make_case_input

pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-10     # north star: "singular values within ~1e-10"
# block residuals at or below the reference's own (north star) with the
# default "fast" rotation; measured ratios for every case are in
# profiles/r02_block_residual_ratios.md (worst: dU 0.96, VtJV 0.37, recon
# 0.30).  The "dd" variant (the reference's double-double rotation_tc inside
# the block inner pass, a cross-check, not the default or benchmarked path)
# measures up to 1.6x on recon / VtJV (same table): band 2.0.
RESID_FACTOR = 1.0
RESID_FACTOR_ROT = {"fast": 1.0, "dd": 2.0}

CASES = [
    # n, r, p, seed, kind, b
    (64, 64, 32, 0, "gauss", 16),
    (96, 64, 20, 3, "gauss", 16),
    (128, 128, 64, 1, "gauss", 32),
    (128, 128, 128, 1, "gauss", 16),
    (256, 256, 128, 0, "gauss", 32),
    (256, 256, 128, 0, "graded12", 32),
    (256, 256, 0, 5, "gauss", 32),
    (512, 512, 384, 0, "gauss", 32),
    (520, 512, 200, 2, "gauss", 32),
]


@pytest.mark.parametrize("rot", ["fast", "dd"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"n{c[0]}r{c[1]}p{c[2]}{c[4]}b{c[5]}")
def test_block_matches_reference(case, rot):
    n, r, p, seed, kind, b = case
    G = make_case_input(n, r, seed, kind)
    signs = np.array([1] * p + [-1] * (r - p), np.int8)
    ref = O.drive(G, signs, p)
    res = H.drive(G, H.SignatureVector(signs, p),
                  H.SolverConfig(mode="block", block_cols=b, block_rotation=rot))
    assert res.stop_reason in ("orthogonal", "quadratic")
    d = sigma_class_reldiff(res.sigma, res.lam, ref.sigma, ref.lam)
    assert d <= SIGMA_RTOL, d
    rb, rr = residuals(G, res, signs), residuals(G, ref, signs)
    for k in rb:
        assert rb[k] <= RESID_FACTOR_ROT[rot] * rr[k], (k, rb[k], rr[k])
    # block sweeps: the full inner ordering (default) rotates every pair of
    # the pivot block at every step; it never needs more sweeps than the
    # reference in any measured case (7-11 vs 8-14)
    assert res.sweeps_used <= ref.sweeps_used, (res.sweeps_used, ref.sweeps_used)


def test_block_big_golden(golden_big):
    import os
    here = os.path.join(os.path.dirname(__file__), "golden")
    for c in golden_big["drive"]:
        G = make_case_input(c["n"], c["r"], c["seed"], c["kind"])
        signs = np.array([1] * c["p"] + [-1] * (c["r"] - c["p"]), np.int8)
        sig_ref = np.load(os.path.join(here, f"sigma_{c['name']}.npy"))
        lam_ref = sig_ref ** 2 * np.sign(np.array([1.0] * c["p"] + [-1.0] * (c["r"] - c["p"])))
        res = H.drive(G, H.SignatureVector(signs, c["p"]),
                      H.SolverConfig(mode="block", block_cols=32))
        # the reference's lam carries the sign of each ORIGINAL column
        d = sigma_class_reldiff(res.sigma, res.lam, sig_ref, lam_ref)
        assert d <= SIGMA_RTOL, (c["name"], d)
        rb = residuals(G, res, signs)
        assert rb["dU"] <= RESID_FACTOR * c["dU"], (c["name"], rb, c["dU"])
        assert rb["vjv"] <= RESID_FACTOR * c["VtJV"], (c["name"], rb, c["VtJV"])
        assert rb["recon"] <= RESID_FACTOR * c["recon"], (c["name"], rb, c["recon"])
        assert res.sweeps_used <= c["sweeps_used"]


def test_block_deterministic():
    G = make_case_input(256, 256, 0, "gauss")
    J = H.SignatureVector.from_p(256, 128)
    cfg = H.SolverConfig(mode="block", block_cols=32)
    a = H.drive(G, J, cfg)
    b = H.drive(G, J, cfg)
    assert np.array_equal(a.U, b.U) and np.array_equal(a.sigma, b.sigma)


def test_block_full_inner_ordering():
    G = make_case_input(256, 256, 0, "gauss")
    signs = np.array([1] * 128 + [-1] * 128, np.int8)
    ref = O.drive(G, signs, 128)
    res = H.drive(G, H.SignatureVector(signs, 128),
                  H.SolverConfig(mode="block", block_cols=32, inner_ordering="full"))
    assert sigma_class_reldiff(res.sigma, res.lam, ref.sigma, ref.lam) <= SIGMA_RTOL


@pytest.mark.parametrize("case", [
    # n, r, p, seed, kind, b: r not a multiple of 2b (inert zero-column padding)
    (1000, 1000, 500, 4, "gauss", 32),
    (520, 514, 200, 2, "gauss", 32),
    (96, 70, 30, 1, "gauss", 16),
    (300, 258, 258, 3, "graded12", 32),
    (64, 62, 0, 5, "gauss", 16),
], ids=lambda c: f"n{c[0]}r{c[1]}p{c[2]}{c[4]}b{c[5]}")
def test_block_any_even_r(case):
    """Block mode for r not a multiple of 2b (solver.py:289-341 purpose):
    sigma per class within 1e-10 of the reference, residuals within the
    same band as the aligned cases, the input never mutated."""
    n, r, p, seed, kind, b = case
    G = make_case_input(n, r, seed, kind)
    G0 = G.copy()
    signs = np.array([1] * p + [-1] * (r - p), np.int8)
    ref = O.drive(G, signs, p)
    res = H.drive(G, H.SignatureVector(signs, p), H.SolverConfig(mode="block", block_cols=b))
    assert np.array_equal(G, G0)
    assert res.U.shape == (n, r) and res.Vinv_t.shape == (r, r) and res.sigma.shape == (r,)
    assert res.stop_reason in ("orthogonal", "quadratic")
    assert np.all(np.isfinite(res.U)) and np.all(np.isfinite(res.Vinv_t))
    assert sigma_class_reldiff(res.sigma, res.lam, ref.sigma, ref.lam) <= SIGMA_RTOL
    rb, rr = residuals(G, res, signs), residuals(G, ref, signs)
    for k in rb:
        assert rb[k] <= RESID_FACTOR * rr[k], (k, rb[k], rr[k])


def test_block_padding_identity_diag():
    G = np.asfortranarray(np.diag(np.arange(40, 0, -1, dtype=np.float64)))
    res = H.drive(G, H.SignatureVector.from_p(40, 20), H.SolverConfig(mode="block", block_cols=32))
    assert res.stop_reason == "orthogonal" and res.rotations == 0 and res.sweeps_used == 1
    assert np.array_equal(np.sort(res.sigma), np.arange(1.0, 41.0))
    # pairs with a padding column are not visits: r_pad = 64, one slot, two
    # steps of the full ordering, 40 * 39 / 2 real pairs each
    assert res.skips == 2 * (40 * 39 // 2)


def test_block_config3_n4096_p3072_against_pointwise():
    """BASELINE config 3 (n = 4096, p = 3072): block mode against the
    pointwise mode, which is bit-exact with the reference (test_gpu_parity);
    sigma per class within the north-star 1e-10, residuals at or below the
    reference's own (factor 2 band), sweeps not above the reference's."""
    n, p = 4096, 3072
    G = make_case_input(n, n, 0, "gauss")
    signs = np.array([1] * p + [-1] * (n - p), np.int8)
    J = H.SignatureVector(signs, p)
    ref = H.drive(G, J, H.SolverConfig(mode="pointwise"))
    res = H.drive(G, J, H.SolverConfig(mode="block"))
    assert sigma_class_reldiff(res.sigma, res.lam, ref.sigma, ref.lam) <= SIGMA_RTOL
    rb, rr = residuals(G, res, signs), residuals(G, ref, signs)
    for k in rb:
        assert rb[k] <= rr[k], (k, rb[k], rr[k])
    assert res.sweeps_used <= ref.sweeps_used


def _definiteness_case(n=64, p=32):
    """Columns p-1 (J = +1) and p (J = -1) identical, every other column a
    unit vector orthogonal to them: the hyperbolic pair has |theta| = 1 and
    no other rotation can change it first (the reference raises
    DefinitenessLostError on it, _kernels.py:163-171)."""
    G = np.eye(n)
    G[:, p - 1] = 0.0
    G[:, p] = 0.0
    G[p - 1, p - 1] = G[p, p - 1] = 1.0
    G[p - 1, p] = G[p, p] = 1.0
    return np.asfortranarray(G), H.SignatureVector.from_p(n, p)


@pytest.mark.parametrize("rot", ["fast", "dd"])
def test_block_definiteness_lost_raises(rot):
    G, J = _definiteness_case()
    with pytest.raises(RuntimeError) as ei:
        O.drive(G, J.signs, J.p)  # the reference's behaviour on this input
    assert ei.value.args[0] == 1   # status 1: definiteness lost
    with pytest.raises(H.DefinitenessLostError):
        H.drive(G, J, H.SolverConfig(mode="block", block_cols=16, block_rotation=rot))


@pytest.mark.parametrize("N", [1, 2])
def test_sharded_definiteness_lost_raises(N):
    G, J = _definiteness_case()
    with pytest.raises(H.DefinitenessLostError):
        H.drive_local_shards(G, J, H.SolverConfig(mode="block", block_cols=16), nshards=N)


@pytest.mark.parametrize("streams", [1, 2])
def test_block_allskip_reuse_is_exact(streams, monkeypatch):
    """Replaying recorded all-skip visits (k_plan, the late sweeps) gives the
    bits, sweeps and statistics of recomputing them (_kernels.py:210-213:
    the skip decision is a function of the pair's columns alone)."""
    for kind, n, p in (("gauss", 1024, 512), ("graded12", 512, 256)):
        G = make_case_input(n, n, 3, kind)
        J = H.SignatureVector.from_p(n, p)
        cfg = H.SolverConfig(mode="block", block_streams=streams)
        monkeypatch.setenv("HSVD_REUSE", "0")
        a = H.drive(G, J, cfg)
        monkeypatch.setenv("HSVD_REUSE", "1")
        b = H.drive(G, J, cfg)
        assert (a.sweeps_used, a.stop_reason, a.rotations, a.skips) == \
            (b.sweeps_used, b.stop_reason, b.rotations, b.skips)
        assert a.telemetry == b.telemetry
        for f in ("sigma", "lam", "U", "Vinv_t"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("case", [
    (1024, 1024, 512, 0, "gauss", 32),
    (520, 512, 200, 2, "gauss", 32),     # n not a multiple of the k-tile
    (1000, 1000, 500, 4, "gauss", 32),   # padded r, ragged n
    (256, 256, 100, 3, "graded12", 16),
], ids=lambda c: f"n{c[0]}r{c[1]}p{c[2]}{c[4]}b{c[5]}")
def test_gram_tma_bit_identical_to_cp_async(case, monkeypatch):
    """k_gram_tma (TMA gather4 + mbarrier ring) issues the cp.async
    kernel's DMMA sequence on the same segments: the whole solve is bit for
    bit the same (rows beyond n come in as TMA zero fill)."""
    n, r, p, seed, kind, b = case
    G = make_case_input(n, r, seed, kind)
    J = H.SignatureVector.from_p(r, p)
    cfg = H.SolverConfig(mode="block", block_cols=b)
    monkeypatch.setenv("HSVD_GRAM_TMA", "0")
    a = H.drive(G, J, cfg)
    monkeypatch.setenv("HSVD_GRAM_TMA", "1")
    t = H.drive(G, J, cfg)
    assert (a.sweeps_used, a.rotations, a.skips) == (t.sweeps_used, t.rotations, t.skips)
    for f in ("sigma", "lam", "U", "Vinv_t"):
        assert np.array_equal(getattr(a, f), getattr(t, f)), f


# The inner kernel's other schedules (csrc/hsvd_inner.cuh): the oriented
# ordering (b rounds, the j half of the W row positions cycling), several
# passes per step (the W warps' per-pass hand-off), and b = 16.  sigma is
# held to the same 1e-10; the residual band is 2x the reference's own (these
# are not the benchmarked schedule: measured ratios up to ~1.2, see
# DESIGN "Knobs"); U and V^{-T} are checked for orthogonality directly.
@pytest.mark.parametrize("ordering,passes", [("oriented", 1), ("full", 2), ("oriented", 2), ("full", 3)])
@pytest.mark.parametrize("b", [16, 32])
def test_block_inner_schedules(ordering, passes, b):
    n, r, p = 256, 256, 96
    G = make_case_input(n, r, 7, "gauss")
    signs = np.array([1] * p + [-1] * (r - p), np.int8)
    ref = O.drive(G, signs, p)
    res = H.drive(G, H.SignatureVector(signs, p),
                  H.SolverConfig(mode="block", block_cols=b, inner_ordering=ordering,
                                 inner_passes=passes))
    assert res.stop_reason in ("orthogonal", "quadratic")
    d = sigma_class_reldiff(res.sigma, res.lam, ref.sigma, ref.lam)
    assert d <= SIGMA_RTOL, (ordering, passes, b, d)
    rb, rr = residuals(G, res, signs), residuals(G, ref, signs)
    for k in rb:
        assert rb[k] <= 2.0 * rr[k], (ordering, passes, b, k, rb[k], rr[k])
    # deterministic: the same schedule twice gives the same bits
    again = H.drive(G, H.SignatureVector(signs, p),
                    H.SolverConfig(mode="block", block_cols=b, inner_ordering=ordering,
                                   inner_passes=passes))
    assert np.array_equal(again.U, res.U) and np.array_equal(again.sigma, res.sigma)


def test_block_auto_inner_passes():
    """inner_passes = 0 (auto, default): two passes per step in the dense
    sweeps for >= 32 block columns, one pass for small problems.  At r = 256
    (8 blocks) auto is exactly the one-pass solve; at r = 1024 (32 blocks) it
    is not, and it meets the same sigma / residual gates against the oracle
    in no more sweeps."""
    def solve(n, r, p, passes):
        G = make_case_input(n, r, 11, "gauss")
        signs = np.array([1] * p + [-1] * (r - p), np.int8)
        return G, signs, H.drive(G, H.SignatureVector(signs, p),
                                 H.SolverConfig(mode="block", inner_passes=passes))

    _, _, a = solve(256, 256, 100, 0)
    _, _, one = solve(256, 256, 100, 1)
    assert np.array_equal(a.U, one.U) and a.sweeps_used == one.sweeps_used
    G, signs, auto = solve(1024, 1024, 400, 0)
    _, _, one = solve(1024, 1024, 400, 1)
    assert not np.array_equal(auto.U, one.U)
    assert auto.sweeps_used <= one.sweeps_used
    ref = O.drive(G, signs, 400)
    assert sigma_class_reldiff(auto.sigma, auto.lam, ref.sigma, ref.lam) <= SIGMA_RTOL
    rb, rr = residuals(G, auto, signs), residuals(G, ref, signs)
    for k in rb:
        assert rb[k] <= rr[k], (k, rb[k], rr[k])
