"""CPU-only tests of the host side: the C-ABI library loads and exports
every declared symbol, config/struct plumbing, the host stepper against the
reference's golden sequences, convergence decisions, bordering, and that
the product path refuses to run without a GPU (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest
import torch

import paper_1008_1371_b200 as H
from paper_1008_1371_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hsvd_b200.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"HSVD_API[^;(]*?\b(hsvd_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_default_config_matches_solverconfig():
    L = _lib.load()
    c = _lib.HsvdConfigC()
    L.hsvd_default_config(c)
    py = H.SolverConfig().to_c()
    for name, _ in _lib.HsvdConfigC._fields_:
        if name in ("block_cols",):
            continue
        assert getattr(c, name) == getattr(py, name), name


def test_solverconfig_defaults_mirror_reference():
    cfg = H.SolverConfig()
    assert cfg.max_sweeps == 30 and cfg.eps == 2.0 ** -52
    assert cfg.teps == 2.0 ** -27 and cfg.chunk == 32
    assert cfg.accumulate_v and cfg.use_rel_orth_skip and cfg.sort
    assert cfg.schedule == "modulus" and cfg.workers == 1
    with pytest.raises(ValueError):
        H.SolverConfig(schedule="bogus")
    with pytest.raises(ValueError):
        H.SolverConfig(workers=0)


def test_block_cols_validated():
    """block_cols outside {16, 32} is rejected on the host, and the
    workspace query never divides by it (no SIGFPE through the C ABI)."""
    for b in (0, -1, 8, 64):
        with pytest.raises(ValueError):
            H.SolverConfig(mode="block", block_cols=b)
    L = _lib.load()
    c = H.SolverConfig(mode="block").to_c()
    c.block_cols = 0
    assert L.hsvd_drive_workspace_size(256, 256, c) > 0
    assert L.hsvd_sharded_workspace_size(256, 256, 2, 0, c) == -1


def test_struct_sizes():
    """The ctypes mirrors have the C layouts (sizes reported by the library)."""
    out = (ctypes.c_int64 * 3)()
    _lib.load().hsvd_abi_sizes(out)
    assert ctypes.sizeof(_lib.HsvdConfigC) == out[0]
    assert ctypes.sizeof(_lib.HsvdResultC) == out[1]
    assert ctypes.sizeof(_lib.HsvdTelemetryC) == out[2]


def test_workspace_size_query():
    L = _lib.load()
    c = H.SolverConfig().to_c()
    assert L.hsvd_drive_workspace_size(256, 256, c) > 24 * 256


def test_check_convergence():
    assert H.check_convergence(np.array([0, 0, 0], np.uint8)) == "stop_orthogonal"
    assert H.check_convergence(np.array([1, 0, 1], np.uint8)) == "stop_quadratic"
    assert H.check_convergence(np.array([1, 3, 0], np.uint8)) == "continue"


def test_host_stepper_matches_reference(golden):
    for r, seq in golden["stepper"].items():
        S = H.stepper_init(int(r))
        for ib, jb in seq:
            assert list(S.iblk) == ib and list(S.jblk) == jb
            for k in range(int(r) // 2):
                H.stepper_advance(S, k)


def test_schedule_table_covers_all_pairs():
    for r in (2, 4, 8, 16, 34):
        T = H.schedule_table(r, r)
        seen = set()
        for s in range(r):
            flat = T[s].ravel()
            assert len(set(flat.tolist())) == r  # disjoint pairs in a step
            seen |= {tuple(p) for p in T[s].tolist()}
        assert len(seen) == r * (r - 1) // 2


def test_signature_vector():
    J = H.SignatureVector.from_p(5, 2)
    assert list(J.signs) == [1, 1, -1, -1, -1] and len(J) == 5
    with pytest.raises(ValueError):
        H.SignatureVector(np.array([1, -1, 1], np.int8), 2)


def test_border_and_strip():
    G = np.arange(9.0).reshape(3, 3) + 1.0
    J = H.SignatureVector.from_p(3, 3)
    G2, J2, info = H.border(G, J, 4, 4)
    assert info.synthetic_col == 3 and G2[3, 3] == 1.0 and J2.p == 4
    rng = np.random.default_rng(2)
    G = rng.standard_normal((4, 3))
    G2, J2, info = H.border(G, H.SignatureVector.from_p(3, 1), 4, 5)
    assert info.synthetic_col == 1 and J2.p == 2 and G2[4, 1] == 1.0
    with pytest.raises(H.ShapeError):
        H.border(G, H.SignatureVector.from_p(3, 1), 4, 4)


def test_recover_v():
    rng = np.random.default_rng(0)
    W = rng.standard_normal((4, 4))
    assert np.array_equal(H.recover_V(W, H.SignatureVector.from_p(4, 4)), W)
    assert np.array_equal(H.recover_V(np.eye(4), H.SignatureVector.from_p(4, 2)),
                          np.eye(4))


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only behaviour")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        H.drive(np.eye(4), H.SignatureVector.from_p(4, 2))


def test_sharded_api_validation():
    """The sharded entry points reject bad calls before touching a device."""
    G = np.zeros((64, 64))
    J = H.SignatureVector.from_p(64, 32)
    with pytest.raises(ValueError):
        H.drive_sharded(G, J, H.SolverConfig(mode="block"), comm=None)
    L = _lib.load()
    # 2 slots of b=16 cannot feed 4 shards; r not a multiple of b
    assert L.hsvd_shard_columns(64, 16, 4, 0) == -1
    assert L.hsvd_shard_columns(63, 16, 1, 0) == -1
    assert L.hsvd_shard_columns(128, 16, 2, 1) == 64
    c = H.SolverConfig(mode="block", block_cols=16).to_c()
    assert L.hsvd_sharded_workspace_size(128, 128, 2, 0, c) > 0
