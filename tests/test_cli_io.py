"""GJH1 / CSV files and the hsvd/eig command line (the reference's
test_io.py and test_cli.py::TestEig, on the solver path)."""

import filecmp
import os

import numpy as np
import pytest
from numpy.testing import assert_allclose

import paper_1008_1371_b200 as H
from paper_1008_1371_b200.cli import main
from paper_1008_1371_b200.matio import (read_csv_matrix, read_gjh, write_csv_matrix,
                                        write_gjh)


def run(*argv):
    return main([str(a) for a in argv])


def write_bundle(path, G, p, lambda_true=None):
    os.makedirs(path, exist_ok=True)
    write_gjh(os.path.join(path, "G.gjh"), G, p)
    if lambda_true is not None:
        write_csv_matrix(os.path.join(path, "lambda_true.csv"),
                         np.asarray(lambda_true)[np.newaxis, :])


# ---- files (CPU) ------------------------------------------------------------

def test_gjh_round_trip_bit_exact(tmp_path):
    M = np.random.default_rng(0).standard_normal((5, 3))
    write_gjh(tmp_path / "m.gjh", M, 2)
    M2, p = read_gjh(tmp_path / "m.gjh")
    assert p == 2 and M2.flags.f_contiguous and np.array_equal(M, M2)


def test_gjh_layout(tmp_path):
    M = np.arange(6.0).reshape(2, 3)
    write_gjh(tmp_path / "m.gjh", M, 1)
    raw = (tmp_path / "m.gjh").read_bytes()
    assert raw[:4] == b"GJH1" and len(raw) == 16 + 48
    payload = np.frombuffer(raw[16:], dtype="<f8")
    assert np.array_equal(payload, M.ravel(order="F"))  # column-major


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XJH1" + b[4:], "bad magic"),
    (lambda b: b[:10], "truncated GJH1 header"),
    (lambda b: b[:-8], "truncated GJH1 payload"),
])
def test_gjh_errors(tmp_path, mutate, msg):
    write_gjh(tmp_path / "m.gjh", np.eye(2), 1)
    (tmp_path / "m.gjh").write_bytes(mutate((tmp_path / "m.gjh").read_bytes()))
    with pytest.raises(ValueError, match=msg):
        read_gjh(tmp_path / "m.gjh")


def test_gjh_invalid_p(tmp_path):
    with pytest.raises(ValueError):
        write_gjh(tmp_path / "m.gjh", np.eye(2), 3)


def test_csv_round_trip_exact(tmp_path):
    M = np.random.default_rng(1).standard_normal((3, 4)) * 1e-300
    write_csv_matrix(tmp_path / "m.csv", M)
    assert np.array_equal(read_csv_matrix(tmp_path / "m.csv"), M)
    write_csv_matrix(tmp_path / "v.csv", np.arange(3.0))
    assert read_csv_matrix(tmp_path / "v.csv").shape == (1, 3)


# ---- command line: usage and I/O errors (CPU, before any device work) --------

def test_missing_bundle_exit_3(tmp_path):
    assert run("eig", "--in", tmp_path / "nope", "--out", tmp_path / "r") == 3


def test_odd_r_without_border_exit_2(tmp_path):
    G = np.random.default_rng(1).standard_normal((3, 3))
    write_bundle(tmp_path / "b", G, 3)
    assert run("eig", "--in", tmp_path / "b", "--out", tmp_path / "r") == 2


# ---- command line on the GPU ---------------------------------------------------

@pytest.mark.gpu
def test_eig_diagonal_bundle(tmp_path):
    write_bundle(tmp_path / "b", np.diag([2.0, 1.0]), 1, [-1.0, 4.0])
    assert run("eig", "--in", tmp_path / "b", "--out", tmp_path / "r") == 0
    lam = read_csv_matrix(tmp_path / "r" / "lambda.csv").ravel()
    assert_allclose(np.sort(lam), [-1.0, 4.0], rtol=0)
    rec = (tmp_path / "r" / "record.csv").read_text().splitlines()
    assert rec[0].startswith("n,r,p,sweeps") and rec[1].split(",")[3] == "1"


@pytest.mark.gpu
def test_eig_nonconvergence_exit_6(tmp_path):
    write_bundle(tmp_path / "b", np.random.default_rng(0).standard_normal((8, 8)), 4)
    assert run("eig", "--in", tmp_path / "b", "--out", tmp_path / "r", "--max-sweeps", 1) == 6


@pytest.mark.gpu
def test_eig_border(tmp_path):
    G = np.random.default_rng(1).standard_normal((3, 3))
    lam = np.linalg.eigvalsh(G @ G.T)
    write_bundle(tmp_path / "b", G, 3, lam)
    assert run("eig", "--in", tmp_path / "b", "--out", tmp_path / "r", "--border") == 0
    out = read_csv_matrix(tmp_path / "r" / "lambda.csv").ravel()
    assert out.shape == (3,)
    assert_allclose(np.sort(out), lam, rtol=1e-12)


@pytest.mark.gpu
def test_eig_workers_identical_files_and_no_v(tmp_path):
    G = np.random.default_rng(3).standard_normal((12, 12))
    write_bundle(tmp_path / "b", G, 5)
    run("eig", "--in", tmp_path / "b", "--out", tmp_path / "r1")
    run("eig", "--in", tmp_path / "b", "--out", tmp_path / "r2", "--workers", 4)
    for name in ("lambda.csv", "sigma.csv", "U.gjh", "V.gjh"):
        assert filecmp.cmp(tmp_path / "r1" / name, tmp_path / "r2" / name, shallow=False)
    assert run("eig", "--in", tmp_path / "b", "--out", tmp_path / "r3",
               "--no-accumulate-v") == 0
    assert not (tmp_path / "r3" / "V.gjh").exists()


@pytest.mark.gpu
def test_hsvd_block_and_shards(tmp_path):
    n, p = 256, 100
    G = np.random.default_rng(4).standard_normal((n, n))
    J = H.SignatureVector.from_p(n, p)
    ref = H.drive(G, J)  # pointwise: bit-exact with the reference
    write_bundle(tmp_path / "b", G, p, ref.lam)
    for extra in ([], ["--shards", "2"]):
        out = tmp_path / ("r" + "".join(extra))
        assert run("hsvd", "--in", tmp_path / "b", "--out", out, "--mode", "block",
                   "--block-cols", 16, *extra) == 0
        rec = (out / "record.csv").read_text().splitlines()[1].split(",")
        assert float(rec[6]) <= 1e-10  # max_rel_eig_err against lambda_true


# ---- gen / factor / bench (cli.py:92-106, 198-222) --------------------------
import hashlib  # noqa: E402
import json  # noqa: E402

_GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "factor.json")))


@pytest.mark.gpu
@pytest.mark.parametrize("case", _GOLD["cli_gen"], ids=lambda c: f"gen-{c['n']}-{c['seed']}")
def test_gen_bundle_byte_identical(tmp_path, case):
    args = ["gen", "--n", case["n"], "--seed", case["seed"], "--out", tmp_path / "b"]
    if case["pos_count"] is not None:
        args += ["--pos-count", case["pos_count"]]
    assert run(*args) == 0
    for name, h in case["files"].items():
        assert hashlib.sha256((tmp_path / "b" / name).read_bytes()).hexdigest() == h, name


@pytest.mark.gpu
def test_gen_factor_eig_pipeline(tmp_path):
    assert run("gen", "--n", 64, "--seed", 3, "--out", tmp_path / "b") == 0
    # factor M.gjh again: the same G as the bundle's (rounded M in, so the
    # factor may differ from G.gjh in the last bits; check the eigenvalues)
    assert run("factor", "--in", tmp_path / "b" / "M.gjh", "--out", tmp_path / "G2.gjh") == 0
    assert run("eig", "--in", tmp_path / "b", "--out", tmp_path / "r", "--mode", "block",
               "--block-cols", 16) == 0
    lam = np.sort(read_csv_matrix(tmp_path / "r" / "lambda.csv").ravel())
    lt = np.sort(read_csv_matrix(tmp_path / "b" / "lambda_true.csv").ravel())
    assert np.max(np.abs(lam - lt) / np.abs(lt)) <= 1e-12


@pytest.mark.gpu
def test_bench_records(tmp_path):
    assert run("bench", "--orders", "16,32", "--seed", 1, "--out", tmp_path / "rec.csv") == 0
    rows = (tmp_path / "rec.csv").read_text().splitlines()
    assert rows[0].startswith("n,r,p,sweeps") and len(rows) == 1 + 2 * 3 * 2


@pytest.mark.gpu
def test_factor_singular_exit_4(tmp_path):
    write_gjh(tmp_path / "M.gjh", np.ones((3, 3)), 3)
    assert run("factor", "--in", tmp_path / "M.gjh", "--out", tmp_path / "G.gjh") == 4


@pytest.mark.gpu
@pytest.mark.parametrize("shape,chunk", [((7, 4), 40), ((300, 256), 1 << 16), ((64, 64), 1 << 30)])
def test_gjh_device_streaming_round_trip(tmp_path, shape, chunk):
    """GJH1 straight to HBM through page-locked chunks (read_gjh_device) and
    back (write_gjh_device): bit-exact, the solver's (r, n) layout, the same
    bytes as the numpy writer, multi-chunk paths included."""
    import torch

    from paper_1008_1371_b200.matio import read_gjh_device, write_gjh_device
    M = np.random.default_rng(5).standard_normal(shape)
    write_gjh(tmp_path / "a.gjh", M, 3)
    Gt, p = read_gjh_device(tmp_path / "a.gjh", chunk_bytes=chunk)
    assert p == 3 and Gt.is_cuda and tuple(Gt.shape) == (shape[1], shape[0])
    assert np.array_equal(Gt.cpu().numpy().T, M)
    write_gjh_device(tmp_path / "b.gjh", Gt, 3, chunk_bytes=chunk)
    assert (tmp_path / "a.gjh").read_bytes() == (tmp_path / "b.gjh").read_bytes()
    # truncation is reported before any device work
    (tmp_path / "c.gjh").write_bytes((tmp_path / "a.gjh").read_bytes()[:-8])
    with pytest.raises(ValueError, match="truncated"):
        read_gjh_device(tmp_path / "c.gjh")
