"""The sharded block solver on one GPU: the local
transport drives N shards -- each with its own storage, slots, stream and
Gram partition -- through the same plan, per-step ring exchange, sweep-end
norm all-gather, sort and all-to-all redistribution as the NCCL transport.
One shard must reproduce the one-GPU block solver bit for bit; N shards
must meet the same tolerance against the reference (oracle) and keep its
sweep count.  The NCCL transport itself runs at world size 1 (its
collectives and groups execute; there is no peer on a 1-GPU box)."""

import os
import socket

import numpy as np
import pytest
import torch

import paper_1008_1371_b200 as H
from oracle import oracle as O
from tests.block_metrics import residuals, sigma_class_reldiff
from tests.golden.inputs import make_case_input

pytestmark = pytest.mark.gpu

SIGMA_RTOL = 1e-10


def _assert_same(a, b):
    assert (a.sweeps_used, a.stop_reason) == (b.sweeps_used, b.stop_reason)
    assert (a.rotations, a.skips) == (b.rotations, b.skips)
    for f in ("sigma", "lam", "U", "Vinv_t"):
        x, y = getattr(a, f), getattr(b, f)
        assert (x is None and y is None) or np.array_equal(x, y), f


def _case(n, r, p, seed, kind="gauss"):
    G = make_case_input(n, r, seed, kind)
    signs = np.array([1] * p + [-1] * (r - p), np.int8)
    return G, signs, H.SignatureVector(signs, p)


@pytest.mark.parametrize("b", [16, 32])
def test_one_shard_is_the_one_gpu_solver(b):
    G, signs, J = _case(256, 256, 128, 0)
    cfg = H.SolverConfig(mode="block", block_cols=b)
    a = H.drive(G, J, cfg)
    s = H.drive_local_shards(G, J, cfg, nshards=1)
    assert s.sweeps_used == a.sweeps_used and s.stop_reason == a.stop_reason
    assert (s.rotations, s.skips) == (a.rotations, a.skips)
    for f in ("sigma", "lam", "U", "Vinv_t"):
        assert np.array_equal(getattr(s, f), getattr(a, f)), f


@pytest.mark.parametrize("case", [
    (256, 256, 128, 0, "gauss", 16, 2),
    (256, 256, 128, 0, "gauss", 16, 3),
    (512, 512, 384, 1, "gauss", 32, 2),
    (512, 512, 128, 2, "gauss", 32, 4),
    (520, 512, 200, 2, "gauss", 32, 8),
    (512, 512, 256, 0, "graded12", 32, 4),
    # >= 4 slots per shard: split-stream steps with the overlapped exchange
    (1024, 1024, 512, 4, "gauss", 32, 2),
    (1024, 1024, 700, 5, "gauss", 32, 3),
    (1024, 1024, 256, 6, "graded12", 16, 4),
], ids=lambda c: f"n{c[0]}r{c[1]}p{c[2]}{c[4]}b{c[5]}N{c[6]}")
def test_sharded_matches_reference(case):
    n, r, p, seed, kind, b, N = case
    G, signs, J = _case(n, r, p, seed, kind)
    cfg = H.SolverConfig(mode="block", block_cols=b)
    ref = O.drive(G, signs, p)
    one = H.drive(G, J, cfg)
    s = H.drive_local_shards(G, J, cfg, nshards=N)
    assert s.stop_reason in ("orthogonal", "quadratic")
    assert sigma_class_reldiff(s.sigma, s.lam, ref.sigma, ref.lam) <= SIGMA_RTOL
    # worker-count invariance (solver.py:127-131, test_solver.py:167-173):
    # the Gram's K segmentation depends on n only, so N shards give the
    # one-GPU solver's bits, sweeps and statistics
    _assert_same(s, one)


@pytest.mark.parametrize("N", [1, 2])
def test_sharded_split_matches_one_stream(N):
    """Split-stream steps (two slot halves + overlapped exchange per shard)
    against the one-stream sharded solver and the one-GPU solver: bit for
    bit."""
    G, signs, J = _case(1024, 1024, 512, 7)
    a = H.drive_local_shards(G, J, H.SolverConfig(mode="block", block_streams=1), nshards=N)
    b = H.drive_local_shards(G, J, H.SolverConfig(mode="block", block_streams=2), nshards=N)
    one = H.drive(G, J, H.SolverConfig(mode="block", block_streams=1))
    _assert_same(a, b)
    _assert_same(a, one)


@pytest.mark.parametrize("streams", [1, 2])
@pytest.mark.parametrize("graph", [False, True])
def test_one_gpu_stream_split_invariance(streams, graph):
    """One GPU: one stream vs two slot halves, eager vs graph replay: the
    same bits (the Gram's segmentation does not follow the launch)."""
    G, signs, J = _case(2048, 2048, 1024, 0)
    ref = H.drive(G, J, H.SolverConfig(mode="block", block_streams=2))
    x = H.drive(G, J, H.SolverConfig(mode="block", block_streams=streams, use_graph=graph))
    _assert_same(x, ref)


def test_sharded_n8_large_bit_identical():
    """8 local shards at n = 2048 (8 slots per shard, split steps): the
    one-GPU solver's bits."""
    G, signs, J = _case(2048, 2048, 1024, 0)
    cfg = H.SolverConfig(mode="block")
    _assert_same(H.drive_local_shards(G, J, cfg, nshards=8), H.drive(G, J, cfg))


def test_sharded_is_deterministic():
    G, signs, J = _case(256, 256, 100, 3)
    cfg = H.SolverConfig(mode="block", block_cols=16)
    a = H.drive_local_shards(G, J, cfg, nshards=4)
    b = H.drive_local_shards(G, J, cfg, nshards=4)
    assert np.array_equal(a.U, b.U) and np.array_equal(a.sigma, b.sigma)


def test_sharded_without_v():
    G, signs, J = _case(256, 256, 128, 0)
    cfg = H.SolverConfig(mode="block", block_cols=16, accumulate_v=False)
    s = H.drive_local_shards(G, J, cfg, nshards=2)
    full = H.drive_local_shards(G, J, H.SolverConfig(mode="block", block_cols=16), nshards=2)
    assert s.Vinv_t is None
    assert np.array_equal(s.sigma, full.sigma)


def test_sharded_errors():
    G, signs, J = _case(256, 256, 128, 0)
    G[:, 17] = 0.0
    with pytest.raises(H.RankDeficiencyError):
        H.drive_local_shards(G, J, H.SolverConfig(mode="block", block_cols=16), nshards=2)
    G, signs, J = _case(64, 64, 32, 0)
    with pytest.raises(NotImplementedError):  # 1 slot cannot feed 2 shards
        H.drive_local_shards(G, J, H.SolverConfig(mode="block", block_cols=32), nshards=2)


def test_nccl_transport_world1():
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        comm = H.ShardComm()
        G, signs, J = _case(256, 256, 128, 0)
        cfg = H.SolverConfig(mode="block", block_cols=16)
        part = H.drive_sharded(G, J, cfg, comm)
        full = H.gather_result(part, 256, 256)
        one = H.drive(G, J, cfg)
        for f in ("sigma", "lam", "U", "Vinv_t"):
            assert np.array_equal(getattr(full, f), getattr(one, f)), f
        comm.close()
    finally:
        dist.destroy_process_group()
