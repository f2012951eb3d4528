"""The shard plan of the multi-GPU block solver, on CPU:
the C++ plan in libhsvd_b200 (hsvd_plan_*) is checked for its invariants
over many (blocks, shards) shapes, and the exchange protocol it drives --
one block column per shard and step over send/recv, the all-to-all column
redistribution after each sweep's sort -- is executed between two gloo
processes with labelled columns, so a wrong move shows up as a wrong label."""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1008_1371_b200 import _lib


class Plan:
    """Thin ctypes view of hsvd_plan_* (test helper)."""

    def __init__(self, nb, N):
        self.L = _lib.load()
        self.nb, self.N, self.S = nb, N, nb // 2
        self.h = self.L.hsvd_plan_create(nb, N)
        assert self.h, _lib.last_error()

    def advance(self):
        buf = np.zeros(5 * self.N + 5, np.int64)
        k = self.L.hsvd_plan_advance(self.h, buf.ctypes.data, self.N + 1)
        assert k >= 0, _lib.last_error()
        return [tuple(int(v) for v in buf[5 * i:5 * i + 5]) for i in range(k)]

    def state(self):
        ib = np.zeros(self.S, np.int64)
        jb = np.zeros(self.S, np.int64)
        ow = np.zeros(self.nb, np.int32)
        ar = np.zeros(self.nb, np.int32)
        s0 = np.zeros(self.N + 1, np.int64)
        self.L.hsvd_plan_state(self.h, ib.ctypes.data, jb.ctypes.data, ow.ctypes.data,
                               ar.ctypes.data, s0.ctypes.data)
        return ib, jb, ow, ar, s0

    def redistribute(self, b, rho_old, rho_new, g):
        r = len(rho_old)
        send = np.zeros(r, np.int64)
        recv = np.zeros(r, np.int64)
        sc = np.zeros(self.N, np.int64)
        rc = np.zeros(self.N, np.int64)
        ro = np.ascontiguousarray(rho_old, np.int64)
        rn = np.ascontiguousarray(rho_new, np.int64)
        self.L.hsvd_plan_redistribute(self.h, b, ro.ctypes.data, rn.ctypes.data, r, g,
                                      send.ctypes.data, sc.ctypes.data, recv.ctypes.data,
                                      rc.ctypes.data)
        return send[:sc.sum()], sc, recv[:rc.sum()], rc

    def place(self):
        self.L.hsvd_plan_place(self.h)

    def __del__(self):
        self.L.hsvd_plan_destroy(self.h)


def reference_pairs(nb, steps):
    """advance_stepper (_kernels.py:238-251) on nb block indices."""
    S = nb // 2
    ip = list(range(S))
    jp = [nb - k - 1 for k in range(S)]
    ib, jb = ip[:], jp[:]
    out = []
    for _ in range(steps):
        for k in range(S):
            if ip[k] + jp[k] >= nb - 1:
                ip[k] += 1
                if ip[k] == jp[k]:
                    ip[k] -= S
                    jp[k] = ip[k]
                ib[k] = ip[k]
            else:
                jp[k] += 1
                jb[k] = jp[k]
        out.append((ib[:], jb[:]))
    return out


def check_state(pl):
    ib, jb, ow, ar, s0 = pl.state()
    for k in range(pl.S):
        g = int(np.searchsorted(s0, k, side="right") - 1)
        assert ow[ib[k]] == g and ow[jb[k]] == g, "a pair is not resident on its shard"
    for g in range(pl.N):
        a = ar[ow == g]
        assert len(set(a.tolist())) == len(a), "two blocks share an area"
        m = s0[g + 1] - s0[g]
        assert len(a) == 2 * m and a.max() <= 2 * m


@pytest.mark.parametrize("nb", [4, 6, 8, 16, 34, 64, 256])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
def test_plan_invariants(nb, N):
    if nb // 2 < N:
        assert _lib.load().hsvd_plan_create(nb, N) is None
        return
    pl = Plan(nb, N)
    check_state(pl)
    ref = reference_pairs(nb, 3 * nb)
    for t in range(3 * nb):
        mv = pl.advance()
        ib, jb, *_ = pl.state()
        assert list(ib) == ref[t][0] and list(jb) == ref[t][1], "stepper differs from reference"
        ins = np.bincount([m[3] for m in mv], minlength=N)
        outs = np.bincount([m[1] for m in mv], minlength=N)
        assert ins.max(initial=0) <= 1 and (ins == outs).all()
        if N == 1:
            assert not mv
        if N > 1:  # the ring: every shard exchanges exactly one block per step
            assert (ins == 1).all()
        check_state(pl)


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_redistribution_counts(N):
    nb, b = 16, 4
    r = nb * b
    pl = Plan(nb, N)
    rng = np.random.default_rng(1)
    for t in range(nb):
        pl.advance()
    rho_old = rng.permutation(r)
    rho_new = rng.permutation(r)
    lists = [pl.redistribute(b, rho_old, rho_new, g) for g in range(N)]
    for g in range(N):
        for h in range(N):
            assert lists[g][1][h] == lists[h][3][g], "send/recv counts disagree"
    assert sum(len(x[0]) for x in lists) == r


# ---- the exchange protocol between two processes (gloo) -------------------

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nb, b, sweeps, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pl = Plan(nb, world)
        r = nb * b
        rng = np.random.default_rng(7)  # identical stream on every rank
        rho = rng.permutation(r)
        # storage: areas x b columns; a column's payload is its original index
        _, _, ow, ar, s0 = pl.state()
        A = 2 * (s0[rank + 1] - s0[rank]) + 1
        store = torch.full((A * b,), -1, dtype=torch.int64)
        for P in range(nb):
            if ow[P] == rank:
                store[ar[P] * b:(ar[P] + 1) * b] = torch.as_tensor(rho[P * b:(P + 1) * b])
        for sweep in range(sweeps):
            for step in range(nb):
                mv = pl.advance()
                reqs = []
                for (P, fr, fa, to, ta) in mv:
                    if fr == rank:
                        reqs.append(dist.isend(store[fa * b:(fa + 1) * b].clone(), to))
                    if to == rank:
                        buf = torch.empty(b, dtype=torch.int64)
                        reqs.append(("recv", dist.irecv(buf, fr), buf, ta))
                for x in reqs:
                    if isinstance(x, tuple):
                        x[1].wait()
                        store[x[3] * b:(x[3] + 1) * b] = x[2]
                    else:
                        x.wait()
                ib, jb, ow, ar, s0 = pl.state()
                for k in range(s0[rank], s0[rank + 1]):
                    for P in (ib[k], jb[k]):
                        got = store[ar[P] * b:(ar[P] + 1) * b].numpy()
                        assert (got == rho[P * b:(P + 1) * b]).all(), "wrong block resident"
            # sweep end: a new order (the sort), redistribute to the canonical placement
            rho_new = rng.permutation(r)
            send, sc, recv, rc = pl.redistribute(b, rho, rho_new, rank)
            pl.place()
            so = np.concatenate([[0], np.cumsum(sc)])
            ro = np.concatenate([[0], np.cumsum(rc)])
            newstore = torch.full_like(store, -1)
            reqs = []
            for h in range(world):
                out = store[torch.as_tensor(send[so[h]:so[h + 1]])].clone()
                if h == rank:
                    newstore[torch.as_tensor(recv[ro[h]:ro[h + 1]])] = out
                    continue
                if len(out):
                    reqs.append(dist.isend(out, h))
                if rc[h]:
                    buf = torch.empty(int(rc[h]), dtype=torch.int64)
                    reqs.append(("recv", dist.irecv(buf, h), buf, h))
            for x in reqs:
                if isinstance(x, tuple):
                    x[1].wait()
                    newstore[torch.as_tensor(recv[ro[x[3]]:ro[x[3] + 1]])] = x[2]
                else:
                    x.wait()
            store = newstore
            rho = rho_new
            ib, jb, ow, ar, s0 = pl.state()
            for k in range(s0[rank], s0[rank + 1]):
                for P in (ib[k], jb[k]):
                    got = store[ar[P] * b:(ar[P] + 1) * b].numpy()
                    assert (got == rho[P * b:(P + 1) * b]).all(), "redistribution wrong"
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as e:  # report to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("nb,b", [(8, 2), (16, 4), (34, 3)])
def test_gloo_exchange_world2(nb, b):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(k, 2, port, nb, b, 2, q)) for k in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
