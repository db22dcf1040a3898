"""N>1 path on CPU: world_size-2 gloo processes shard (phantom, shot) units with
the engine's shard_range, each computes its partial imaging sum / misfit with the
float64 oracle, and the engine's combine_partials (one all_reduce of the packed
buffer) must reproduce the single-process gradient of every phantom."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2603_04070_b200.engine import combine_partials, shard_range

DX, DT = 1e-4, 2e-8


def _problem():
    rng = np.random.default_rng(5)
    pml, n, nt = 4, 20, 90
    N = n + 2 * pml
    B, S = 2, 3
    c = 1540.0 + rng.uniform(-20, 20, (B, N, N))
    d = oracle.pml_damping(N, N, pml, DX)
    t = np.arange(nt) * DT
    f = 1.5e6
    pulse = np.sin(2 * np.pi * f * (t - 2 / f)) * np.exp(-((t - 2 / f) * f) ** 2)
    el = np.stack([pml + 1 + 3 * np.arange(6), np.full(6, pml)], 1)
    tx = el[[0, 2, 5]]
    rx = np.repeat(el[None], S, axis=0)
    obs = []
    for b in range(B):
        tr, _ = oracle.forward_sweep(c[b] + 6.0, d, DX, DT, pulse, tx, rx)
        obs.append(tr)
    return c, d, pulse, el, tx, rx, np.concatenate(obs), B, S


def _partials(units, c, d, pulse, el, tx, rx, obs, S):
    """Unmasked, unscaled per-phantom partial sums for a unit range."""
    B, N = c.shape[0], c.shape[1]
    red = np.zeros(B * N * N + B + 1)
    acc = red[:B * N * N].reshape(B, N, N)
    for u in range(*units):
        b, s = divmod(u, S)
        m, g, _ = oracle.misfit_gradient(c[b], d, DX, DT, pulse, tx[s:s + 1], rx[s:s + 1],
                                         obs[u:u + 1], el, mask=False)
        acc[b] += g
        red[B * N * N + b] += m
    return red


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, d, pulse, el, tx, rx, obs, B, S = _problem()
        units = shard_range(B * S, rank, world)
        packed = torch.from_numpy(_partials(units, c, d, pulse, el, tx, rx, obs, S))
        combine_partials(packed)
        if rank == 0:
            q.put(packed.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_combine_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c, d, pulse, el, tx, rx, obs, B, S = _problem()
    full = _partials((0, B * S), c, d, pulse, el, tx, rx, obs, S)
    assert np.linalg.norm(got - full) <= 1e-13 * np.linalg.norm(full)
    # and equals the stacked reference-form gradient of each phantom
    N = c.shape[1]
    for b in range(B):
        m, g, _ = oracle.misfit_gradient(c[b], d, DX, DT, pulse, tx, rx, obs[b * S:(b + 1) * S], el,
                                         mask=False)
        assert np.linalg.norm(got[b * N * N:(b + 1) * N * N].reshape(N, N) - g) <= 1e-12 * np.linalg.norm(g)
        assert abs(got[B * N * N + b] - m) <= 1e-12 * m


# ------------------------------------------------- Reconstructor under gloo
class _StubEngine:
    """Host stand-in for PhysicsEngine: records the unit ranges it is asked for and
    returns a rank-dependent 'gradient' (what diverging replicated state would do)."""

    def __init__(self, rank, B=2, n=6):
        self.rank, self.B, self.n, self.n_units = rank, B, n, 4 * B
        self.calls = []

    def set_model(self, c, rho=None):
        self.c = c

    def misfit_and_gradient(self, obs, guard_radius=2, check_finite=True, units=None):
        self.calls.append(units)
        g = torch.full((self.B, self.n, self.n), 1e-3 * (1 + self.rank), dtype=torch.float64)
        return torch.zeros(self.B, dtype=torch.float64), g

    def last_flags(self):
        return torch.zeros(2, dtype=torch.int32)


class _RankNet:
    """Update network whose output differs per rank (e.g. other cuDNN algorithms)."""

    def __init__(self, rank):
        self.rank = rank

    def predict_update_device(self, c, g):
        return g * 1e3 + 0.25 * self.rank


def _recon_worker(rank, world, port, q):
    from paper_2603_04070_b200.unfold import Reconstructor

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        for collective in (True, False):
            eng = _StubEngine(rank)
            rec = Reconstructor(eng, [_RankNet(rank)] * 3, (1000.0, 2000.0), graph=False,
                                collective=collective)
            maps = rec.reconstruct(torch.zeros(8, 1, 1), torch.full((2, 6, 6), 1500.0))
            out[collective] = (np.stack([m.numpy() for m in maps]), eng.calls)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_reconstructor_collective_one_owner_per_phantom():
    """Collective reconstructions run each phantom's update on one rank and combine
    the stage maps with an all_reduce of exact zeros (ranks cannot diverge, no
    replicated network work); per-sample ones (collective=False) compute all
    units locally."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_recon_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    coll0, calls0 = got[0][True]
    coll1, calls1 = got[1][True]
    assert np.array_equal(coll0, coll1)  # the same bits on both ranks
    assert np.array_equal(coll0[0, 0], np.full((6, 6), 1500.0 + 1.0))  # rank 0's update: 1e-3*1e3 + 0
    assert np.array_equal(coll0[0, 1], np.full((6, 6), 1500.0 + 2.25))  # rank 1's: 2e-3*1e3 + 0.25
    assert calls0 == [None] * 3 and calls1 == [None] * 3  # sharded default ranges
    loc0, lcalls0 = got[0][False]
    loc1, _ = got[1][False]
    assert lcalls0 == [(0, 8)] * 3  # every unit, locally
    assert not np.array_equal(loc0, loc1)  # no hidden collective
