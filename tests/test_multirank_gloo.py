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
