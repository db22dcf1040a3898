"""The torch.distributed paths on the device: two gloo ranks, both on cuda:0
(the sharded sweeps of one rank never wait on the other's kernels; only the
host-side all_reduce / broadcast couple them).

* PhysicsEngine.misfit_and_gradient with the default unit range is a collective:
  units are sharded, partials combined with one all_reduce.  With one phantom
  per rank the sum adds exact zeros, so the result equals the single-process
  gradient bit for bit.
* The per-sample public misfit_and_gradient is NOT a collective: every rank
  gets the single-process value (not world_size times it).
* unfold_infer_batch is a collective: each phantom's update network runs on one
  rank and the stage maps are combined with an all_reduce of exact zeros, so all
  ranks return the same bits; against the single-process call the maps agree to
  the rounding of the fp32 networks (cuDNN may pick another algorithm for a batch
  of one than for the batch of all phantoms), the physics bit for bit.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case():
    import paper_2603_04070_b200 as pk
    from tests._cases import small_linear

    wl, grid, geom, pulse, damp = small_linear(n=40, pml=6, nt=220, seed=6)
    truths = [wl.c_true[0], wl.c_true[0] * 0.998 + 4.0]
    obs = [pk.simulate_all(pk.SosMap(grid, c), geom, pulse, damp) for c in truths]
    c0 = [pk.homogeneous_map(grid, 1540.0), pk.homogeneous_map(grid, 1535.0)]
    return pk, grid, geom, pulse, damp, obs, c0


def _compute():
    import torch

    from paper_2603_04070_b200 import forward as fwd
    from paper_2603_04070_b200.network import make_update_nets

    pk, grid, geom, pulse, damp, obs, c0 = _case()
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                         pulse.samples, damp, n_phantoms=2)
    eng.set_model(np.stack([c.values for c in c0]))
    o = torch.as_tensor(np.concatenate([x.traces for x in obs])).to(eng.device)
    mis, g = eng.misfit_and_gradient(o)  # collective under torch.distributed
    m1, g1 = pk.misfit_and_gradient(c0[0], obs[0], pulse, damp)  # never a collective
    nets = make_update_nets(2, seed=2, device=eng.device)
    setup = pk.InversionSetup(pulse, damp, (1300.0, 1800.0))
    maps = pk.unfold_infer_batch(obs, c0, nets, setup)
    return {"mis": mis.cpu().numpy(), "g": g.cpu().numpy(), "m1": np.float64(m1),
            "g1": g1.values, "maps": np.stack([[m.values for m in per] for per in maps])}


def _worker(rank, world, port, q):
    import sys

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.getcwd())
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _compute()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_match_single_process(gpu):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = _compute()
    for r in (0, 1):
        out = got[r]
        assert np.array_equal(out["mis"], single["mis"]), r
        assert np.array_equal(out["g"], single["g"]), r
        assert out["m1"] == single["m1"] and np.array_equal(out["g1"], single["g1"]), r
        err = np.linalg.norm(out["maps"] - single["maps"]) / np.linalg.norm(single["maps"])
        assert err <= 1e-6, (r, err)
        # stage 1 sees the same gradient bits; only the network's batch shape differs
        err1 = np.abs(out["maps"][:, 0] - single["maps"][:, 0]).max()
        assert err1 <= 1e-3, (r, err1)  # m/s
    assert np.array_equal(got[0]["maps"], got[1]["maps"])
