"""Every stepwise kernel family and history store against the float64 oracle.

The f32 tile kernels (default arithmetic) and the f64 lean kernels (arith="f64")
cover nz % 4 == 0 grids with separable damping and a rectangular undamped box
(all BASELINE configs).  The others are reached by inputs a user of the
reference can hand over:
  * nz % 4 != 0                       -> stream kernels (with and without density)
  * a damping map that is not max(px, pz) (DampingProfile(grid, values) from disk)
                                       -> vec kernels (constant density), stream (density)
  * no rectangular undamped box        -> no strips: full history or checkpointing
A plain build_pml map handed over without its profiles is recognised as
separable and takes the lean kernels.  Checkpointing recomputes the same f32
fields as the first forward, so its gradient equals full storage bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd

from ._cases import rel_l2, small_linear

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _sum_damping(grid, pml, island=False):
    """Non-separable damping: px[i] + pz[j] (same undamped box as build_pml), optionally
    with a damped 3x3 island far from the array (no rectangular box left)."""
    prof = pk.build_pml(grid, pml).profiles
    d = prof[0][:, None] + prof[1][None, :]
    if island:
        cx, cz = grid.nx // 2, grid.nz - pml - 8
        d[cx - 1:cx + 2, cz - 1:cz + 2] = 2.0e6
    return pk.DampingProfile(grid, d)


CASES = {
    # name: (small_linear kwargs, damping builder, expected kernel family, stores)
    "nz_odd": (dict(n=41), None, "stream", ("full", "strips", "checkpoint")),
    "nz_odd_rho": (dict(n=41, rho=True), None, "stream", ("full", "strips", "checkpoint")),
    "sum_damping": (dict(n=40), "sum", "vec", ("full", "strips", "checkpoint")),
    "sum_damping_rho": (dict(n=40, rho=True), "sum", "stream", ("full", "strips")),
    "island": (dict(n=40), "island", "vec", ("full", "checkpoint")),
    "island_rho": (dict(n=40, rho=True), "island", "stream", ("full", "checkpoint")),
    "tile": (dict(n=40), None, "tile", ("strips", "checkpoint", "full")),
    "tile_rho": (dict(n=40, rho=True), None, "tile", ("strips", "checkpoint", "full")),
    "lean_f64": (dict(n=40), None, "lean", ("strips", "checkpoint", "full")),
    "lean_f64_rho": (dict(n=40, rho=True), None, "lean", ("strips", "full")),
}


@pytest.mark.parametrize("name", list(CASES))
def test_stepwise_family_vs_oracle(gpu, name):
    kw, dkind, family, stores = CASES[name]
    wl, grid, geom, pulse, damp = small_linear(pml=6, nt=240, n_el=12, n_tx=3, seed=4, **kw)
    if dkind is not None:
        damp = _sum_damping(grid, 6, island=dkind == "island")
        assert damp.profiles is None
    rho = wl.rho[0] if wl.rho is not None else None
    tx, rx = geom.tx_nodes(), geom.rx_nodes()
    obs, _ = oracle.forward_sweep(wl.c_true[0], damp.values, grid.dx, grid.dt, pulse.samples, tx,
                                  rx, rho=rho)
    # trial model 20 m/s below the background: residual/trace L2 3.7% (config 0: 1.3%);
    # a 1540 start leaves 5e-4, where f32 storage rounding alone exceeds 1e-4
    c0 = np.full(grid.shape, 1520.0)
    m_ref, g_ref, tr_ref = oracle.misfit_gradient(c0, damp.values, grid.dx, grid.dt, pulse.samples,
                                                  tx, rx, obs, geom.element_nodes, rho=rho)
    eng = fwd.get_engine(grid, tx, rx, geom.element_nodes, pulse.samples, damp,
                         has_rho=rho is not None, engine="stepwise",
                         arith="f64" if name.startswith("lean_f64") else "f32")
    assert eng.info()["stepwise_kernels"] == family
    assert (eng.box is None) == (dkind == "island")
    eng.set_model(wl.c_true, None if rho is None else rho[None])
    assert rel_l2(eng.forward().cpu().numpy(), obs) <= TOL
    eng.set_model(c0[None], None if rho is None else rho[None])
    grads = {}
    for store in stores:
        mis, g, tr = eng.misfit_and_gradient(torch.as_tensor(obs).to(gpu), store=store,
                                             return_traces=True)
        assert eng.last_engine == "stepwise"
        grads[store] = g[0].cpu().numpy()
        assert rel_l2(tr.cpu().numpy(), tr_ref) <= TOL, store
        assert rel_l2(grads[store], g_ref) <= TOL, store
        assert abs(float(mis[0]) - m_ref) <= TOL * m_ref, store
    if "checkpoint" in grads and "full" in grads:
        assert np.array_equal(grads["checkpoint"], grads["full"])


def test_pml_values_without_profiles_take_the_lean_kernels(gpu):
    """DampingProfile(grid, values) of a build_pml map (e.g. read from disk) is
    recognised as separable: same kernels and bits as build_pml's own profile."""
    wl, grid, geom, pulse, damp = small_linear(n=40, pml=6, nt=200, seed=2)
    plain = pk.DampingProfile(grid, np.array(damp.values))
    assert plain.profiles is not None
    assert np.array_equal(np.maximum(plain.profiles[0][:, None], plain.profiles[1][None, :]),
                          damp.values)
    c = pk.SosMap(grid, wl.c_true[0])
    a = pk.simulate_all(c, geom, pulse, damp)
    b = pk.simulate_all(c, geom, pulse, plain)
    assert np.array_equal(a.traces, b.traces)
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                         pulse.samples, plain, engine="stepwise")
    assert eng.info()["stepwise_kernels"] == "tile"
    eng64 = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                           pulse.samples, plain, engine="stepwise", arith="f64")
    assert eng64.info()["stepwise_kernels"] == "lean"


def test_checkpoint_auto_when_full_history_does_not_fit(gpu):
    """auto store without a rectangular box falls back to checkpointing when one
    unit's full history exceeds the memory budget."""
    wl, grid, geom, pulse, damp = small_linear(n=40, pml=6, nt=240, seed=4)
    damp = _sum_damping(grid, 6, island=True)
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                         pulse.samples, damp, engine="stepwise")
    from paper_2603_04070_b200.engine import STORE_CHECKPOINT, STORE_FULL

    eng._auto_store.clear()
    assert eng.pick_store(True) == STORE_FULL
    frac = eng.memory_fraction
    try:
        eng.memory_fraction = 1e-9
        eng._auto_store.clear()
        assert eng.pick_store(True) == STORE_CHECKPOINT
    finally:
        eng.memory_fraction = frac
        eng._auto_store.clear()
