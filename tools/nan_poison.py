"""Debug aid: poison torch's caching allocator with NaN, then run small
gradient cases on both engines and stores — any read of uninitialised
workspace shows up as a non-finite result."""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_04070_b200 as pk  # noqa: E402
from paper_2603_04070_b200 import forward as fwd  # noqa: E402
from tests._cases import gradcheck16, ring48, rel_l2  # noqa: E402


def poison():
    x = torch.full((1 << 28,), float("nan"), device="cuda")
    del x
    torch.cuda.synchronize()


def run(name, z, grid, geom, pulse, damp):
    for engine in ("cluster", "stepwise"):
        for store in ("full", "strips", "auto"):
            poison()
            fwd._ENGINE_CACHE.clear()
            eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes,
                                 pulse.samples, damp, n_phantoms=1, engine=engine)
            eng.set_model(z["c0"][None])
            try:
                mis, g = eng.misfit_and_gradient(torch.as_tensor(z["obs"]).cuda(), store=store)
                print(name, engine, store, "rel", rel_l2(g[0].cpu().numpy(), z["grad"]), flush=True)
            except Exception as e:  # noqa: BLE001
                print(name, engine, store, "ERR", type(e).__name__, e, flush=True)


z, grid, geom, pulse = gradcheck16()
run("gc16", z, grid, geom, pulse, pk.zero_damping(grid))
z, grid, geom, pulse, damp = ring48()
run("ring48", z, grid, geom, pulse, damp)
