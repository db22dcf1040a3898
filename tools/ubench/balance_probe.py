"""Probe: cluster sweep times on config 0 with the x damping ramp removed (z ramp
only), i.e. with every CTA of a cluster carrying the same share of damped cells,
against the real PML.  If the two end CTAs that lie in the x band set the pace,
the balanced case shows how much a balanced row assignment could gain."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import bench
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd

torch.cuda.set_device(0)
wl, grid, geom, pulse, damp, bounds = bench.build_problem(0, 1, 0)
px, pz = damp.profiles
cases = {"pml": damp,
         "z_only": pk.DampingProfile(grid, np.maximum(np.zeros_like(px)[:, None], pz[None, :])),
         "none": pk.zero_damping(grid)}
for name, d in cases.items():
    eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples, d,
                         engine="cluster")
    eng.set_model(wl.c_true)
    obs = torch.zeros((eng.n_units, geom.n_r, grid.nt), dtype=torch.float64, device="cuda")
    for store in ("lap", "strips"):
        try:
            p = eng.time_sweeps(obs, reps=3, store=store)
            print(name, store, "fwd %.4f adj %.4f" % (p["forward_ms"], p["adjoint_ms"]), eng.info()["cluster_ctas"],
                  eng.info()["rows_per_thread"])
        except Exception as e:  # noqa: BLE001
            print(name, store, "failed", str(e)[:80])
