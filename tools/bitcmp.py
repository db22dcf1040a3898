"""Dump traces and gradient of a short config run (diagnostics: compare library
builds bit for bit).  usage: bitcmp.py CONFIG UNITS NT OUT.txt [STORE] [norho] (sha256 per array)   (DUFWI_LIB selects the build)"""
import dataclasses
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import configs
from paper_2603_04070_b200 import forward as fwd

cfg, units, nt, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
store = sys.argv[5] if len(sys.argv) > 5 else "auto"
norho = len(sys.argv) > 6 and sys.argv[6] == "norho"
torch.cuda.set_device(0)
spec = dataclasses.replace(configs.get_config(cfg), nt=nt)
B = max(1, -(-units // spec.n_tx))
wl = configs.make_workload(spec, seed=0, n_phantoms=B)
if norho:
    wl = dataclasses.replace(wl, rho=None)
grid = pk.Grid2D(spec.n, spec.n, spec.dx, spec.dt, spec.nt)
geom = pk.AcquisitionGeometry(grid, wl.nodes, wl.rx, 0.0, tx_elements=wl.tx)
damp = pk.build_pml(grid, spec.pml)
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, wl.pulse, damp,
                     n_phantoms=B, has_rho=wl.rho is not None, engine=os.environ.get("BITCMP_ENGINE", "stepwise"))
eng.set_model(wl.c_true, wl.rho)
obs = eng.forward(units=(0, eng.n_units)).double()
c1 = wl.c_true * 0.999 + 1.5
eng.set_model(c1, wl.rho)
mis, g = eng.misfit_and_gradient(obs, store=store)
import hashlib  # noqa: E402
arrs = {"obs": obs.cpu().numpy(), "mis": mis.cpu().numpy(), "g": g.cpu().numpy()}
with open(out, "w") as f:
    for k, a in arrs.items():
        f.write(f"{k} {hashlib.sha256(a.tobytes()).hexdigest()[:16]} {float(np.abs(a).max()):.6e}\n")
