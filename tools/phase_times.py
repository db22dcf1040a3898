"""Per-phase CUDA-event timing of one config-1 DUFWI reconstruction (diagnostics)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2603_04070_b200 import forward as fwd
from paper_2603_04070_b200.network import make_update_nets

torch.cuda.set_device(0)
wl, grid, geom, pulse, damp, bounds = bench.build_problem(1, 1, 0)
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples, damp)
nets = make_update_nets(5, seed=0, device="cuda")
eng.set_model(wl.c_true)
obs = eng.forward().double()
c = torch.full((1, grid.nx, grid.nz), 1540.0, dtype=torch.float64, device="cuda")
E = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(3):
    ev = [E() for _ in range(6)]
    ev[0].record()
    eng.set_model(c)
    ev[1].record()
    mis, g = eng.misfit_and_gradient(obs)
    ev[2].record()
    upd = nets[0].predict_update_device(c, g)
    ev[3].record()
    c2 = torch.clamp(c + upd, *bounds)
    ev[4].record()
    torch.cuda.synchronize()
    print([round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(4)], "ms: set_model, gradient, net, clamp")
prof = eng.time_sweeps(obs, reps=3)
print(prof)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as p:
    eng.misfit_and_gradient(obs)
    nets[0].predict_update_device(c, g)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=15))
