"""Diagnostics: where the end-to-end (public API, host buffers) time goes on config 1."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd
from paper_2603_04070_b200.network import make_update_nets

torch.cuda.set_device(0)
wl, grid, geom, pulse, damp, bounds = bench.build_problem(1, 1, 0)
t0 = time.perf_counter()
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples, damp)
torch.cuda.synchronize()
print("engine create s", round(time.perf_counter() - t0, 3), eng.info())
nets = make_update_nets(5, seed=0, device="cuda")
eng.set_model(wl.c_true)
obs = eng.forward().double()
obs_host = pk.ChannelData(obs.cpu().numpy(), geom, grid.dt)
c0 = pk.SosMap(grid, np.full(grid.shape, 1540.0))
setup = pk.InversionSetup(pulse, damp, bounds)
for k in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pk.unfold_infer(obs_host, c0, nets, setup)
    torch.cuda.synchronize()
    print("unfold_infer s", round(time.perf_counter() - t0, 4))
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for k in range(3):
    pk.unfold_infer(obs_host, c0, nets, setup)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as p:
    pk.unfold_infer(obs_host, c0, nets, setup)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cpu_time_total", row_limit=25))
