"""Diagnostics: cProfile of config-1 unfold_infer calls (host side of the public API)."""
import cProfile
import pstats
import sys
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
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples, damp)
nets = make_update_nets(5, seed=0, device="cuda")
eng.set_model(wl.c_true)
obs_host = pk.ChannelData(eng.forward().double().cpu().numpy(), geom, grid.dt)
c0 = pk.SosMap(grid, np.full(grid.shape, 1540.0))
setup = pk.InversionSetup(pulse, damp, bounds)
for _ in range(4):
    pk.unfold_infer(obs_host, c0, nets, setup)
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    pk.unfold_infer(obs_host, c0, nets, setup)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(28)
