"""Diagnostics: wall-clock phases of one config-1 unfold_infer call (public API,
host arrays): upload of the observed traces and the initial map, graph replay,
download of the maps."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
import paper_2603_04070_b200 as pk
from paper_2603_04070_b200 import forward as fwd
from paper_2603_04070_b200 import unfold as uf
from paper_2603_04070_b200.network import make_update_nets

torch.cuda.set_device(0)
wl, grid, geom, pulse, damp, bounds = bench.build_problem(1, 1, 0)
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples, damp)
nets = make_update_nets(5, seed=0, device="cuda")
eng.set_model(wl.c_true)
obs = eng.forward().double()
obs_host = pk.ChannelData(obs.cpu().numpy(), geom, grid.dt)
c0 = pk.SosMap(grid, np.full(grid.shape, 1540.0))
setup = pk.InversionSetup(pulse, damp, bounds)
for _ in range(3):
    pk.unfold_infer(obs_host, c0, nets, setup)
rec = uf._reconstructor(eng, nets, setup.bounds, None, False, grid)
sync = torch.cuda.synchronize
for k in range(5):
    sync()
    t0 = time.perf_counter()
    o = uf._upload([obs_host.traces], eng.device)
    t1 = time.perf_counter()
    c = uf._upload([np.asarray(c0.values, dtype=np.float64)[None]], eng.device)
    t2 = time.perf_counter()
    maps = rec.reconstruct(o, c)
    t3 = time.perf_counter()
    host = uf._download(maps)
    t4 = time.perf_counter()
    out = [pk.SosMap(grid, host[k, 0]) for k in range(host.shape[0])]
    t5 = time.perf_counter()
    sync()
    t6 = time.perf_counter()
    tf = time.perf_counter()
    pk.unfold_infer(obs_host, c0, nets, setup)
    tg = time.perf_counter()
    print(f"upload obs {1e3*(t1-t0):.3f} ms, upload c {1e3*(t2-t1):.3f}, reconstruct(+sync) {1e3*(t3-t2):.3f}, "
          f"download {1e3*(t4-t3):.3f}, wrap {1e3*(t5-t4):.3f}; sum {1e3*(t5-t0):.3f}; full unfold_infer {1e3*(tg-tf):.3f}")
