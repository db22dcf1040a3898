"""Forward / adjoint sweep times of the config-1 problem (CUDA events; diagnostics).
DUFWI_LIB selects the library build under test."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import bench
from paper_2603_04070_b200 import forward as fwd

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
torch.cuda.set_device(0)
wl, grid, geom, pulse, damp, bounds = bench.build_problem(cfg, 1, 0)
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples, damp)
eng.set_model(wl.c_true)
obs = eng.forward().double()
for _ in range(2):
    prof = eng.time_sweeps(obs, reps=5)
print(f"forward_ms {prof['forward_ms']:.4f} adjoint_ms {prof['adjoint_ms']:.4f} {eng.info()}")
