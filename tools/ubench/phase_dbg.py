import ctypes, os, sys
sys.path.insert(0, os.getcwd())
os.environ["DUFWI_LIB"] = os.path.abspath("tools/ubench/lib_TIMING.so")
import torch, numpy as np
import bench
from paper_2603_04070_b200 import forward as fwd, _lib
torch.cuda.set_device(0)
wl, grid, geom, pulse, damp, bounds = bench.build_problem(1, 1, 0)
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples, damp, engine="cluster")
eng.set_model(wl.c_true)
so = _lib.lib()
buf = (ctypes.c_ulonglong * 256)()
eng.forward(); so.dufwi_debug_counters(buf, 256)
obs = eng.forward().double(); so.dufwi_debug_counters(buf, 256)
print("warp: [sync+wait, compute, fast steps/1000] cycles per step, loop cycles per step")
for w in range(15):
    print(w, [round(buf[w * 4 + k] / 1000.0) for k in range(4)], "loop", round(buf[128 + w] / 1000.0))
