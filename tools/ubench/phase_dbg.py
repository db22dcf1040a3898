"""Per-warp step timing of the cluster sweeps (library built with -DDUFWI_EXP_TIMING):
CTA rank 0 (x damping band) and rank DUFWI_DBG_RANK (default 4, interior; the library must be
built with the same -DDUFWI_DBG_RANK) of the first cluster."""
import ctypes
import os
import sys

sys.path.insert(0, os.getcwd())
os.environ.setdefault("DUFWI_LIB", os.path.abspath("tools/ubench/lib_TIMING.so"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_04070_b200 import _lib, forward as fwd  # noqa: E402

torch.cuda.set_device(0)
wl, grid, geom, pulse, damp, bounds = bench.build_problem(1, 1, 0)
eng = fwd.get_engine(grid, geom.tx_nodes(), geom.rx_nodes(), geom.element_nodes, pulse.samples,
                     damp, engine="cluster")
print(eng.info())
eng.set_model(wl.c_true)
obs = eng.forward().double()
so = _lib.lib()
buf = (ctypes.c_ulonglong * 512)()
eng.misfit_and_gradient(obs)
so.dufwi_debug_counters(buf, 512)
eng.misfit_and_gradient(obs)
so.dufwi_debug_counters(buf, 512)
nt = grid.nt
paths = {0: "plain", 1: "full", 2: "generic", 3: "unif", 4: "xpml", 5: "io-plain"}
for sweep in (0, 1):
    print(["forward", "adjoint"][sweep], "cycles per step: before the body [of which __syncthreads, halo wait] / body, path")
    for cta in (0, 1):
        row = []
        for w in range(32):
            d = ((sweep * 2 + cta) * 32 + w) * 4
            p = round(buf[d + 2] / nt)
            bar_c, halo_c = (buf[d + 3] & 0xffffffff) // nt, (buf[d + 3] >> 32) // nt
            row.append(f"{buf[d] // nt}[bar {bar_c} halo {halo_c}]/{buf[d + 1] // nt}{paths.get(p, '?')[0]}")
        print("  cta", [0, int(os.environ.get("DUFWI_DBG_RANK", "4"))][cta], " ".join(row))
