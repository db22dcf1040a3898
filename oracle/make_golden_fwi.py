"""Golden fixtures for the ADMM-TV FWI row, made by running the
REAL reference package.  TEST INFRASTRUCTURE, build container only:

    python oracle/make_golden_fwi.py

Writes tests/golden/fwi.npz:
* ``fwilab.fwi.tv_prox`` on a seeded 12x14 map (weight 0.7, 20 iterations) and
  ``total_variation`` of it;
* ``fwilab.fwi.lbfgs_minimize`` on a seeded convex quadratic (7 steps, memory 3,
  projection onto a box);
* ``fwilab.fwi.admm_fwi`` on the ring48 case (tests/golden/ring48.npz geometry,
  PML 8): 3 outer x 3 inner iterations from the homogeneous map, final map and
  misfit log.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = "/root/reference/pkg/src"
OUT = ROOT / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import fwilab as fw
    from fwilab import fwi

    rng = np.random.default_rng(77)
    v = 1500.0 + 20.0 * rng.standard_normal((12, 14))
    tv_out = fwi.tv_prox(v, 0.7, iters=20)

    n = 30
    M = rng.standard_normal((n, n))
    A = M @ M.T / n + np.eye(n)
    b = rng.standard_normal(n)

    def quad(x):
        xf = x.ravel()
        return float(0.5 * xf @ A @ xf - b @ xf), (A @ xf - b).reshape(x.shape)

    x0 = rng.standard_normal((5, 6))
    lb_x, lb_vals = fwi.lbfgs_minimize(quad, x0, iters=7, lr=0.8, memory=3,
                                       project=lambda x: np.clip(x, -0.5, 0.5))

    z = np.load(OUT / "ring48.npz")
    grid = fw.Grid2D(nx=48, nz=48, dx=float(z["dx"]), dt=float(z["dt"]), nt=z["pulse"].shape[0])
    geom = fw.build_geometry(8, 0.028, 3, grid)
    assert np.array_equal(geom.element_nodes, z["nodes"])
    pulse = fw.make_source_pulse(2e5, grid.dt, grid.nt)
    damp = fw.build_pml(grid, 8)
    obs = fw.ChannelData(z["obs"], geom, grid.dt)
    c0 = fw.homogeneous_map(grid, 1500.0)
    cfg = fwi.FwiConfig(outer_iters=3, inner_lbfgs_iters=3)
    c_fin, log = fwi.admm_fwi(obs, c0, cfg, pulse, damp)
    np.savez_compressed(OUT / "fwi.npz", tv_in=v, tv_weight=0.7, tv_out=tv_out,
                        tv_value=fwi.total_variation(tv_out), quad_A=A, quad_b=b, lb_x0=x0,
                        lb_x=lb_x, lb_values=np.array(lb_vals), admm_map=c_fin.values,
                        admm_log=np.array(log), admm_outer=3, admm_inner=3)
    print("wrote fwi.npz; admm log", log)


if __name__ == "__main__":
    main()
