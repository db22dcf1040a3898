"""Generate the full-size parity fixtures under ``tests/golden/large/``.

TEST INFRASTRUCTURE.  Runs the C float64 checker (``oracle/c_oracle.py``, a
restatement of forward.py:273-313 / adjoint.py:94-138 / unfold.py:253-267
pinned bit-for-bit on traces against the NumPy restatement, which is itself
pinned against the reference) at BASELINE.json's stated sizes, with f64
snapshot checkpointing in place of the reference's full field history:

  A  config 3 gradient: 560^2, nt 4000, variable density, 2 transmits, fixed
     float64 observations of the true model (stored as f32; the oracle's
     gradient uses exactly the stored f32 values)
  B  config 4 gradient: 1088^2, nt 6000, 2 phantoms x 2 transmits, each side
     simulating its own observations (SURVEY §8(c) protocol)
  C  config 2 DUFWI: K = 5, phantoms 0 and 1 of the batch of 8, density,
     f64 copies of the seeded stage networks, own observations
  D  config 3 DUFWI: K = 3, all 128 transmits, density, own observations

Every fixture holds f32 gradients, f64 misfits, f32 traces decimated in time
(every ``DEC``-th sample: exact values, for trace parity) and sha256 of the
full f64 traces.  Usage (build container; takes ~1 h on 8 cores):

    python oracle/make_golden_large.py [A B C D]
"""

from __future__ import annotations

import copy
import dataclasses
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
OUT = ROOT / "tests" / "golden" / "large"
DEC = 8  # time decimation of the stored traces

import oracle  # noqa: E402
from oracle import c_oracle as co  # noqa: E402
from paper_2603_04070_b200 import configs  # noqa: E402

# transmits used by the partial-shot cases (spread across the aperture)
SHOTS_A = (20, 100)
SHOTS_B = (37, 200)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def setup(cfg: int, n_phantoms: int, shots=None):
    spec = configs.get_config(cfg)
    wl = configs.make_workload(spec, seed=0, n_phantoms=n_phantoms)
    d = oracle.pml_damping(spec.n, spec.n, spec.pml, spec.dx)
    sel = np.arange(len(wl.tx)) if shots is None else np.asarray(shots)
    tx = wl.nodes[wl.tx[sel]]
    rx = wl.nodes[wl.rx[sel]]
    return spec, wl, d, sel, tx, rx


def cfl_bounds(spec, lo=1300.0, hi=3200.0):
    """unfold.py:117-131 (cfl_safe_bounds, safety 0.999)."""
    limit = 0.999 * spec.dx / (spec.dt * np.sqrt(2.0))
    return (lo, min(hi, limit))


def nets_f64(k: int, seed: int = 0):
    from paper_2603_04070_b200.network import make_update_nets

    nets = make_update_nets(k, seed=seed)
    h = hashlib.sha256()
    for n in nets:
        for p in n.parameters():
            h.update(p.detach().cpu().numpy().tobytes())
    return [copy.deepcopy(n).double() for n in nets], h.hexdigest()


def case_a(meta):
    spec, wl, d, sel, tx, rx = setup(3, 1, SHOTS_A)
    rho = wl.rho[0]
    t0 = time.time()
    obs64, _ = co.forward_sweep(wl.c_true[0], d, spec.dx, spec.dt, wl.pulse, tx, rx, rho=rho)
    obs32 = obs64.astype(np.float32)
    c0 = np.full(d.shape, 1540.0)
    mis, g, trial = co.misfit_gradient(c0, d, spec.dx, spec.dt, wl.pulse, tx, rx,
                                       obs32.astype(np.float64), wl.nodes, rho=rho)
    np.savez_compressed(OUT / "config3_grad.npz", shots=np.asarray(SHOTS_A), obs_f32=obs32,
                        grad=g.astype(np.float32), misfit=mis,
                        trial_dec=trial[:, :, ::DEC].astype(np.float32))
    meta["A_config3_grad"] = {"shots": list(SHOTS_A), "nt": spec.nt, "density": True,
                              "misfit": mis, "obs_sha256_f64": sha(obs64),
                              "trial_sha256_f64": sha(trial), "grad_sha256_f64": sha(g),
                              "seconds": time.time() - t0}


def case_b(meta):
    spec, wl, d, sel, tx, rx = setup(4, 2, SHOTS_B)
    t0 = time.time()
    c0 = np.full(d.shape, 1540.0)
    grads, mis, obs_dec, trial_dec, info = [], [], [], [], []
    for b in range(2):
        obs, _ = co.forward_sweep(wl.c_true[b], d, spec.dx, spec.dt, wl.pulse, tx, rx)
        m, g, trial = co.misfit_gradient(c0, d, spec.dx, spec.dt, wl.pulse, tx, rx, obs, wl.nodes)
        grads.append(g.astype(np.float32))
        mis.append(m)
        obs_dec.append(obs[:, :, ::DEC].astype(np.float32))
        trial_dec.append(trial[:, :, ::DEC].astype(np.float32))
        info.append({"obs_sha256_f64": sha(obs), "trial_sha256_f64": sha(trial),
                     "grad_sha256_f64": sha(g)})
    np.savez_compressed(OUT / "config4_grad.npz", shots=np.asarray(SHOTS_B), grad=np.stack(grads),
                        misfit=np.asarray(mis), obs_dec=np.stack(obs_dec),
                        trial_dec=np.stack(trial_dec))
    meta["B_config4_grad"] = {"shots": list(SHOTS_B), "phantoms": [0, 1], "nt": spec.nt,
                              "misfit": mis, "per_phantom": info, "seconds": time.time() - t0}


def dufwi_case(cfg: int, n_phantoms: int, out_name: str, key: str, meta):
    spec, wl, d, sel, tx, rx = setup(cfg, n_phantoms)
    bounds = cfl_bounds(spec)
    nets, wsha = nets_f64(spec.k_stages, seed=0)
    upd = [lambda c, g, n=n: n.predict_update(c, g) for n in nets]
    t0 = time.time()
    S = len(tx)
    sel_dec = np.array([0, S // 2, S - 1])  # transmits whose decimated traces are kept
    grads, maps, obs_dec, info = [], [], [], []
    for b in range(n_phantoms):
        rho = wl.rho[b] if wl.rho is not None else None
        obs, _ = co.forward_sweep(wl.c_true[b], d, spec.dx, spec.dt, wl.pulse, tx, rx, rho=rho)
        c0 = np.full(d.shape, 1540.0)
        mk, gk = co.unfold_reconstruct(obs, c0, upd, bounds, d, spec.dx, spec.dt, wl.pulse, tx, rx,
                                       wl.nodes, rho=rho)
        grads.append(np.stack(gk).astype(np.float32))
        maps.append(np.stack(mk).astype(np.float32))
        obs_dec.append(obs[sel_dec, :, ::DEC].astype(np.float32))
        info.append({"obs_sha256_f64": sha(obs), "final_sha256_f64": sha(mk[-1]),
                     "update_absmax": [float(np.abs(mk[i] - (mk[i - 1] if i else np.clip(c0, *bounds))).max())
                                       for i in range(len(mk))]})
        print(f"[{key}] phantom {b} done {time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(OUT / out_name, grads=np.stack(grads), maps=np.stack(maps),
                        obs_dec=np.stack(obs_dec), obs_dec_shots=sel_dec, bounds=np.asarray(bounds))
    meta[key] = {"config": cfg, "phantoms": list(range(n_phantoms)), "K": spec.k_stages,
                 "net_seed": 0, "net_weights_sha256_f32": wsha, "bounds": list(bounds),
                 "per_phantom": info, "seconds": time.time() - t0}


def main(which):
    OUT.mkdir(parents=True, exist_ok=True)
    mpath = OUT / "meta.json"
    meta = json.loads(mpath.read_text()) if mpath.exists() else {}
    meta["numpy"] = np.__version__
    meta["threads"] = co.default_threads()
    meta["trace_decimation"] = DEC
    runs = {"A": lambda: case_a(meta), "B": lambda: case_b(meta),
            "C": lambda: dufwi_case(2, 2, "config2_dufwi.npz", "C_config2_dufwi", meta),
            "D": lambda: dufwi_case(3, 1, "config3_dufwi.npz", "D_config3_dufwi", meta)}
    for w in which:
        t = time.time()
        runs[w]()
        mpath.write_text(json.dumps(meta, indent=1, sort_keys=True))
        print(f"[{w}] written in {time.time() - t:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["A", "B", "C", "D"])
