"""Generate tests/golden/mc_small.npz from the reference Monte-Carlo harness (simulate.py).

Run in the build container, where the reference imports from /root/reference/pkg/src:
    python tests/golden/make_mc_golden.py
Records, for a small (kappa, SNR, method) sweep: the reference's demo geometry, every
realization's synthesized pixel and nested solver seed (simulate.py:309-329), the per-realization
detection outcome of run_pipeline_realization, and the per-cell DetectionResult fields.
"""
import os
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from tomobpdn import simulate as S  # noqa: E402
from tomobpdn.model import ParameterGrid, build_steering_matrix  # noqa: E402
from tomobpdn.rng import derive_seed, substream  # noqa: E402
from tomobpdn.solver import SolverConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mc_small.npz")
KAPPAS = [0.5, 1.0, 1.5]
SNRS = [6.0, 20.0]
METHODS = ["fista", "rbpg", "svd_wiener"]
R = 24
SEED = 31


def main():
    geom = S.demo_geometry()
    base = S.Scenario(geometry=geom, seed=SEED)
    out = {"baselines": geom.baselines, "times": geom.times, "kappas": np.array(KAPPAS), "snrs": np.array(SNRS),
           "methods": np.array(METHODS), "realizations": np.array(R), "seed": np.array(SEED)}
    for tag, dphi in (("phi0", 0.0), ("phirand", None)):
        setup = S.MonteCarloSetup(delta_phi=dphi, solver=SolverConfig(max_iters=300, tol=1e-6))
        unit = S.separation_unit(geom)
        grid = ParameterGrid.uniform((-setup.grid_halfspan * unit, setup.grid_halfspan * unit), setup.grid_size)
        a = build_steering_matrix(geom, grid).entries
        tol = setup.tol_factor * unit
        cells = [(k, s, m) for k in KAPPAS for s in SNRS for m in METHODS]
        pix, seeds, oks = [], [], []
        for c, (k, s, m) in enumerate(cells):
            for r in range(R):
                sid = c * R + r
                rng = substream(SEED, sid)
                ph = float(rng.uniform(0.0, 2.0 * np.pi)) if dphi is None else dphi
                half = k * S.separation_unit(geom) / 2.0
                truth = replace(base, scatterers=(S.Scatterer(S._snap(grid, -half), amplitude=1.0, phase=0.0),
                                                  S.Scatterer(S._snap(grid, half), amplitude=1.0, phase=ph)),
                                snr_db=(s, s), motion_bases=())
                pix.append(S.synthesize_pixel(truth, rng))
                seeds.append(derive_seed(rng))
                oks.append(S.run_pipeline_realization(base, a, grid, k, s, m, setup, tol, sid))
        res = S.monte_carlo_detection(base, KAPPAS, SNRS, METHODS, R, setup)
        out[f"{tag}/pixels"] = np.array(pix)
        out[f"{tag}/seeds"] = np.array(seeds, dtype=np.uint64)
        out[f"{tag}/outcomes"] = np.array(oks, dtype=bool).reshape(len(cells), R)
        out[f"{tag}/p_d"] = np.array([x.p_d for x in res])
        out[f"{tag}/ci"] = np.array([[x.ci_low, x.ci_high] for x in res])
        assert np.array_equal(out[f"{tag}/p_d"], out[f"{tag}/outcomes"].mean(axis=1))
        print(tag, "p_d", out[f"{tag}/p_d"])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
