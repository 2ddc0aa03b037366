"""Golden fixtures for the SURVEY §8(f) drivers -- parameter search,
continuation (autoparam.py) and the multi-resolution experiment
(experiment.py) -- generated from the LIVE reference under
/root/reference/pkg/src.  Build container only; outputs are committed.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_search.py

Inputs: the C2 sphere -> deformed sphere generator at 32^3 (cubic, n_t=4), the
template/reference/labels stored as the f32/int32 arrays the device consumes.
"""
from __future__ import annotations

import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import velreg as V  # noqa: E402
from velreg.autoparam import continuation_ladder, format_trial_log  # noqa: E402
from velreg.experiment import format_trend_table  # noqa: E402

from make_golden import meta, sphere  # noqa: E402

SEARCH = dict(j_min_bound=0.6, beta_v_max=1.0, beta_v_min=1e-5, beta_w_max=1e-4, beta_w_min=1e-6,
              binary_search_rel_tol=0.5)   # decisions keep >= 0.4 % margin to the J bound
CFG = dict(beta_v=1e-2, beta_w=0.0, n_t=4, interp_order="cubic")


def trial_dict(t):
    return {k: getattr(t, k) for k in ("beta_v", "beta_w", "j_min", "j_max", "residual", "gn_iterations",
                                       "accepted")}


def main():
    g = V.make_grid((32, 32, 32))
    m0, lab0 = sphere(g)
    vt = V.VectorField(g, 0.2 * V.make_velocity(2, g).data)
    cfg_t = V.TransportConfig(4, "cubic")
    tops = V.TransportOperators(vt, cfg_t)
    m1 = V.solve_state(V.ScalarField(g, m0), vt, cfg_t, tops).values.astype(np.float32)
    lab1 = V.transport_labels(V.LabelMap(g, lab0), vt, cfg_t, tops).labels.astype(np.int32)
    M0, M1 = V.ScalarField(g, m0), V.ScalarField(g, m1)
    out = {"dims": [32, 32, 32], "meta": meta(), "search_config": SEARCH, "registration_config": CFG}

    cfg = V.RegistrationConfig(**CFG)
    sc = V.SearchConfig(**SEARCH)
    t0 = time.perf_counter()
    res = V.search_parameters(M0, M1, cfg, sc)
    out["search"] = {"beta_v_star": res.beta_v_star, "beta_w_star": res.beta_w_star,
                     "total_solves": res.total_solves, "trials": [trial_dict(t) for t in res.trials],
                     "log": format_trial_log(res.trials, include_seconds=False),
                     "residual": res.diagnostics.relative_residual,
                     "seconds": time.perf_counter() - t0}
    print(out["search"]["log"])

    t0 = time.perf_counter()
    v, diag = V.continuation_register(M0, M1, res.beta_v_star, res.beta_w_star, cfg, sc)
    out["continuation"] = {"rungs": [list(r) for r in diag.rungs], "relative_residual": diag.relative_residual,
                           "j_min": diag.j_min, "j_max": diag.j_max, "reason": diag.termination_reason,
                           "ladder_v": continuation_ladder(res.beta_v_star, sc.beta_v_max),
                           "ladder_w": continuation_ladder(res.beta_w_star, sc.beta_w_max),
                           "seconds": time.perf_counter() - t0}
    print(out["continuation"])

    t0 = time.perf_counter()
    plan = V.ExperimentPlan(M0, M1, V.LabelMap(g, lab0), V.LabelMap(g, lab1), factors=(1, 2),
                            base_config=V.RegistrationConfig(beta_v=1e-2, beta_w=1e-4, n_t=4,
                                                             interp_order="cubic"),
                            betas=(1e-2, 1e-4))
    pre, rows, vels = V.run_experiment(plan)
    out["experiment"] = {"pre": [pre.d_a, pre.d_vw, pre.d_ivw],
                         "rows": [{k: (list(getattr(r, k)) if k == "dims" else getattr(r, k))
                                   for k in ("factor", "dims", "n_t", "beta_v", "beta_w", "j_min", "j_max",
                                             "residual", "d_a", "d_vw", "d_ivw", "gn_iterations")}
                                  for r in rows],
                         "table": format_trend_table(pre, rows, include_seconds=False),
                         "v_l2": [float(np.linalg.norm(x.data)) for x in vels],
                         "seconds": time.perf_counter() - t0}
    print(out["experiment"]["table"])
    np.savez_compressed(os.path.join(HERE, "search_32.npz"), m0=m0, m1=m1, labels0=lab0, labels1=lab1)
    with open(os.path.join(HERE, "search_32.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
