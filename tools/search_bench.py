"""Parameter search and continuation at C2 size on ONE GPU.

    python tools/search_bench.py [--n 256] [--out FILE]

C2 sphere -> deformed sphere (cubic, n_t=4), the SearchConfig of the parity
fixture (tests/golden/search_32.json: J bound 0.6, beta_v 1 -> 1e-5,
beta_w 1e-4 -> 1e-6, bisection tolerance 0.5).  Prints one JSON line for the
two-stage search (per-trial log) and one for the continuation replay,
device-synchronised wall time; the warm-start chain never leaves HBM.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2209_08189_b200 as P  # noqa: E402
from paper_2209_08189_b200.synth import c2_problem_device  # noqa: E402

SEARCH = dict(j_min_bound=0.6, beta_v_max=1.0, beta_v_min=1e-5, beta_w_max=1e-4, beta_w_min=1e-6,
              binary_search_rel_tol=0.5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    g = P.make_grid((a.n,) * 3)
    m0, m1, _, _, _ = c2_problem_device(g, "cubic", 4)
    cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=0.0, n_t=4, interp_order="cubic")
    sc = P.SearchConfig(**SEARCH)
    P.gauss_newton_register(m0, m1, cfg)          # warm-up (plans, allocator)
    lines = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.search_parameters(m0, m1, cfg, sc)
    torch.cuda.synchronize()
    t_search = time.perf_counter() - t0
    lines.append({"phase": "search", "n": a.n, "seconds": t_search, "solves": res.total_solves,
                  "gn_iterations": sum(t.gn_iterations for t in res.trials), "beta_v_star": res.beta_v_star,
                  "beta_w_star": res.beta_w_star,
                  "trials": [[t.beta_v, t.beta_w, t.j_min, t.j_max, t.residual, t.gn_iterations, t.seconds,
                              t.accepted] for t in res.trials]})
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, diag = P.continuation_register(m0, m1, res.beta_v_star, res.beta_w_star, cfg, sc)
    torch.cuda.synchronize()
    lines.append({"phase": "continuation", "n": a.n, "seconds": time.perf_counter() - t0,
                  "rungs": [list(r) for r in diag.rungs], "relative_residual": diag.relative_residual,
                  "j_min": diag.j_min, "j_max": diag.j_max})
    for d in lines:
        print(json.dumps(d), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write("\n".join(json.dumps(d) for d in lines) + "\n")


if __name__ == "__main__":
    main()
