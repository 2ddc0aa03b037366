"""C4 downsampling study on ONE GPU.

    python tools/c4_pipeline.py [--n 1024] [--factors 4 2] [--nt 16] [--order linear] [--out FILE]

Inputs: C2's sphere generator at n^3 evaluated on the device
(synth.c2_problem_device; m1/labels1 = transport along 0.2*make_velocity(2)
with n_t steps).  Then `run_experiment` (experiment.py:100-146) with fixed
betas (beta_v=1e-2, beta_w=1e-4): restrict by each factor, register at the
coarse level, prolong spectrally back to n^3, transport template + labels at
n^3 and score residual / Dice there -- every field stays in HBM.  One JSON
line per level (device-synchronised wall time per phase, peak HBM).
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--factors", type=int, nargs="+", default=[4, 2])
    ap.add_argument("--nt", type=int, default=16)
    ap.add_argument("--order", default="linear")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    g = P.make_grid((a.n,) * 3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m0, m1, l0, l1, vtrue = c2_problem_device(g, a.order, a.nt)
    del vtrue
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    torch.cuda.empty_cache()
    lines = []

    def emit(d):
        s = json.dumps(d)
        print(s, flush=True)
        lines.append(s)

    emit({"phase": "generate", "n": a.n, "n_t": a.nt, "order": a.order, "seconds": t_gen,
          "peak_hbm_gb": torch.cuda.max_memory_allocated() / 2 ** 30})
    base_cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=1e-4, n_t=a.nt, interp_order=a.order)
    for f in a.factors:
        torch.cuda.reset_peak_memory_stats()
        plan = P.ExperimentPlan(m0, m1, l0, l1, factors=(f,), base_config=base_cfg, betas=(1e-2, 1e-4))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pre, rows, vels = P.run_experiment(plan)
        torch.cuda.synchronize()
        r = rows[0]
        emit({"phase": "level", "factor": f, "coarse_dims": list(r.dims), "n_t": r.n_t, "seconds": time.perf_counter() - t0,
              "gn_iterations": r.gn_iterations, "j_min": r.j_min, "j_max": r.j_max, "residual": r.residual,
              "dice_pre": pre.d_a, "dice": r.d_a, "peak_hbm_gb": torch.cuda.max_memory_allocated() / 2 ** 30})
        del vels
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as fh:
            fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
