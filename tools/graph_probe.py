"""Host-overhead probe: one GN Hessian matvec at C2 size, eager vs CUDA-graph replay.

    python tools/graph_probe.py [--n 256]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import _lib, optim
    from paper_2209_08189_b200.synth import c2_problem
    g = P.make_grid((args.n,) * 3)
    m0, m1, _, _, vtrue = c2_problem(g)
    cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=0.0, n_t=4, interp_order="cubic")
    ops = P.RegOperators.for_grid(g, cfg.beta_v, cfg.beta_w)
    v = P.VectorField(g, 0.5 * vtrue.data)
    st = optim.ObjectiveState(m0, m1, v, cfg, ops)
    _ = st.objective
    _ = st.gradient
    p = torch.randn_like(v.data)
    out = torch.empty_like(p)

    def mv():
        optim.hessian_matvec_t(p, st, cfg, out=out)
        _lib._deferred.clear()   # probe only: no reduction follows to read the flags

    def pc():
        ops.workspace.apply(_lib.SPEC_INVSHIFT, p, out=out, beta_v=1e-2, shift=1.0)

    def timeit(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / args.reps

    for name, fn in (("matvec", mv), ("precond", pc)):
        eager = timeit(fn)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        ref = out.clone()
        graph = timeit(gr.replay)
        fn()
        same = torch.equal(ref, out)
        print(f"{name:8s} eager {eager:7.3f} ms   graph {graph:7.3f} ms   identical={same}", flush=True)


if __name__ == "__main__":
    main()
