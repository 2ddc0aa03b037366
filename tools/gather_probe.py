"""A/B timing of the staged vs direct semi-Lagrangian sweeps (vr_set_gather_mode).

    python tools/gather_probe.py [--n 256] [--reps 10]
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
    from paper_2209_08189_b200 import _lib, transport
    from paper_2209_08189_b200.synth import velocity_array
    n = args.n
    dims = (n, n, n)
    g = P.make_grid(dims)
    N = g.num_voxels
    f = torch.rand(dims, device="cuda")
    v = P.VectorField(g, 0.2 * velocity_array(2, g))
    tops = P.TransportOperators(v, P.TransportConfig(4, "cubic"))
    topl = P.TransportOperators(v, P.TransportConfig(4, "linear"))
    vt = torch.randn((3,) + dims, device="cuda")
    gm = torch.randn((3,) + dims, device="cuda")
    out = torch.empty_like(f)
    l2 = torch.empty(64 * 1024 * 1024, device="cuda")
    lib = _lib.lib()
    ops = {
        "advect": (lambda: transport.advect(f, tops.forward.displacement, "cubic", out=out), 20 * N),
        "advect_fac": (lambda: transport.advect(f, tops.backward.displacement, "cubic", factor=tops.adj_factor,
                                                out=out), 24 * N),
        "advect_lin": (lambda: transport.advect(f, topl.forward.displacement, "linear", out=out), 20 * N),
        "advect_lin_fac": (lambda: transport.advect(f, topl.backward.displacement, "linear", factor=topl.adj_factor,
                                                    out=out), 24 * N),
        "incstep_lin": (lambda: lib.vr_incstate_step(f.data_ptr(), _lib.dims_arg(dims),
                                                     topl.forward.displacement.data_ptr(), vt.data_ptr(), gm.data_ptr(),
                                                     0.25, 1, 0, out.data_ptr(), None, _lib.stream()), 44 * N),
        "incstep": (lambda: lib.vr_incstate_step(f.data_ptr(), _lib.dims_arg(dims),
                                                 tops.forward.displacement.data_ptr(), vt.data_ptr(), gm.data_ptr(),
                                                 0.25, 3, 0, out.data_ptr(), None, _lib.stream()), 44 * N),
    }
    for name, (fn, nbytes) in ops.items():
        for quad in [int(x) for x in os.environ.get('VR_MODES', '0,1,5').split(',')]:
            lib.vr_set_gather_mode(quad)
            fn()
            torch.cuda.synchronize()
            tot = 0.0
            for _ in range(args.reps):
                l2.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                b.synchronize()
                tot += a.elapsed_time(b)
            ms = tot / args.reps
            print(f"{name:10s} mode={quad}  {ms:8.4f} ms  {nbytes / ms / 1e6:8.1f} GB/s  {N / ms / 1e6:7.1f} Gpts/s",
                  flush=True)
    lib.vr_set_gather_mode(1)


if __name__ == "__main__":
    main()
