"""Per-operator timing at C2 size (CUDA events), used with ncu for launch lists.

    python tools/prof_ops.py [--n 256] [--reps 5] [--ops spec,advect,trace,fd8,body,dots]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ops", default="spec_A,spec_inv,spec_K,advect_cubic,advect_linear,trace_cubic,fd8_grad,"
                                      "fd8_div,body,incstep,dots,h1")
    ap.add_argument("--slab", action="store_true", help="also time the x1-slab kernels at world size 1")
    args = ap.parse_args()
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import _lib, transport, reductions
    from paper_2209_08189_b200.synth import velocity_array
    n = args.n
    g = P.make_grid((n, n, n))
    N = g.num_voxels
    v = P.VectorField(g, 0.2 * velocity_array(2, g))
    rng = np.random.default_rng(0)
    f = torch.rand((n, n, n), device="cuda")
    w = torch.randn((3, n, n, n), device="cuda")
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    ws = ops.workspace
    tc = P.TransportOperators(v, P.TransportConfig(4, "cubic"))
    tl = P.TransportOperators(v, P.TransportConfig(4, "linear"))
    out3 = torch.empty_like(w)
    out1 = torch.empty_like(f)
    lam = torch.rand((5, n, n, n), device="cuda")
    gm = torch.randn((5, 3, n, n, n), device="cuda")
    l2 = torch.empty(64 * 1024 * 1024, device="cuda")
    from paper_2209_08189_b200.synth import sphere_template
    sph = torch.from_numpy(sphere_template(g)[0]).cuda()
    table = {
        "fd8_grad_sphere": (lambda: P.diffops.fd8_gradient_t(sph, out=out3), N * 16),
        "spec_A": (lambda: ws.apply(_lib.SPEC_A, w, out=out3), 3 * N * 8),
        "spec_inv": (lambda: ws.apply(_lib.SPEC_INVSHIFT, w, out=out3, beta_v=1e-2, shift=1.0), 3 * N * 8),
        "spec_K": (lambda: ws.apply(_lib.SPEC_K, w, out=out3, beta_v=1e-2, beta_w=1e-4), 3 * N * 8),
        "advect_cubic": (lambda: transport.advect(f, tc.forward.displacement, "cubic", out=out1), N * 20),
        "advect_linear": (lambda: transport.advect(f, tl.forward.displacement, "linear", out=out1), N * 20),
        "trace_cubic": (lambda: transport._trace(v.data, g.dims, 0.25, "cubic", tc.div), N * 12 + N * 4 + N * 32),
        "fd8_grad": (lambda: P.diffops.fd8_gradient_t(f, out=out3), N * 16),
        "fd8_div": (lambda: P.diffops.fd8_divergence_t(w, out=out1), N * 16),
        "body": (lambda: _lib.lib().vr_body_force(lam.data_ptr(), gm.data_ptr(), 4, _lib.dims_arg(g.dims), 0.25,
                                                  out3.data_ptr(), _lib.stream()), N * (5 * 16 + 12)),
        "incstep": (lambda: _lib.lib().vr_incstate_step(f.data_ptr(), _lib.dims_arg(g.dims),
                                                        tc.forward.displacement.data_ptr(), w.data_ptr(),
                                                        gm[1].data_ptr(), 0.25, 3, 0, out1.data_ptr(), None,
                                                        _lib.stream()), N * (4 + 12 + 12 + 12 + 4)),
        "dots": (lambda: reductions.dots([(w, w), (w, out3)]), 3 * N * 4 * 3),
        "h1": (lambda: ws.h1_energy(f), N * 4),
    }
    names = args.ops.split(",")
    if args.slab:
        import torch.distributed as tdist
        from paper_2209_08189_b200 import dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        ctx = dist.SlabContext(g.dims)
        with dist.activate(ctx):
            tcs = P.TransportOperators(v, P.TransportConfig(4, "cubic"))
        vlo, vhi = ctx.ghosts(v.data, tcs.w)
        dlo, dhi = ctx.ghosts(tcs.div, tcs.w)
        flo, fhi = ctx.ghosts(f, tcs.w)
        dims_l = _lib.dims_arg(g.dims)
        vext = ctx.halo(v.data, tcs.w)
        dext = ctx.halo(tcs.div, tcs.w)
        table["trace_cubic_slab"] = (lambda: _lib.lib().vr_trace_rk2_slab(
            vext.data_ptr(), dims_l, n, tcs.w, 0.25, 3, out3.data_ptr(), w.data_ptr(), dext.data_ptr(),
            out1.data_ptr(), f.data_ptr(), _lib.stream()), N * 48)
        table["advect_cubic_slab"] = (lambda: _lib.lib().vr_advect_slab(
            f.data_ptr(), flo.data_ptr(), fhi.data_ptr(), dims_l, tcs.w, tcs.forward.displacement.data_ptr(), None,
            3, out1.data_ptr(), None, _lib.stream()), N * 20)
        names += ["trace_cubic_slab", "advect_cubic_slab"]
    res = {}
    for name in names:
        fn, nbytes = table[name]
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
        res[name] = {"ms": round(ms, 4), "alg_GBps": round(nbytes / ms / 1e6, 1)}
        print(f"{name:14s} {ms:8.4f} ms  {nbytes / ms / 1e6:8.1f} GB/s algorithmic", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
