"""A/B of the four-step vs Stockham spectral kernels (vr_set_fft_mode): relative
difference of every operator and per-call time.

    python tools/fft_probe.py [--n 256] [--reps 10]
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
    from paper_2209_08189_b200 import _lib
    from paper_2209_08189_b200.synth import velocity_array
    n = args.n
    g = P.make_grid((n, n, n))
    v = P.VectorField(g, 0.2 * velocity_array(2, g)).data
    w = torch.randn((3, n, n, n), device="cuda")
    f = torch.rand((n, n, n), device="cuda")
    ws = P.RegOperators.for_grid(g, 1e-2, 1e-4).workspace
    lib = _lib.lib()
    l2 = torch.empty(64 * 1024 * 1024, device="cuda")
    ops = {
        "A": lambda x: ws.apply(_lib.SPEC_A, x),
        "inv": lambda x: ws.apply(_lib.SPEC_INVSHIFT, x, beta_v=1e-2, shift=1.0),
        "K": lambda x: ws.apply(_lib.SPEC_K, x, beta_v=1e-2, beta_w=1e-4),
    }
    for name, fn in ops.items():
        res = {}
        for mode in (0, 1):
            lib.vr_set_fft_mode(mode)
            outs = [fn(v).clone(), fn(w).clone()]
            torch.cuda.synchronize()
            tot = 0.0
            for _ in range(args.reps):
                l2.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                fn(w)
                b.record()
                b.synchronize()
                tot += a.elapsed_time(b)
            res[mode] = (outs, tot / args.reps)
        rel = [float((x.double() - y.double()).norm() / y.double().norm()) for x, y in zip(res[1][0], res[0][0])]
        print(f"{name:4s} stockham {res[0][1]:.4f} ms  four-step {res[1][1]:.4f} ms  rel diff smooth {rel[0]:.2e} "
              f"random {rel[1]:.2e}", flush=True)
    lib.vr_set_fft_mode(1)
    h0 = ws.h1_energy(f)
    lib.vr_set_fft_mode(0)
    h1 = ws.h1_energy(f)
    lib.vr_set_fft_mode(1)
    print(f"h1 rel diff {abs(h0 / h1 - 1):.2e}")


if __name__ == "__main__":
    main()
