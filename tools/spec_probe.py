"""Spectral operators: accuracy and timing of the hand-written engine against a
cuFFT cross-check (torch.fft, test/tool only -- the north star allows cuFFT
only as a correctness / performance cross-check, never on the product path).

    python tools/spec_probe.py [--n 256] [--reps 20] [--out gpurun_out/spec_probe.json]

For each operator (A, shifted inverse, K) at n^3 on a realistic velocity
(0.2 * make_velocity(2), the C2 generator) and on a smooth-plus-noise field:
  * relative L2 error of the engine vs torch.fft in float64 on the identical
    float32 input (the reference's pocketfft computes in float64);
  * device time per call (CUDA events on the launching stream, 256 MB L2 flush
    between reps) for every engine mode, and for the equivalent torch.fft
    (cuFFT) implementations in float32 and float64.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def kgrid(dims, device):
    n1, n2, n3 = dims
    k1 = torch.fft.fftfreq(n1, d=1.0 / n1, dtype=torch.float64, device=device).view(n1, 1, 1)
    k2 = torch.fft.fftfreq(n2, d=1.0 / n2, dtype=torch.float64, device=device).view(1, n2, 1)
    k3 = torch.arange(n3 // 2 + 1, dtype=torch.float64, device=device).view(1, 1, n3 // 2 + 1)
    return k1, k2, k3


def cufft_op(kind, v, beta_v=1e-2, beta_w=1e-4, shift=1.0, dtype=torch.float64):
    """diffops.py:108-146 on torch.fft (cuFFT): the cross-check."""
    dims = tuple(v.shape[-3:])
    k1, k2, k3 = kgrid(dims, v.device)
    ksq = k1 ** 2 + k2 ** 2 + k3 ** 2
    F = torch.fft.rfftn(v.to(dtype), dim=(-3, -2, -1))
    cd = F.dtype
    if kind == "A":
        F = F * ksq.to(cd)
    elif kind == "invshift":
        F = F * (1.0 / (beta_v * ksq + shift)).to(cd)
    elif kind == "K":
        cb = beta_w * (1 + ksq) / (beta_v * ksq + beta_w * (1 + ksq))
        safe = torch.where(ksq > 0, ksq, torch.ones_like(ksq))
        kd = k1 * F[0] + k2 * F[1] + k3 * F[2]
        f = torch.where(ksq > 0, cb / safe, torch.zeros_like(ksq))
        F = torch.stack([F[0] - k1 * f * kd, F[1] - k2 * f * kd, F[2] - k3 * f * kd])
    return torch.fft.irfftn(F, s=dims, dim=(-3, -2, -1))


def timeit(fn, reps, flush):
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[256])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import _lib
    lib = _lib.lib()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    res = []
    for n in args.n:
        g = P.make_grid((n, n, n))
        ws = P.diffops.workspace_for(g)
        v_real = P.synth.make_velocity(2, g).data * 0.2
        gen = torch.Generator(device="cuda").manual_seed(0)
        v_noise = v_real + 1e-3 * torch.randn(v_real.shape, device="cuda", generator=gen)
        kinds = {"A": (_lib.SPEC_A, {}), "invshift": (_lib.SPEC_INVSHIFT, {"beta_v": 1e-2, "shift": 1.0}),
                 "K": (_lib.SPEC_K, {"beta_v": 1e-2, "beta_w": 1e-4})}
        for name, (kind, kw) in kinds.items():
            for fname, v in (("c2_velocity", v_real), ("velocity_plus_noise", v_noise)):
                ref = cufft_op(name, v)
                modes = [("engine_percomp", (None, 1)), ("engine_allcomp", (None, 0))]
                if name == "A":
                    modes = [("separable_f64_128t", (1, 1)), ("separable_f64_256t", (2, 1)),
                             ("3d_f64_forward_percomp", (0, 1)), ("3d_f64_forward_allcomp", (0, 0))]
                if name == "K":
                    modes = [("engine", (None, 1))]
                for mname, (mode, pc) in modes:
                    lib.vr_set_spectral_tuning(1, pc)
                    if mode is not None:
                        lib.vr_set_spec_a_mode(mode)
                    out = ws.apply(kind, v, **kw)
                    err = float(torch.linalg.vector_norm((out.double() - ref).flatten())
                                / torch.linalg.vector_norm(ref.flatten()))
                    t = timeit(lambda: ws.apply(kind, v, out=out, **kw), args.reps, flush)
                    res.append({"n": n, "op": name, "field": fname, "impl": mname, "rel_l2_vs_cufft_f64": err,
                                "ms": t, "gbs_24B": 24 * n ** 3 / (t * 1e-3) / 1e9})
                    print(json.dumps(res[-1]), flush=True)
                lib.vr_set_spec_a_mode(1)
                lib.vr_set_spectral_tuning(1, 1)
                for dt, dname in ((torch.float32, "cufft_f32"), (torch.float64, "cufft_f64")):
                    if fname != "c2_velocity":
                        continue
                    o = cufft_op(name, v, dtype=dt)
                    err = float(torch.linalg.vector_norm((o.double() - ref).flatten())
                                / torch.linalg.vector_norm(ref.flatten()))
                    t = timeit(lambda: cufft_op(name, v, dtype=dt), max(3, args.reps // 4), flush)
                    res.append({"n": n, "op": name, "field": fname, "impl": dname, "rel_l2_vs_cufft_f64": err,
                                "ms": t, "note": "torch.fft (cuFFT) incl. torch elementwise symbol kernels"})
                    print(json.dumps(res[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            for r in res:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
