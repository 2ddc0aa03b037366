"""Scattered interpolation throughput (SURVEY.md §8(a) a1, §8(d) operator
micro-inputs): `interpolate_values` / vr_interp_points in Gpts/s.

    python tools/interp_bench.py [--sizes 256 1024] [--out FILE]

Sources: C2's smooth m0 and uniform [0,1) noise.  Points, float64 radians as
the reference passes them (interp.py:112-128): (i) realistic -- the forward
RK2 departure points of 0.25*make_velocity(2), dt = 1/4; (ii) worst case --
uniform in [0, 2pi)^3.  CUDA events on the launching stream, median of 5,
L2 flushed between reps.  Algorithmic bytes per point: 24 (f64 coordinates)
+ 4 (output) + 4 (compulsory source read) = 32 B.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2209_08189_b200 as P  # noqa: E402
from paper_2209_08189_b200 import _lib  # noqa: E402
from paper_2209_08189_b200.synth import c2_problem_device  # noqa: E402

BYTES_PER_POINT = 32


def time_interp(src, pts, order, flush):
    lib = _lib.lib()
    out = torch.empty(src.shape, dtype=torch.float32, device="cuda")
    npts = src.numel()
    ts = []
    for rep in range(6):
        flush.fill_(float(rep))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = lib.vr_interp_points(src.data_ptr(), _lib.dims_arg(src.shape), pts.data_ptr(), 1, npts,
                                  _lib.ORDER[order], out.data_ptr(), _lib.stream())
        b.record()
        _lib.check(rc, "vr_interp_points")
        torch.cuda.synchronize()
        if rep:
            ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[256, 1024])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    flush = torch.empty(64 * 2 ** 20, device="cuda")
    peak = None
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as fh:
            peak = json.load(fh).get("hbm_gbs")
    except Exception:
        pass
    lines = []
    for n in a.sizes:
        g = P.make_grid((n,) * 3)
        m0 = c2_problem_device(g, "linear", 4)[0].values if n <= 256 else None
        if m0 is None:   # 1024^3: the smooth template alone (skip the transport of the generator)
            ax = [torch.arange(k, dtype=torch.float64, device="cuda") * (2 * math.pi / k) for k in g.dims]
            r = torch.sqrt((ax[0].view(-1, 1, 1) - math.pi) ** 2 + (ax[1].view(1, -1, 1) - math.pi) ** 2 +
                           (ax[2].view(1, 1, -1) - math.pi) ** 2)
            m0 = (0.5 * (1.0 - torch.tanh((r - 1.2) / 0.19635))).to(torch.float32)
            del r
        noise = torch.rand(g.dims, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
        v = P.VectorField(g, 0.25 * torch.stack([c for c in _velocity(g)]))
        real = P.TransportOperators(v, P.TransportConfig(4, "linear")).forward.points
        del v
        torch.cuda.empty_cache()
        rnd = torch.rand((3,) + g.dims, dtype=torch.float64, device="cuda",
                         generator=torch.Generator(device="cuda").manual_seed(1)) * (2 * math.pi)
        for kind, pts in (("realistic", real), ("random", rnd)):
            for order in ("linear", "cubic"):
                for sname, src in (("smooth", m0), ("noise", noise)):
                    ms = time_interp(src, pts, order, flush)
                    npts = src.numel()
                    d = {"n": n, "points": kind, "order": order, "source": sname, "ms": ms,
                         "gpts_per_s": npts / ms / 1e6, "alg_gbs": npts * BYTES_PER_POINT / ms / 1e6}
                    if peak:
                        d["hbm_frac"] = d["alg_gbs"] / peak
                    print(json.dumps(d), flush=True)
                    lines.append(d)
        del real, rnd, noise, m0
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as fh:
            fh.write("\n".join(json.dumps(d) for d in lines) + "\n")


def _velocity(g):
    """make_velocity(2) on the device (the same formulas as synth.velocity_array)."""
    x, y, z = (torch.arange(k, dtype=torch.float64, device="cuda") * (2 * math.pi / k) - math.pi for k in g.dims)
    x, y, z = x.view(-1, 1, 1), y.view(1, -1, 1), z.view(1, 1, -1)
    out = []
    for c in range(3):
        acc = torch.zeros(g.dims, dtype=torch.float64, device="cuda")
        for k in (1, 2):
            a = k ** -0.5
            if c == 0:
                acc += a * torch.cos(k * y) * torch.cos(k * x)
            elif c == 1:
                acc += a * torch.sin(k * z) * torch.sin(k * y)
            else:
                acc += a * torch.cos(k * x) * torch.cos(k * z)
        out.append(acc.to(torch.float32))
        del acc
    return out


if __name__ == "__main__":
    main()
