"""x1 pass of the 3-D engine: 16 kz of one x2 row per CTA vs lines over the
flat (x2, kz) plane (vr_set_spectral_tuning key 4).  Device time per
shifted inverse and per 3-D A (CUDA events, 256 MB L2 flush between reps)
and bit-identity of the two layouts.

    python tools/xflat_probe.py [--n 256] [--reps 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import _lib
    lib = _lib.lib()
    g = P.make_grid((a.n,) * 3)
    ws = P.diffops.workspace_for(g)
    v = P.synth.make_velocity(2, g).data * 0.2
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    res = {"n": a.n}
    for name, kind, kw, amode in (("invshift", _lib.SPEC_INVSHIFT, dict(beta_v=1e-2, shift=1.0), 1),
                                  ("A3d", _lib.SPEC_A, {}, 0)):
        outs = {}
        prev_a = lib.vr_set_spec_a_mode(amode)
        for mode in (0, 1, 0, 1):
            lib.vr_set_spectral_tuning(4, mode)
            out = torch.empty_like(v)
            ws.apply(kind, v, out=out, **kw)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ws.apply(kind, v, out=out, **kw)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            res[f"{name}_flat{mode}_ms"] = ts[len(ts) // 2]
            outs[mode] = out
        lib.vr_set_spec_a_mode(prev_a)
        res[f"{name}_bit_identical"] = bool(torch.equal(outs[0], outs[1]))
    lib.vr_set_spectral_tuning(4, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
