"""Separable A with long x1 lines: one tile per CTA vs the persistent
cp.async-pipelined long kernel (vr_set_spectral_tuning key 5).  Device time
per A (CUDA events, 256 MB L2 flush between reps) and bit-identity.

    python tools/long_pipe_probe.py [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import _lib
    lib = _lib.lib()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for dims in ((512, 256, 256), (1024, 128, 256), (2048, 128, 128)):
        g = P.make_grid(dims)
        ws = P.diffops.workspace_for(g)
        v = torch.randn((3,) + dims, device="cuda")
        res, outs = {"dims": dims}, {}
        for mode in (0, 1, 0, 1):
            lib.vr_set_spectral_tuning(5, mode)
            out = torch.empty_like(v)
            ws.apply(_lib.SPEC_A, v, out=out, alpha=1e-2)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                flush.fill_(1.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ws.apply(_lib.SPEC_A, v, out=out, alpha=1e-2)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            res[f"pipe{mode}_ms"] = ts[len(ts) // 2]
            outs[mode] = out
        res["bit_identical"] = bool(torch.equal(outs[0], outs[1]))
        lib.vr_set_spectral_tuning(5, 1)
        print(json.dumps(res), flush=True)
        del ws, v, outs
        P.diffops._ws_cache.clear()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
