"""One call of each spectral operator at n^3 (for ncu launch lists / captures).

    python tools/spec_once.py [--n 256] [--ops A,A3d,invshift,K]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--ops", default="A,A3d,invshift,K")
    args = ap.parse_args()
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import _lib
    lib = _lib.lib()
    g = P.make_grid((args.n,) * 3)
    ws = P.diffops.workspace_for(g)
    v = P.synth.make_velocity(2, g).data * 0.2
    out = torch.empty_like(v)
    for op in args.ops.split(","):
        if op == "A":
            lib.vr_set_spec_a_mode(1)
            ws.apply(_lib.SPEC_A, v, out=out)
        elif op == "A3d":
            lib.vr_set_spec_a_mode(0)
            ws.apply(_lib.SPEC_A, v, out=out)
            lib.vr_set_spec_a_mode(1)
        elif op == "invshift":
            ws.apply(_lib.SPEC_INVSHIFT, v, out=out, beta_v=1e-2, shift=1.0)
        elif op == "K":
            ws.apply(_lib.SPEC_K, v, out=out, beta_v=1e-2, beta_w=1e-4)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
