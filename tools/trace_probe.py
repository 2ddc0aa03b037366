"""A/B timing of the single-domain RK2 trace (vr_set_trace_mode 0 = float4
velocity gathers, 2 = general SoA gathers) at C2
size: CUDA events around TransportOperators construction (trace + FD8 div),
L2 flushed between reps; prints ms per construction and the max difference."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2209_08189_b200 as P  # noqa: E402
from paper_2209_08189_b200 import _lib  # noqa: E402
from paper_2209_08189_b200.synth import velocity_array  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
g = P.make_grid((n,) * 3)
v = P.VectorField(g, 0.2 * velocity_array(2, g))
flush = torch.empty(64 * 2 ** 20, device="cuda")
lib = _lib.lib()
res = {}
for order in ("cubic", "linear"):
    for mode in (0, 2, 0, 2):
        lib.vr_set_trace_mode(mode)
        cfg = P.TransportConfig(4, order)
        P.TransportOperators(v, cfg)
        ts = []
        for _ in range(5):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            t = P.TransportOperators(v, cfg)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[(order, mode)] = t.forward.displacement.clone()
        print(order, "mode", mode, "ms", sorted(ts)[len(ts) // 2], flush=True)
    print(order, "maxdiff", float((res[(order, 0)] - res[(order, 2)]).abs().max()))
lib.vr_set_trace_mode(0)
