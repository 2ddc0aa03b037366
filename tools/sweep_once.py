"""One cubic advect sweep at C2 size per gather mode (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_08189_b200 as P
from paper_2209_08189_b200 import _lib, transport
from paper_2209_08189_b200.synth import velocity_array
g = P.make_grid((256,) * 3)
f = torch.rand(g.dims, device="cuda")
v = P.VectorField(g, 0.2 * velocity_array(2, g))
tops = P.TransportOperators(v, P.TransportConfig(4, "cubic"))
out = torch.empty_like(f)
lib = _lib.lib()
for mode in [int(x) for x in os.environ.get("VR_MODES", "1,4").split(",")]:
    lib.vr_set_gather_mode(mode)
    transport.advect(f, tops.forward.displacement, "cubic", out=out)
torch.cuda.synchronize()
