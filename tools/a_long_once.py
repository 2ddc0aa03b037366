"""One separable A at (512, 256, 256): the x1 pass runs the three-step long_kernel
(for ncu captures of the kernel the distributed A uses on 2-rank blocks)."""
import sys, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_08189_b200 as P
from paper_2209_08189_b200 import _lib
g = P.make_grid((512, 256, 256))
ws = P.diffops.workspace_for(g)
v = torch.randn((3, 512, 256, 256), device="cuda")
out = torch.empty_like(v)
for _ in range(2):
    ws.apply(_lib.SPEC_A, v, out=out, alpha=1e-2)
torch.cuda.synchronize()
print("ok")
