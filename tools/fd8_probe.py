"""FD8 gradient timing on the C2 state series (far-field values reach the
float32 subnormal range, which exercises the kernel's IEEE-division fallback).

    python tools/fd8_probe.py
"""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import paper_2209_08189_b200 as P
from paper_2209_08189_b200 import optim
from paper_2209_08189_b200.synth import c2_problem
g = P.make_grid((256,) * 3)
m0, m1, _, _, vtrue = c2_problem(g)
cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=0.0, n_t=4, interp_order="cubic")
ops = P.RegOperators.for_grid(g, cfg.beta_v, cfg.beta_w)
st = optim.ObjectiveState(m0, m1, P.VectorField(g, 0.5 * vtrue.data), cfg, ops)
ms = st.m_series
out = torch.empty((3,) + ms.shape[1:], device="cuda")
rnd = torch.rand(ms.shape[1:], device="cuda")
for name, f in [("rand", rnd)] + [(f"m{j}", ms[j]) for j in range(5)] + [("m4copy", ms[4].clone())]:
    for _ in range(2):
        P.diffops.fd8_gradient_t(f, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        P.diffops.fd8_gradient_t(f, out=out)
    b.record(); b.synchronize()
    a_ = f.abs()
    tiny = ((a_ > 0) & (a_ < 2.0 ** -60)).float().mean().item()
    print(name, f"{a.elapsed_time(b) / 10:.4f} ms", "tiny-input frac", tiny, flush=True)
