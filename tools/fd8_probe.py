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
from paper_2209_08189_b200 import _lib
lib = _lib.lib()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
v3 = torch.randn((3,) + ms.shape[1:], device="cuda")
dv = torch.empty(ms.shape[1:], device="cuda")
for mode in (1, 0):
    lib.vr_set_fd8_mode(mode)
    for what, fn in (("grad", lambda: P.diffops.fd8_gradient_t(rnd, out=out)),
                     ("div", lambda: P.diffops.fd8_divergence_t(v3, out=dv))):
        ts = []
        for _ in range(12):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        t = sorted(ts)[6]
        print(f"mode {mode} {what}: {t:.4f} ms (L2 flushed), {16 * rnd.numel() / (t * 1e-3) / 1e9:.0f} GB/s algorithmic",
              flush=True)
lib.vr_set_fd8_mode(1)
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
