"""C4 parity fixture: the 256^3 level of the 1024^3
downsampling study, where the CPU reference can run.

m1 at 1024^3 (linear, n_t=16 transport of the C2 sphere) is beyond the CPU
(the reference's two f64 traces alone are ~52 GB), so it is generated on the
GPU and restricted by 4 there; the reference then registers exactly those
256^3 inputs here.  Two steps:

  1. GPU box (two calls, gpurun returns <= 64 MiB each):
                python tests/golden/make_golden_c4.py --dump gpurun_out/c4_p0.npz --part 0
                python tests/golden/make_golden_c4.py --dump gpurun_out/c4_p1.npz --part 1
  2. here:      NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
                    python tests/golden/make_golden_c4.py --ref gpurun_out/c4_p0.npz,gpurun_out/c4_p1.npz

Step 2 writes tests/golden/c4_256.json (trajectory, residual, J range, Dice of
the restricted labels at 256^3, and a checksum of the restricted m1 so the GPU
test can prove it regenerated the same inputs).  The 64 MB m1 itself is not
committed: tests/test_gpu_c4.py regenerates it on the device.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CFG = dict(beta_v=1e-2, beta_w=1e-4, n_t=4, interp_order="linear")   # nt_for_factor(16, 4) = 4


def digest(a) -> str:
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dump(path, part):
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200.synth import c2_problem_device
    g = P.make_grid((1024,) * 3)
    m0, m1, l0, l1, _ = c2_problem_device(g, "linear", 16)
    out = {k: P.restrict(f, 4) for k, f in (("m0", m0), ("m1", m1), ("labels0", l0), ("labels1", l1))}
    m1c = out["m1"].numpy()
    # gpurun copies back <= 64 MiB per call: the 64 MB m1 travels in two x1 halves
    half = slice(part * 128, (part + 1) * 128)
    np.savez_compressed(path, m0=out["m0"].numpy(), m1=m1c[half], labels0=out["labels0"].numpy(),
                        labels1=out["labels1"].numpy())
    print("dumped", path, "part", part, "m1 sha256", digest(m1c))


def reference(path):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, HERE)
    import numpy as np
    import velreg as V
    from make_golden import diag_to_dict, meta, sphere
    parts = [np.load(p) for p in path.split(",")]
    a = dict(parts[0])
    a["m1"] = np.concatenate([p["m1"] for p in parts])
    g = V.make_grid(a["m0"].shape)
    m0_c2, lab0_c2 = sphere(g)
    # the device generator's tanh/sqrt round differently from numpy's in the last f32 bit on a few
    # voxels; the reference registers the device's inputs, the difference is only recorded
    m0_dev_vs_numpy = float(np.abs(m0_c2 - a["m0"]).max())
    labels0_equal = bool(np.array_equal(lab0_c2, a["labels0"]))
    cfg = V.RegistrationConfig(**CFG)
    t0 = time.perf_counter()
    v, diag = V.gauss_newton_register(V.ScalarField(g, a["m0"]), V.ScalarField(g, a["m1"]), cfg)
    secs = time.perf_counter() - t0
    tc = V.TransportConfig(cfg.n_t, cfg.interp_order)
    moved = V.transport_labels(V.LabelMap(g, a["labels0"]), v, tc)
    L1 = V.LabelMap(g, a["labels1"])
    d = diag_to_dict(diag)
    d.update(seconds=secs, dice_pre=V.dice_averages(V.LabelMap(g, a["labels0"]), L1).d_a,
             dice_post=V.dice_averages(moved, L1).d_a, m1_sha256=digest(a["m1"]),
             m0_sha256=digest(a["m0"]), m0_dev_vs_numpy=m0_dev_vs_numpy, labels0_equal_numpy=labels0_equal,
             labels1_sha256=digest(a["labels1"]), config=CFG, meta=meta(),
             inputs="restrict(., 4) of the 1024^3 C2 pair generated on the GPU (linear, n_t=16)")
    print(json.dumps(d))
    with open(os.path.join(HERE, "c4_256.json"), "w") as fh:
        json.dump(d, fh, indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--dump")
    ap.add_argument("--part", type=int, default=0)
    ap.add_argument("--ref", help="comma-separated dumps of parts 0 and 1")
    a = ap.parse_args()
    if a.dump:
        dump(a.dump, a.part)
    if a.ref:
        reference(a.ref)
