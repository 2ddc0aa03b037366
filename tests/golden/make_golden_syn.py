"""SYN benchmark fixtures from the LIVE reference (velreg/synth.py:22-141):
template labels for three specs (default 10-shape l=8/m=6 at 64^3, a small
non-cubic spec, the fixed-radius hook), make_velocity(K=4) statistics, and the
transported reference image / labels of the default spec.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_syn.py
"""
import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import velreg as V  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

SPECS = {
    "default64": dict(dims=(64, 64, 64), kw={}),
    "small": dict(dims=(32, 48, 40), kw=dict(num_shapes=4, degree=5, order=2, seed=3)),
    "fixed": dict(dims=(32, 32, 32), kw=dict(num_shapes=3, fixed_radius=0.9, seed=7)),
}


def main():
    arrays, meta = {}, {"numpy": np.__version__, "velreg": V.__version__, "specs": {}}
    for name, sp in SPECS.items():
        g = V.make_grid(sp["dims"])
        spec = V.SynthSpec(g, **sp["kw"])
        m0, lab = V.make_template(spec)
        arrays[f"labels_{name}"] = lab.labels.astype(np.int8)
        meta["specs"][name] = {"dims": list(sp["dims"]), "kw": sp["kw"],
                               "counts": np.bincount(lab.labels.ravel(), minlength=spec.num_shapes + 1).tolist()}
    g = V.make_grid((64, 64, 64))
    spec = V.SynthSpec(g)
    m0, lab = V.make_template(spec)
    v = V.make_velocity(4, g)
    meta["velocity_K4"] = {"l2": float(np.linalg.norm(v.data)), "maxabs": float(np.abs(v.data).max())}
    t0 = time.perf_counter()
    cfg = V.TransportConfig(4, "cubic")
    m1, l1 = V.make_reference(m0, lab, v, cfg)
    meta["seconds_reference"] = time.perf_counter() - t0
    arrays["m1_default64"] = m1.values.astype(np.float32)
    arrays["labels1_default64"] = l1.labels.astype(np.int8)
    meta["dice_pre_default64"] = V.dice_averages(lab, l1).d_a
    np.savez_compressed(os.path.join(HERE, "syn.npz"), **arrays)
    with open(os.path.join(HERE, "syn.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps(meta)[:800])


if __name__ == "__main__":
    main()
