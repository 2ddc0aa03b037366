"""Generate golden parity fixtures from the LIVE reference (`velreg` under
/root/reference/pkg/src).  Run in the build container only (the reference does
not exist on the GPU box); the outputs are committed under tests/golden/.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [ops] [gn] [c1] [c2]

The environment variables matter: numba's cache=True otherwise writes into the
read-only reference tree.

Fixture policy: every input a GPU kernel consumes is stored as float32 (what the
device computes on); the reference is evaluated on the float64 up-cast of those
float32 inputs, so the stored outputs are the reference's answer for exactly the
device's inputs.  Where the reference's own dtype behaviour matters (image data
f32, velocity f64) the fixture says so.
"""
from __future__ import annotations

import json
import math
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import numpy as np  # noqa: E402
import numba  # noqa: E402
import velreg as V  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def meta():
    return {"numpy": np.__version__, "numba": numba.__version__,
            "velreg": V.__version__, "generator": "tests/golden/make_golden.py"}


def blob(grid, c, s):
    x = grid.coords()
    d2 = sum((x[i] - c[i]) ** 2 for i in range(3))
    return np.exp(-d2 / (2 * s * s))


def c1_raw(grid):
    pi = math.pi
    return (blob(grid, (pi, pi, pi), 0.5)
            + 0.6 * blob(grid, (pi - 1.0, pi + 0.6, pi), 0.35)).astype(np.float32)


def sphere(grid, radius=1.2, width=0.19635):
    x = grid.coords()
    r = np.sqrt(sum((x[i] - math.pi) ** 2 for i in range(3)))
    m0 = (0.5 * (1.0 - np.tanh((r - radius) / width))).astype(np.float32)
    return m0, (r <= radius).astype(np.int32)


def c1_pair(grid, order):
    m0 = c1_raw(grid)
    v = V.VectorField(grid, 0.25 * V.make_velocity(2, grid).data)
    m1 = V.solve_state(V.ScalarField(grid, m0), v, V.TransportConfig(4, order)).values
    lo = min(m0.min(), m1.min())
    hi = max(m0.max(), m1.max())
    return (((m0 - lo) / (hi - lo)).astype(np.float32),
            ((m1 - lo) / (hi - lo)).astype(np.float32), m1)


def ops_fixture(dims, name):
    """Per-operator inputs/outputs on one grid (both interpolation orders)."""
    g = V.make_grid(dims)
    rng0 = np.random.default_rng(0)
    rng1 = np.random.default_rng(1)
    out = {"dims": np.array(dims)}
    f_smooth = c1_raw(g)
    f_rand = rng0.random(dims).astype(np.float32)
    v32 = (0.25 * V.make_velocity(2, g).data).astype(np.float32)
    vt32 = (0.5 * V.make_velocity(1, g).data[[2, 0, 1]]).astype(np.float32)
    w32 = rng0.standard_normal((3,) + tuple(dims)).astype(np.float32)
    out.update(f_smooth=f_smooth, f_rand=f_rand, v=v32, vt=vt32, w=w32)
    v = V.VectorField(g, v32.astype(np.float64))
    vt = V.VectorField(g, vt32.astype(np.float64))
    w = V.VectorField(g, w32.astype(np.float64))
    # scattered points: realistic (RK2 trace) and worst case (uniform, incl. out of box)
    pts_rand = rng1.uniform(-2 * math.pi, 4 * math.pi, size=(3,) + tuple(dims))
    out["pts_rand"] = pts_rand.astype(np.float32)
    pr64 = out["pts_rand"].astype(np.float64)
    for order in ("linear", "cubic"):
        tr = V.trace_characteristics(v, 0.25, order)
        out[f"trace_fwd_{order}"] = tr.points
        trb = V.trace_characteristics(V.VectorField(g, -v.data), 0.25, order)
        out[f"trace_bwd_{order}"] = trb.points
        for src in ("smooth", "rand"):
            vals = out[f"f_{src}"].astype(np.float64)
            out[f"interp_{order}_{src}_trace"] = V.interp.interpolate_values(
                vals, tr.points, order, g.spacing)
            out[f"interp_{order}_{src}_rand"] = V.interp.interpolate_values(
                vals, pr64, order, g.spacing)
        cfg = V.TransportConfig(4, order)
        tops = V.TransportOperators(v, cfg)
        out[f"jac_numer_{order}"] = tops.jac_numer
        out[f"jac_denom_{order}"] = tops.jac_denom
        out[f"adj_numer_{order}"] = tops.adj_numer
        out[f"adj_denom_{order}"] = tops.adj_denom
        m0 = V.ScalarField(g, f_smooth.astype(np.float64))
        series = V.solve_state_series(m0, v, cfg, tops)
        out[f"state_series_{order}"] = series
        lam = V.solve_adjoint(V.ScalarField(g, f_rand.astype(np.float64) - 0.5), v, cfg, tops)
        out[f"adjoint_series_{order}"] = lam
        out[f"incstate_{order}"] = V.solve_incremental_state(series, v, vt, cfg, tops).values
        out[f"jacobian_{order}"] = V.jacobian_determinant(v, cfg, tops).values
    # FD8 (f32 in -> f32 arithmetic in the reference; also f64 target)
    out["fd8_grad_f32"] = V.fd8_gradient(V.ScalarField(g, f_rand)).data
    out["fd8_grad"] = V.fd8_gradient(V.ScalarField(g, f_rand.astype(np.float64))).data
    out["fd8_div_f32"] = V.fd8_divergence(V.VectorField(g, w32)).values
    out["fd8_div"] = V.fd8_divergence(w).values
    # spectral operators (velocity space: f64 in the reference)
    ops = V.RegOperators.for_grid(g, 1e-2, 1e-4)
    out["apply_A_v"] = V.apply_A(v, ops).data
    out["apply_A_w"] = V.apply_A(w, ops).data
    out["inv_shifted_A_w_1"] = V.apply_inv_shifted_A(w, ops, 1.0).data
    out["inv_shifted_A_w_037"] = V.apply_inv_shifted_A(w, ops, 0.37).data
    out["apply_K_w"] = V.apply_K(w, ops).data
    out["apply_K_v"] = V.apply_K(v, ops).data
    ops2 = V.RegOperators.for_grid(g, 1e-2, 3.0)
    out["apply_K_w_bw3"] = V.apply_K(w, ops2).data
    div = V.fd8_divergence(v)
    out["h1_energy_divv"] = np.float64(V.diffops.h1_energy(div, ops.workspace))
    out["h1_energy_frand"] = np.float64(V.diffops.h1_energy(
        V.ScalarField(g, f_rand.astype(np.float64)), ops.workspace))
    # objective / gradient / Gauss-Newton matvec at a non-zero iterate
    for order in ("cubic", "linear"):
        m0n, m1n, _ = c1_pair(g, order)
        out[f"obj_m0_{order}"] = m0n
        out[f"obj_m1_{order}"] = m1n
        for bw in (0.0, 1e-4):
            cfg = V.RegistrationConfig(beta_v=1e-2, beta_w=bw, n_t=4, interp_order=order)
            ops_r = V.RegOperators.for_grid(g, 1e-2, bw)
            st = V.ObjectiveState(V.ScalarField(g, m0n), V.ScalarField(g, m1n),
                                  V.VectorField(g, 0.5 * v.data), cfg, ops_r)
            tag = f"{order}_bw{bw:g}"
            out[f"objective_{tag}"] = np.float64(st.objective)
            out[f"gradient_{tag}"] = st.gradient.data
            out[f"matvec_{tag}"] = V.hessian_matvec(w, st).data
            out[f"deformed_{tag}"] = st.deformed.values
    # labels + Dice
    m0s, lab0 = sphere(g, 1.2, 0.19635 * 64 / dims[0])
    lab0 = lab0.copy()
    x = g.coords()
    lab0[(lab0 == 1) & (x[0] > math.pi)] = 3   # three labels, one split
    lab0[(lab0 == 0) & (np.abs(x[1] - 1.0) < 0.4) & (np.abs(x[0] - 1.0) < 0.5)] = 7
    L0 = V.LabelMap(g, lab0)
    out["labels0"] = lab0
    for order in ("cubic", "linear"):
        L1 = V.transport_labels(L0, v, V.TransportConfig(4, order))
        out[f"labels_moved_{order}"] = L1.labels
        rep = V.dice_averages(L1, L0)
        out[f"dice_{order}"] = np.array(rep.dice)
        out[f"dice_avgs_{order}"] = np.array([rep.d_a, rep.d_vw, rep.d_ivw])
        out[f"dice_ids_{order}"] = np.array(rep.label_ids)
    # resampling
    out["restrict2_f"] = V.restrict(V.ScalarField(g, f_rand), 2).values
    coarse = V.make_grid(tuple(n // 2 for n in dims))
    cv = V.VectorField(coarse, w32[:, ::2, ::2, ::2].astype(np.float64))
    out["prolong_in"] = w32[:, ::2, ::2, ::2]
    out["prolong_out"] = V.prolong_spectral(cv, g).data
    # compact storage: array targets as f32 (relative 6e-8, far below every
    # parity tolerance); scalars keep f64
    for k, a in list(out.items()):
        a = np.asarray(a)
        if a.dtype == np.float64 and a.ndim > 0:
            out[k] = a.astype(np.float32)
    path = os.path.join(HERE, f"ops_{name}.npz")
    np.savez_compressed(path, **out)
    with open(os.path.join(HERE, f"ops_{name}.meta.json"), "w") as fh:
        json.dump(meta(), fh, indent=1)
    print("wrote", path, os.path.getsize(path))


def diag_to_dict(diag):
    return {
        "objective": [r.objective for r in diag.iterations],
        "rel_grad": [r.rel_grad_norm for r in diag.iterations],
        "pcg": [r.pcg_iterations for r in diag.iterations],
        "step": [r.step_length for r in diag.iterations],
        "cfl": [r.cfl for r in diag.iterations],
        "relative_residual": diag.relative_residual,
        "j_min": diag.j_min, "j_max": diag.j_max,
        "converged": diag.converged, "reason": diag.termination_reason,
        "gn_iterations": diag.gn_iterations,
    }


def gn_fixture(dims, name, configs):
    """Full Gauss-Newton registrations on a C1-style blob pair (small grid)."""
    g = V.make_grid(dims)
    res = {"dims": list(dims), "meta": meta(), "runs": {}}
    arrays = {}
    for order in ("cubic", "linear"):
        m0n, m1n, _ = c1_pair(g, order)
        arrays[f"m0_{order}"] = m0n
        arrays[f"m1_{order}"] = m1n
    for order, bw in configs:
        m0n, m1n = arrays[f"m0_{order}"], arrays[f"m1_{order}"]
        cfg = V.RegistrationConfig(beta_v=1e-2, beta_w=bw, n_t=4, interp_order=order)
        t0 = time.perf_counter()
        vhat, diag = V.gauss_newton_register(V.ScalarField(g, m0n), V.ScalarField(g, m1n), cfg)
        dt = time.perf_counter() - t0
        tag = f"{order}_bw{bw:g}"
        d = diag_to_dict(diag)
        d["seconds"] = dt
        d["v_l2"] = float(np.linalg.norm(vhat.data))
        d["v_maxabs"] = float(np.abs(vhat.data).max())
        res["runs"][tag] = d
        arrays[f"v_{tag}"] = vhat.data.astype(np.float32)
        print(name, tag, d["objective"], d["pcg"], d["relative_residual"], f"{dt:.2f}s")
    np.savez_compressed(os.path.join(HERE, f"gn_{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"gn_{name}.json"), "w") as fh:
        json.dump(res, fh, indent=1)


def c1_fixture():
    """C1: blob 64^3 -- the CPU-runnable headline config."""
    g = V.make_grid((64, 64, 64))
    res = {"dims": [64, 64, 64], "meta": meta(), "runs": {}}
    arrays = {}
    for order in ("cubic", "linear"):
        m0n, m1n, m1raw = c1_pair(g, order)
        arrays[f"m1raw_{order}"] = m1raw
        for bw in (0.0, 1e-4):
            cfg = V.RegistrationConfig(beta_v=1e-2, beta_w=bw, n_t=4, interp_order=order)
            t0 = time.perf_counter()
            vhat, diag = V.gauss_newton_register(V.ScalarField(g, m0n), V.ScalarField(g, m1n), cfg)
            dt = time.perf_counter() - t0
            tag = f"{order}_bw{bw:g}"
            d = diag_to_dict(diag)
            d["seconds"] = dt
            d["v_l2"] = float(np.linalg.norm(vhat.data))
            res["runs"][tag] = d
            print("c1", tag, d["objective"], d["pcg"], d["relative_residual"], f"{dt:.2f}s")
    np.savez_compressed(os.path.join(HERE, "c1_64.npz"), **arrays)
    with open(os.path.join(HERE, "c1_64.json"), "w") as fh:
        json.dump(res, fh, indent=1)


def c2_fixture(n=256):
    """C2: sphere -> deformed sphere; n=256 takes ~10 min here."""
    g = V.make_grid((n, n, n))
    m0, lab0 = sphere(g)
    vtrue = V.VectorField(g, 0.2 * V.make_velocity(2, g).data)
    cfg_t = V.TransportConfig(4, "cubic")
    t0 = time.perf_counter()
    tops = V.TransportOperators(vtrue, cfg_t)
    m1 = V.solve_state(V.ScalarField(g, m0), vtrue, cfg_t, tops).values
    L0 = V.LabelMap(g, lab0)
    L1 = V.transport_labels(L0, vtrue, cfg_t, tops)
    t_gen = time.perf_counter() - t0
    pre = V.dice_averages(L0, L1)
    cfg = V.RegistrationConfig(beta_v=1e-2, beta_w=0.0, n_t=4, interp_order="cubic")
    t0 = time.perf_counter()
    vhat, diag = V.gauss_newton_register(V.ScalarField(g, m0), V.ScalarField(g, m1), cfg)
    t_reg = time.perf_counter() - t0
    t0 = time.perf_counter()
    moved = V.transport_labels(L0, vhat, cfg_t)
    post = V.dice_averages(moved, L1)
    t_post = time.perf_counter() - t0
    d = diag_to_dict(diag)
    res = {"dims": [n] * 3, "meta": meta(), "seconds_register": t_reg,
           "seconds_generate": t_gen, "seconds_post": t_post,
           "m1_sum": float(m1.astype(np.float64).sum()),
           "m1_l2": float(np.linalg.norm(m1.astype(np.float64))),
           "label1_volume": int((L1.labels == 1).sum()),
           "label0_volume": int((lab0 == 1).sum()),
           "dice_pre": pre.d_a, "dice_post": post.d_a,
           "moved_volume": int((moved.labels == 1).sum()),
           "v_l2": float(np.linalg.norm(vhat.data)), "run": d,
           "cores": os.cpu_count(), "numba_threads": numba.get_num_threads()}
    with open(os.path.join(HERE, f"c2_{n}.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print("c2", n, d["objective"], d["pcg"], d["relative_residual"], pre.d_a, post.d_a,
          f"{t_reg:.1f}s")


if __name__ == "__main__":
    what = sys.argv[1:] or ["ops", "gn"]
    if "ops" in what:
        ops_fixture((16, 20, 24), "16x20x24")
    if "gn" in what:
        gn_fixture((32, 32, 32), "32", [("cubic", 0.0), ("cubic", 1e-4),
                                       ("linear", 0.0), ("linear", 1e-4)])
        gn_fixture((16, 20, 24), "16x20x24", [("cubic", 0.0), ("linear", 1e-4)])
    if "c1" in what:
        c1_fixture()
    if "c2" in what:
        c2_fixture(256)
    if "c2_64" in what:
        c2_fixture(64)
