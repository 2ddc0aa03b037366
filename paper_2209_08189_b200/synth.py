"""Synthetic inputs and label transport.

`make_velocity` and `transport_labels` mirror
/root/reference/pkg/src/velreg/synth.py:104-131 (label transport runs on the
device: the first SL step gathers the indicator straight from the int32 label
map and the last step thresholds at 0.5, so no float indicator volume is ever
materialised).  The C1/C2 generators define the benchmark inputs of
SURVEY.md §8(d) (the blob pair and the sphere -> deformed sphere pair).
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .grid import Grid, LabelMap, ScalarField, VectorField
from .transport import TransportConfig, TransportOperators, solve_state


def make_velocity(K: int, grid: Grid) -> VectorField:
    """Per-axis trigonometric sums with amplitudes k^-0.5, k = 1..K, on the
    centred lattice (synth.py:104-118); evaluated in f64 on the host."""
    return VectorField(grid, velocity_array(K, grid))


def _coords(grid: Grid) -> np.ndarray:
    """Lattice coordinates of this rank's part of `grid` (all of it unless an
    x1-slab decomposition is active)."""
    from . import dist
    ctx = dist.for_grid(grid.dims)
    if ctx is not None:
        return ctx.local_coords()
    return grid.coords()


def velocity_array(K: int, grid: Grid) -> np.ndarray:
    if K < 1:
        raise ValueError("K must be >= 1")
    x, y, z = _coords(grid) - math.pi
    vx = np.zeros(x.shape)
    vy = np.zeros(x.shape)
    vz = np.zeros(x.shape)
    for k in range(1, K + 1):
        a = k ** -0.5
        vx += a * np.cos(k * y) * np.cos(k * x)
        vy += a * np.sin(k * z) * np.sin(k * y)
        vz += a * np.cos(k * x) * np.cos(k * z)
    return np.stack([vx, vy, vz])


def transport_labels(labels: LabelMap, v: VectorField, cfg: TransportConfig,
                     ops: TransportOperators = None) -> LabelMap:
    """Advect each label's indicator with the state solver and re-threshold at
    0.5; overlap ties go to the larger label id (synth.py:121-131)."""
    ops = ops or TransportOperators(v, cfg)
    lib = _lib.lib()
    dims = tuple(labels.labels.shape)
    d = _lib.dims_arg(dims)
    st = _lib.stream()
    order = _lib.ORDER[cfg.interp_order]
    disp = ops.forward.displacement.data_ptr()
    out = torch.zeros(dims, dtype=torch.int32, device=labels.labels.device)
    bufs = [torch.empty(dims, dtype=torch.float32, device=out.device) for _ in range(2)]
    if ops.ctx is not None:   # x1 slabs: float indicator + halo'd sweeps
        for lab in labels.label_ids():
            cur = (labels.labels == lab).to(torch.float32)
            for j in range(cfg.n_t):
                if j < cfg.n_t - 1:
                    cur = ops.sweep(cur, ops.forward.displacement, out=bufs[j % 2])
                else:
                    lo, hi = ops.ctx.ghosts(cur, ops.w)
                    _lib.check(lib.vr_label_step_slab(cur.data_ptr(), lo.data_ptr(), hi.data_ptr(), int(lab), d,
                                                      ops.w, disp, order, None, out.data_ptr(), st),
                               "vr_label_step_slab")
        return LabelMap(labels.grid, out, labels.max_id)
    for lab in labels.label_ids():
        src = None
        for j in range(cfg.n_t):
            first, last = j == 0, j == cfg.n_t - 1
            dst = bufs[j % 2]
            rc = lib.vr_label_step(None if first else src.data_ptr(), labels.labels.data_ptr() if first else None,
                                   int(lab), d, disp, order, None if last else dst.data_ptr(),
                                   out.data_ptr() if last else None, st)
            _lib.check(rc, "vr_label_step")
            src = dst
    return LabelMap(labels.grid, out, labels.max_id)


def make_reference(m0: ScalarField, labels: LabelMap, v: VectorField, cfg: TransportConfig):
    """Reference image and labels by transporting the template along v (synth.py:134-141)."""
    ops = TransportOperators(v, cfg)
    return solve_state(m0, v, cfg, ops), transport_labels(labels, v, cfg, ops)


# ---- benchmark problems ---------------------------------------
def _gauss(grid: Grid, c, s) -> np.ndarray:
    x = _coords(grid)
    d2 = sum((x[i] - c[i]) ** 2 for i in range(3))
    return np.exp(-d2 / (2 * s * s))


def c1_template(grid: Grid) -> np.ndarray:
    """C1 raw template: two Gaussian blobs, float32."""
    pi = math.pi
    return (_gauss(grid, (pi, pi, pi), 0.5) + 0.6 * _gauss(grid, (pi - 1.0, pi + 0.6, pi), 0.35)).astype(np.float32)


def c1_problem(grid: Grid, order: str = "cubic"):
    """C1 pair: m1 = transport of m0 along 0.25*make_velocity(2) (n_t = 4, `order`),
    then joint [0,1] normalisation.  Returns device ScalarFields (m0, m1)."""
    m0 = ScalarField(grid, c1_template(grid))
    v = VectorField(grid, 0.25 * velocity_array(2, grid))
    m1 = solve_state(m0, v, TransportConfig(4, order))
    lo = min(float(m0.values.min()), float(m1.values.min()))
    hi = max(float(m0.values.max()), float(m1.values.max()))
    return (ScalarField(grid, (m0.values - lo) / (hi - lo)), ScalarField(grid, (m1.values - lo) / (hi - lo)))


def sphere_template(grid: Grid, radius: float = 1.2, width: float = 0.19635):
    """C2 template: smoothed ball (float32) and its label map (int32)."""
    x = _coords(grid)
    r = np.sqrt(sum((x[i] - math.pi) ** 2 for i in range(3)))
    m0 = (0.5 * (1.0 - np.tanh((r - radius) / width))).astype(np.float32)
    return m0, (r <= radius).astype(np.int32)


def c2_problem(grid: Grid, order: str = "cubic", n_t: int = 4):
    """C2: sphere -> deformed sphere along v_true = 0.2*make_velocity(2); returns
    device (m0, m1, labels0, labels1, v_true)."""
    m0_np, lab_np = sphere_template(grid)
    m0 = ScalarField(grid, m0_np)
    lab0 = LabelMap(grid, lab_np)
    vtrue = VectorField(grid, 0.2 * velocity_array(2, grid))
    cfg = TransportConfig(n_t, order)
    tops = TransportOperators(vtrue, cfg)
    m1 = solve_state(m0, vtrue, cfg, tops)
    lab1 = transport_labels(lab0, vtrue, cfg, tops)
    return m0, m1, lab0, lab1, vtrue


def _device_axes(grid: Grid):
    """Broadcastable f64 lattice coordinates on the device: (N1,1,1), (1,N2,1), (1,1,N3)."""
    dev = _lib.device()
    ax = [torch.arange(n, dtype=torch.float64, device=dev) * (2 * math.pi / n) for n in grid.dims]
    return ax[0].view(-1, 1, 1), ax[1].view(1, -1, 1), ax[2].view(1, 1, -1)


def velocity_tensor(K: int, grid: Grid, scale: float = 1.0) -> torch.Tensor:
    """scale * make_velocity(K) evaluated on the device in f64 (the formulas of
    velocity_array, synth.py:104-118) and rounded once to float32: for grids
    whose host f64 lattice would not fit (1024^3: ~26 GB per array)."""
    if K < 1:
        raise ValueError("K must be >= 1")
    x, y, z = _device_axes(grid)
    xc, yc, zc = x - math.pi, y - math.pi, z - math.pi
    out = torch.empty((3,) + tuple(grid.dims), dtype=torch.float32, device=x.device)
    for c in range(3):
        acc = torch.zeros(grid.dims, dtype=torch.float64, device=x.device)
        for k in range(1, K + 1):
            a = k ** -0.5
            if c == 0:
                acc += a * torch.cos(k * yc) * torch.cos(k * xc)
            elif c == 1:
                acc += a * torch.sin(k * zc) * torch.sin(k * yc)
            else:
                acc += a * torch.cos(k * xc) * torch.cos(k * zc)
        out[c] = (scale * acc).to(torch.float32)
        del acc
    return out


def c2_problem_device(grid: Grid, order: str = "cubic", n_t: int = 4):
    """c2_problem with the inputs evaluated on the device in f64 (same formulas
    as sphere_template / velocity_array, no host volume): for 1024^3 and up,
    where the host-side f64 lattice alone would take ~26 GB per array."""
    x, y, z = _device_axes(grid)
    r = torch.sqrt((x - math.pi) ** 2 + (y - math.pi) ** 2 + (z - math.pi) ** 2)
    m0 = ScalarField(grid, (0.5 * (1.0 - torch.tanh((r - 1.2) / 0.19635))).to(torch.float32))
    lab0 = LabelMap(grid, (r <= 1.2).to(torch.int32))
    del r
    vtrue = VectorField(grid, velocity_tensor(2, grid, 0.2))
    cfg = TransportConfig(n_t, order)
    tops = TransportOperators(vtrue, cfg)
    m1 = solve_state(m0, vtrue, cfg, tops)
    lab1 = transport_labels(lab0, vtrue, cfg, tops)
    del tops
    return m0, m1, lab0, lab1, vtrue
