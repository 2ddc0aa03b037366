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
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import Grid, LabelMap, ScalarField, VectorField
from .transport import TransportConfig, TransportOperators, solve_state


# ---- SYN benchmark (synth.py:22-101; §4 "SYN") ------------------------
@dataclass
class SynthSpec:
    """synth.py:22-39: shape count, spherical-harmonic degree / order,
    velocity frequency K, seed, and the constant-radius test hook."""
    grid: Grid
    num_shapes: int = 10
    degree: int = 8
    order: int = 6
    velocity_frequency: int = 4
    seed: int = 0
    fixed_radius: float = None

    def __post_init__(self):
        if self.num_shapes < 1:
            raise ValueError("num_shapes must be >= 1")
        if not 0 <= self.order <= self.degree:
            raise ValueError("need 0 <= order <= degree")
        if self.velocity_frequency < 1:
            raise ValueError("velocity frequency K must be >= 1")


def assoc_legendre(l: int, m: int, x) -> np.ndarray:
    """Associated Legendre P_l^m with Condon-Shortley phase, upward recurrence
    (synth.py:42-62); host numpy utility -- the device template evaluates the
    same recurrence per voxel (csrc/synth.cu)."""
    if not 0 <= m <= l:
        raise ValueError(f"need 0 <= m <= l, got l={l}, m={m}")
    x = np.asarray(x, dtype=np.float64)
    if np.any(np.abs(x) > 1.0 + 1e-14):
        raise ValueError("associated Legendre argument must satisfy |x| <= 1")
    pmm = np.ones_like(x)
    if m > 0:
        s = np.sqrt(np.clip(1.0 - x * x, 0.0, None))
        pmm = (-1.0) ** m * float(math.prod(range(1, 2 * m, 2))) * s ** m
    if l == m:
        return pmm
    pm1 = x * (2 * m + 1) * pmm
    if l == m + 1:
        return pm1
    for ll in range(m + 2, l + 1):
        pmm, pm1 = pm1, (x * (2 * ll - 1) * pm1 - (ll + m - 1) * pmm) / (ll - m)
    return pm1


def _sh_norm(l: int, m: int) -> float:
    return math.sqrt((2 * l + 1) / (4.0 * math.pi) * math.factorial(l - m) / math.factorial(l + m))


def spherical_harmonic_magnitude(l: int, m: int, theta, phi) -> np.ndarray:
    """|Y_l^m(theta, phi)| (synth.py:65-74): the azimuth only enters a
    unit-modulus phase."""
    del theta
    return _sh_norm(l, m) * np.abs(assoc_legendre(l, m, np.cos(phi)))


QUARTER_TURNS = (0.0, 0.5 * math.pi, math.pi, 1.5 * math.pi)
OFFSET_BOUND = 0.4 * math.pi


def _syn_shapes(spec: SynthSpec) -> np.ndarray:
    """The reference's random draws, in its order (synth.py:88-92): per shape
    a centre in [-0.4 pi, 0.4 pi]^3 and two quarter turns (the azimuthal one
    is drawn but cancels in |Y_l^m|).  Rows {c1, c2, c3, phi_hat}."""
    rng = np.random.default_rng(spec.seed)
    rows = []
    for _ in range(spec.num_shapes):
        center = rng.uniform(-OFFSET_BOUND, OFFSET_BOUND, size=3)
        _theta_hat = QUARTER_TURNS[rng.integers(0, 4)]
        phi_hat = QUARTER_TURNS[rng.integers(0, 4)]
        rows.append([center[0], center[1], center[2], phi_hat])
    return np.ascontiguousarray(rows, dtype=np.float64)


def make_template(spec: SynthSpec):
    """Template image (the label ids as intensities) and its label map
    (synth.py:77-101), evaluated on the device -- one thread per voxel over all
    shapes (csrc/synth.cu) -- for this rank's x1 slab when a decomposition of
    the grid is active."""
    from . import dist
    grid = spec.grid
    ctx = dist.for_grid(grid.dims)
    x0, nx = (ctx.x0, ctx.L1) if ctx is not None else (0, grid.dims[0])
    shape = (nx,) + tuple(grid.dims[1:])
    labels = torch.empty(shape, dtype=torch.int32, device=_lib.device())
    image = torch.empty(shape, dtype=torch.float32, device=labels.device)
    shapes = _syn_shapes(spec)
    fixed = -1.0 if spec.fixed_radius is None else float(spec.fixed_radius)
    l, m = spec.degree, spec.order
    rc = _lib.lib().vr_syn_template(_lib.dims_arg(grid.dims), int(x0), int(nx), shapes.ctypes.data,
                                    int(shapes.shape[0]), int(l), int(m), _sh_norm(l, m),
                                    float(math.prod(range(1, 2 * m, 2))), fixed, labels.data_ptr(),
                                    image.data_ptr(), _lib.stream())
    _lib.check(rc, "vr_syn_template")
    return ScalarField(grid, image), LabelMap(grid, labels, spec.num_shapes)


def make_syn_problem(spec: SynthSpec, n_t: int = 4, order: str = "cubic"):
    """SYN pair (SPEC.md synthgen, §4): template + labels, velocity
    make_velocity(K) evaluated on the device, reference image and labels by
    transport (synth.py:134-141).  Returns (m0, m1, labels0, labels1, v)."""
    m0, l0 = make_template(spec)
    v = VectorField(spec.grid, velocity_tensor(spec.velocity_frequency, spec.grid))
    m1, l1 = make_reference(m0, l0, v, TransportConfig(n_t, order))
    return m0, m1, l0, l1, v


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
    """Broadcastable f64 lattice coordinates on the device: (L1,1,1), (1,N2,1),
    (1,1,N3) -- this rank's x1 planes when a decomposition of the grid is active."""
    from . import dist
    dev = _lib.device()
    ax = [torch.arange(n, dtype=torch.float64, device=dev) * (2 * math.pi / n) for n in grid.dims]
    ctx = dist.for_grid(grid.dims)
    if ctx is not None:
        ax[0] = ax[0][ctx.x0:ctx.x0 + ctx.L1]
    return ax[0].view(-1, 1, 1), ax[1].view(1, -1, 1), ax[2].view(1, 1, -1)


def velocity_tensor(K: int, grid: Grid, scale: float = 1.0) -> torch.Tensor:
    """scale * make_velocity(K) evaluated on the device in f64 (the formulas of
    velocity_array, synth.py:104-118) and rounded once to float32: for grids
    whose host f64 lattice would not fit (1024^3: ~26 GB per array)."""
    if K < 1:
        raise ValueError("K must be >= 1")
    x, y, z = _device_axes(grid)
    xc, yc, zc = x - math.pi, y - math.pi, z - math.pi
    shape = (x.shape[0],) + tuple(grid.dims[1:])
    out = torch.empty((3,) + shape, dtype=torch.float32, device=x.device)
    for c in range(3):
        acc = torch.zeros(shape, dtype=torch.float64, device=x.device)
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
