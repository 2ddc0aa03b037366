"""Semi-Lagrangian transport solvers (drop-in for
/root/reference/pkg/src/velreg/transport.py).

One RK2 (Heun) characteristic trace per velocity iterate is shared by every
solve (forward trace for state / incremental state / Jacobian, backward trace
for the adjoint), with trapezoidal divergence source factors.  All sweeps run
in HBM on the sm_100a kernels of csrc/transport.cu; the host only sequences the
n_t steps and reads the non-finite flag where the reference checks
(transport.py:57-59, 119-121).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _lib
from . import dist as _dist
from .diffops import fd8_divergence_t, fd8_gradient_t
from .errors import TransportError
from .grid import Grid, ScalarField, VectorField

INTERP_ORDERS = ("linear", "cubic")

# slab sweeps with peer-memory ghosts: 0 = exchange, then one full-slab launch
# (default); 1 = interior planes overlap the exchange, boundary planes after
import os as _os
_SWEEP_SPLIT = int(_os.environ.get("VR_SWEEP_SPLIT", "0"))


@dataclass
class TransportConfig:
    n_t: int = 4
    interp_order: str = "cubic"
    direction: str = "forward"

    def __post_init__(self):
        if self.n_t < 1:
            raise ValueError(f"n_t must be >= 1, got {self.n_t}")
        if self.interp_order not in INTERP_ORDERS:
            raise ValueError(f"interp_order must be in {INTERP_ORDERS}")
        if self.direction not in ("forward", "backward"):
            raise ValueError("direction must be 'forward' or 'backward'")

    @property
    def dt(self) -> float:
        return 1.0 / self.n_t


@dataclass
class Characteristics:
    """Departure points of every voxel, stored as index-unit displacements
    (3, N1, N2, N3) float32; `.points` gives the reference's radians in
    [0, 2*pi) (float64) on demand."""

    grid: Grid
    displacement: torch.Tensor
    dt: float

    @property
    def points(self) -> torch.Tensor:
        out = torch.empty((3,) + self.grid.dims, dtype=torch.float64, device=self.displacement.device)
        _lib.check(_lib.lib().vr_disp_to_points(self.displacement.data_ptr(), _lib.dims_arg(self.grid.dims),
                                                out.data_ptr(), _lib.stream()), "vr_disp_to_points")
        return out


def cfl_number(v: VectorField, dt: float) -> float:
    """transport.py:53-54"""
    return dt * v.max_pointwise_norm() / min(v.grid.spacing)


def _check_finite_velocity(v: VectorField) -> None:
    if v.stats()[1] > 0:
        raise TransportError("velocity field contains non-finite values")


def _order(order: str) -> int:
    if order not in INTERP_ORDERS:
        raise ValueError(f"interpolation order must be one of {INTERP_ORDERS}, got {order!r}")
    return _lib.ORDER[order]


def _trace(v: torch.Tensor, dims, dt: float, order: str, div: torch.Tensor | None = None):
    disp_f = torch.empty_like(v)
    disp_b = torch.empty_like(v)
    fac_j = fac_a = None
    if div is not None:
        fac_j = torch.empty_like(div)
        fac_a = torch.empty_like(div)
    rc = _lib.lib().vr_trace_rk2(v.data_ptr(), _lib.dims_arg(dims), float(dt), _order(order), disp_f.data_ptr(),
                                 disp_b.data_ptr(), _lib.ptr(div), _lib.ptr(fac_j), _lib.ptr(fac_a), _lib.stream())
    _lib.check(rc, "vr_trace_rk2")
    return disp_f, disp_b, fac_j, fac_a


def trace_characteristics(v: VectorField, dt: float, order: str = "cubic") -> Characteristics:
    """RK2 (Heun) backward trace: x* = x - dt*v(x), X = x - dt/2*(v(x) + v(x*))
    (transport.py:66-76)."""
    if not dt > 0:
        raise ValueError(f"dt must be positive, got {dt}")
    _check_finite_velocity(v)
    disp_f, _, _, _ = _trace(v.data, v.grid.dims, dt, order)
    return Characteristics(v.grid, disp_f, dt)


def advect(values: torch.Tensor, disp: torch.Tensor, order: str, factor: torch.Tensor | None = None,
           out: torch.Tensor | None = None, flag: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(values.shape, dtype=torch.float32, device=values.device)
    rc = _lib.lib().vr_advect(values.data_ptr(), _lib.dims_arg(values.shape[-3:]), disp.data_ptr(),
                              _lib.ptr(factor), _order(order), out.data_ptr(), _lib.ptr(flag), _lib.stream())
    _lib.check(rc, "vr_advect")
    return out


def interpolate(f: ScalarField, chars: Characteristics, order: str) -> ScalarField:
    if f.grid != chars.grid:
        raise TransportError("field and characteristics grids differ")
    return ScalarField(f.grid, advect(f.values, chars.displacement, order))


class TransportOperators:
    """Shared per-velocity data for all transport solves at one iterate
    (transport.py:89-116): both characteristic traces, the FD8 divergence and
    the trapezoidal source factors, built by ONE fused trace kernel after the
    divergence kernel.  The factors are stored as ratios
    jac_factor = jac_numer / jac_denom and adj_factor = adj_numer / adj_denom."""

    def __init__(self, v: VectorField, cfg: TransportConfig, defer_checks: bool = False):
        self.v = v
        self.cfg = cfg
        self.grid = v.grid
        self.ctx = _dist.for_grid(v.grid.dims)
        if defer_checks and self.ctx is None:
            # read with the caller's next reduction (ObjectiveState): same error
            from .reductions import vecstats_dev
            st = vecstats_dev(v.data)
            _lib.defer_check(st[2:3], TransportError("velocity field contains non-finite values"))
        else:
            _check_finite_velocity(v)
        if self.ctx is None:
            self.div = fd8_divergence_t(v.data)
            disp_f, disp_b, self.jac_factor, self.adj_factor = _trace(v.data, v.grid.dims, cfg.dt, cfg.interp_order,
                                                                      self.div)
        else:
            disp_f, disp_b = self._trace_slab(v.data)
        self.forward = Characteristics(v.grid, disp_f, cfg.dt)
        self.backward = Characteristics(v.grid, disp_b, cfg.dt)
        # non-finite flags: [0] eager checks, [1] / [2] the matvec's deferred
        # incremental-state / adjoint checks, [3] / [4] ObjectiveState's deferred
        # state / adjoint checks
        self.flags = torch.zeros((5, 1), dtype=torch.int32, device=v.data.device)

    # ---- x1-slab decomposition (dist.py) ----------------------------------------
    def _trace_slab(self, v: torch.Tensor):
        """Ghost width from the global max |v1| (allreduce), one halo exchange
        of v (covers both the FD8 divergence and the RK2 star points), one of
        div (for the source factors), then the slab trace kernel."""
        from .reductions import minmax
        ctx, cfg = self.ctx, self.cfg
        mn, mx, _, _ = minmax(v[0])          # allreduced on the device, one read
        vmax1 = max(abs(float(mn)), abs(float(mx)))
        w = _dist.ghost_width(vmax1, cfg.dt, self.grid.dims[0], cfg.interp_order)
        ldims = ctx.local_dims
        self.div = fd8_divergence_t(v)
        disp_f = torch.empty_like(v)
        disp_b = torch.empty_like(v)
        self.jac_factor = torch.empty_like(self.div)
        self.adj_factor = torch.empty_like(self.div)
        while True:
            self.w = w
            v_ext = ctx.halo(v, w)          # contiguous ghost-extended copies, once per iterate
            d_ext = ctx.halo(self.div, w)
            _lib.check(_lib.lib().vr_trace_rk2_slab(v_ext.data_ptr(), _lib.dims_arg(ldims), ctx.dims[0], w,
                                                    float(cfg.dt), _order(cfg.interp_order), disp_f.data_ptr(),
                                                    disp_b.data_ptr(), d_ext.data_ptr(), self.jac_factor.data_ptr(),
                                                    self.adj_factor.data_ptr(), _lib.stream()), "vr_trace_rk2_slab")
            # The width above bounds the Heun star point by max|v1|, but the
            # second stage uses the INTERPOLATED v(x*), which cubic Lagrange can
            # overshoot.  The slab gathers clamp the x1 base index into the
            # ghosts, so check the actual departure displacements (both traces,
            # all ranks) and redo the trace with wider ghosts if any departure
            # stencil -- or an interior-plane stencil of the overlapped sweeps --
            # would leave the exchanged planes.
            mn_f, mx_f, mn_b, mx_b = minmax(disp_f[0], disp_b[0])
            dmax = float(max(abs(mn_f), abs(mx_f), abs(mn_b), abs(mx_b)))
            if not math.isfinite(dmax):
                raise TransportError("characteristic trace produced non-finite displacements")
            need = _dist.ghost_width_for_displacement(dmax, cfg.interp_order)
            if need <= w:
                return disp_f, disp_b
            if need > ldims[0]:
                raise TransportError(f"departure points travel {dmax:.1f} x1 planes, more than the slab depth "
                                     f"{ldims[0]}; use fewer ranks or a larger n_t")
            w = need

    def sweep(self, values: torch.Tensor, disp: torch.Tensor, factor: torch.Tensor | None = None,
              out: torch.Tensor | None = None, flag=None) -> torch.Tensor:
        """One SL step dst = interp(values, departure) [* factor] (halo'd on slabs)."""
        if self.ctx is None:
            return advect(values, disp, self.cfg.interp_order, factor=factor, out=out, flag=flag)
        if out is None:
            out = torch.empty(values.shape, dtype=torch.float32, device=values.device)
        dims = _lib.dims_arg(self.ctx.local_dims)
        order = _order(self.cfg.interp_order)

        def launch(lo, hi, x0, nx):
            _lib.check(_lib.lib().vr_advect_slab(values.data_ptr(), lo.data_ptr(), hi.data_ptr(), dims, self.w,
                                                 disp.data_ptr(), _lib.ptr(factor), order, out.data_ptr(),
                                                 _lib.ptr(flag), x0, nx, _lib.stream()), "vr_advect_slab")

        self._overlapped(values, launch)
        return out

    def _overlapped(self, values: torch.Tensor, launch) -> None:
        """Ghost exchange in flight while the interior planes [w, L1 - w) (whose
        stencils never leave the slab) are swept; boundary planes afterwards."""
        ctx, w = self.ctx, self.w
        L1 = ctx.local_dims[0]
        with _lib.timed("dist.sweep"):
            lo, hi, works = ctx.ghosts_async(values, w)
            if ctx.mesh is not None and _SWEEP_SPLIT == 0:
                # copy-engine ghosts land in ~10 us: wait, then ONE full-slab launch
                # (the interior / boundary split costs two extra launch tails)
                ctx.finish(works)
                launch(lo, hi, 0, L1)
            elif L1 > 2 * w:
                launch(lo, hi, w, L1 - 2 * w)
                ctx.finish(works)
                launch(lo, hi, 0, w)
                launch(lo, hi, L1 - w, w)
            else:
                ctx.finish(works)
                launch(lo, hi, 0, L1)

    def inc_step(self, u: torch.Tensor, vt: torch.Tensor, gnext: torch.Tensor, last: int, out: torch.Tensor,
                 flag=None) -> None:
        """Incremental-state step (transport.py:174-183) along the forward trace."""
        lib = _lib.lib()
        cfg = self.cfg
        dims = _lib.dims_arg(u.shape[-3:])
        disp = self.forward.displacement.data_ptr()
        if self.ctx is None:
            rc = lib.vr_incstate_step(u.data_ptr(), dims, disp, vt.data_ptr(), gnext.data_ptr(), float(cfg.dt),
                                      _order(cfg.interp_order), last, out.data_ptr(), _lib.ptr(flag), _lib.stream())
            _lib.check(rc, "vr_incstate_step")
        else:
            def launch(lo, hi, x0, nx):
                _lib.check(lib.vr_incstate_step_slab(u.data_ptr(), lo.data_ptr(), hi.data_ptr(), dims, self.w, disp,
                                                     vt.data_ptr(), gnext.data_ptr(), float(cfg.dt),
                                                     _order(cfg.interp_order), last, out.data_ptr(), _lib.ptr(flag),
                                                     x0, nx, _lib.stream()), "vr_incstate_step_slab")

            self._overlapped(u, launch)

    def advect_step(self, values: torch.Tensor, out: torch.Tensor | None = None, flag=None) -> torch.Tensor:
        return self.sweep(values, self.forward.displacement, out=out, flag=flag)

    def advect_back_step(self, values: torch.Tensor, out: torch.Tensor | None = None, flag=None) -> torch.Tensor:
        return self.sweep(values, self.backward.displacement, out=out, flag=flag)

    # non-finite guard (transport.py:119-121) read back at the reference's check points
    def arm(self, slot: int = 0) -> torch.Tensor:
        flag = self.flags[slot]
        if _lib.is_deferred(flag):
            _lib.run_deferred()
        flag.zero_()
        return flag

    def raise_if_flagged(self, what: str, slot: int = 0, deferred: bool = False) -> None:
        flag = self.flags[slot]
        exc = TransportError(f"{what} produced non-finite values")
        if deferred:
            _lib.defer_check(flag, exc)
        elif int(flag.item()) != 0:
            raise exc


def _ops_for(v: VectorField, cfg: TransportConfig, ops) -> TransportOperators:
    return ops or TransportOperators(v, cfg)


def solve_state_series(m0: ScalarField, v: VectorField, cfg: TransportConfig,
                       ops: TransportOperators = None, _deferred: bool = False) -> torch.Tensor:
    """All n_t + 1 snapshots of the transported template, shape (n_t+1,) + dims
    (transport.py:124-135)."""
    if m0.grid != v.grid:
        raise TransportError("template and velocity grids differ")
    ops = _ops_for(v, cfg, ops)
    series = torch.empty((cfg.n_t + 1,) + tuple(m0.values.shape), dtype=torch.float32, device=m0.values.device)
    series[0].copy_(m0.values)
    slot = 3 if _deferred else 0
    flag = ops.arm(slot)
    for j in range(cfg.n_t):
        ops.advect_step(series[j], out=series[j + 1], flag=flag if j == cfg.n_t - 1 else None)
    ops.raise_if_flagged("state solve", slot, _deferred)
    return series


def solve_state(m0: ScalarField, v: VectorField, cfg: TransportConfig,
                ops: TransportOperators = None) -> ScalarField:
    """Deformed template m(., 1) after n_t semi-Lagrangian steps (transport.py:138-142);
    ping-pongs two buffers instead of keeping the series."""
    if m0.grid != v.grid:
        raise TransportError("template and velocity grids differ")
    ops = _ops_for(v, cfg, ops)
    a = m0.values
    bufs = [torch.empty_like(a), torch.empty_like(a)]
    flag = ops.arm()
    for j in range(cfg.n_t):
        dst = bufs[j % 2]
        ops.advect_step(a, out=dst, flag=flag if j == cfg.n_t - 1 else None)
        a = dst
    ops.raise_if_flagged("state solve")
    return ScalarField(m0.grid, a)


def solve_adjoint(final_lambda: ScalarField, v: VectorField, cfg: TransportConfig,
                  ops: TransportOperators = None) -> torch.Tensor:
    """Backward continuity solve; all snapshots indexed by forward time
    (transport.py:145-157)."""
    if final_lambda.grid != v.grid:
        raise TransportError("adjoint final condition and velocity grids differ")
    ops = _ops_for(v, cfg, ops)
    series = torch.empty((cfg.n_t + 1,) + tuple(final_lambda.values.shape), dtype=torch.float32,
                         device=v.data.device)
    series[cfg.n_t].copy_(final_lambda.values)
    _adjoint_sweep(series, ops, cfg)
    return series


def _adjoint_sweep(series: torch.Tensor, ops: TransportOperators, cfg: TransportConfig,
                   deferred: bool = False, slot: int | None = None) -> None:
    if slot is None:
        slot = 2 if deferred else 0
    flag = ops.arm(slot)
    for j in range(cfg.n_t - 1, -1, -1):
        ops.sweep(series[j + 1], ops.backward.displacement, factor=ops.adj_factor, out=series[j],
                  flag=flag if j == 0 else None)
    ops.raise_if_flagged("adjoint solve", slot, deferred)


class LazyGradientSeries:
    """grad m^j computed on demand (lean layout): indexing returns the FD8
    gradient of snapshot j in a reused (3,) + dims buffer, valid until the next
    index on the same stream (kernels consuming it are stream-ordered before
    the next FD8 launch overwrites it).  Saves (n_t+1) * 12 B/voxel of HBM --
    what makes C3 (1024^3, n_t = 16) fit on 4 B200s."""

    def __init__(self, m_series: torch.Tensor):
        self.m_series = m_series
        self.buf = torch.empty((3,) + tuple(m_series.shape[1:]), dtype=torch.float32, device=m_series.device)

    def __len__(self):
        return self.m_series.shape[0]

    def __getitem__(self, j: int) -> torch.Tensor:
        return fd8_gradient_t(self.m_series[j], out=self.buf)


def gradient_series(m_series: torch.Tensor) -> torch.Tensor:
    """FD8 gradient of every snapshot, (n_t+1, 3) + dims (optim.py:127-135)."""
    out = torch.empty((m_series.shape[0], 3) + tuple(m_series.shape[1:]), dtype=torch.float32,
                      device=m_series.device)
    for j in range(m_series.shape[0]):
        fd8_gradient_t(m_series[j], out=out[j])
    return out


def _incremental(grad_m_series: torch.Tensor, vt: torch.Tensor, ops: TransportOperators, cfg: TransportConfig,
                 last_mode: int, out: torch.Tensor | None = None, deferred: bool = False) -> torch.Tensor:
    lib = _lib.lib()
    dims = tuple(vt.shape[-3:])
    d = _lib.dims_arg(dims)
    st = _lib.stream()
    u = torch.empty(dims, dtype=torch.float32, device=vt.device)
    _lib.check(lib.vr_incstate_init(vt.data_ptr(), grad_m_series[0].data_ptr(), d, float(cfg.dt), u.data_ptr(), st),
               "vr_incstate_init")
    other = torch.empty_like(u)
    slot = 1 if deferred else 0
    flag = ops.arm(slot)
    for j in range(cfg.n_t):
        last = j == cfg.n_t - 1
        dst = out if (last and out is not None) else other
        ops.inc_step(u, vt, grad_m_series[j + 1], last_mode if last else 0, dst, flag if last else None)
        if not last:
            u, other = dst, u
        else:
            u = dst
    ops.raise_if_flagged("incremental state solve", slot, deferred)
    return u


def solve_incremental_state(m_series: torch.Tensor, v: VectorField, v_tilde: VectorField,
                            cfg: TransportConfig, ops: TransportOperators = None,
                            grad_m_series: torch.Tensor = None) -> ScalarField:
    """Linearized state dm~/dt + v.grad(m~) = -v~.grad(m), m~(0) = 0 (transport.py:160-185)."""
    ops = _ops_for(v, cfg, ops)
    if grad_m_series is None:
        grad_m_series = gradient_series(torch.as_tensor(m_series).to(v.data.device, torch.float32))
    return ScalarField(v.grid, _incremental(grad_m_series, v_tilde.data, ops, cfg, 1))


def jacobian_determinant(v: VectorField, cfg: TransportConfig, ops: TransportOperators = None) -> ScalarField:
    """det of the deformation gradient at t = 1 via dJ/dt + v.grad(J) = J div(v),
    J(0) = 1 (transport.py:188-197)."""
    ops = _ops_for(v, cfg, ops)
    cur = torch.empty(tuple(v.data.shape[1:]), dtype=torch.float32, device=v.data.device)
    from .reductions import fill
    fill(cur, 1.0)
    other = torch.empty_like(cur)
    flag = ops.arm()
    for j in range(cfg.n_t):
        ops.sweep(cur, ops.forward.displacement, factor=ops.jac_factor, out=other,
                  flag=flag if j == cfg.n_t - 1 else None)
        cur, other = other, cur
    ops.raise_if_flagged("Jacobian-determinant solve")
    return ScalarField(v.grid, cur)
