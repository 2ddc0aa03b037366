"""Periodic scattered interpolation (drop-in for
/root/reference/pkg/src/velreg/interp.py:112-128).

`interpolate_values(values, points, order, spacing)` evaluates the periodic
trilinear / tricubic-Lagrange interpolant of `values` at `points` (shape
(3, ...), radians) with the sm_100a gather kernel.  The reference's numba
kernels compute in float64 and cast back to the value dtype; here values are
float32, points are float32 or float64 (index = point / h is formed in float64),
and the weights/accumulation are float32 (relative difference ~1e-7).
"""
from __future__ import annotations

import torch

from . import _lib
from .grid import TWO_PI, to_device

ORDERS = ("linear", "cubic")


def interpolate_values(values, points, order: str, spacing) -> torch.Tensor:
    """Evaluate the periodic interpolant of `values` at `points` (shape (3, ...))."""
    if order not in ORDERS:
        raise ValueError(f"interpolation order must be one of {ORDERS}, got {order!r}")
    vals = to_device(values)
    dims = tuple(vals.shape)
    for n, h in zip(dims, spacing):
        if abs(h - TWO_PI / n) > 1e-12 * TWO_PI:
            raise ValueError("spacing must be 2*pi/N per axis (periodic [0, 2*pi)^3 lattice)")
    if isinstance(points, torch.Tensor) and points.dtype == torch.float64:
        pts = points.to(_lib.device()).contiguous()
    elif not isinstance(points, torch.Tensor) and str(getattr(points, "dtype", "")) == "float64":
        pts = to_device(points, torch.float64)
    else:
        pts = to_device(points, torch.float32)
    npts = pts[0].numel()
    out = torch.empty(tuple(pts.shape[1:]), dtype=torch.float32, device=vals.device)
    rc = _lib.lib().vr_interp_points(vals.data_ptr(), _lib.dims_arg(dims), pts.data_ptr(),
                                     int(pts.dtype == torch.float64), npts, _lib.ORDER[order],
                                     out.data_ptr(), _lib.stream())
    _lib.check(rc, "vr_interp_points")
    return out
