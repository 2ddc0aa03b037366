"""Spectral prolongation on the device FFT engine (drop-in for
/root/reference/pkg/src/velreg/grid.py:181-226): coarse forward transform,
zero-padding with the symmetric Nyquist split, fine inverse transform."""
from __future__ import annotations

import torch

from . import _lib
from .errors import ResampleError
from .grid import Grid, ScalarField, VectorField


def prolong_spectral(field, target: Grid):
    from .diffops import workspace_for
    source = field.grid
    for ns, nt in zip(source.dims, target.dims):
        if nt < ns:
            raise ResampleError(f"prolongation target {target.dims} smaller than source {source.dims}")
    if isinstance(field, ScalarField):
        x, ncomp, shape = field.values, 1, target.dims
    elif isinstance(field, VectorField):
        x, ncomp, shape = field.data, 3, (3,) + target.dims
    else:
        raise TypeError(f"cannot prolong {type(field).__name__}")
    out = torch.empty(shape, dtype=torch.float32, device=x.device)
    wc, wf = workspace_for(source), workspace_for(target)
    rc = _lib.lib().vr_prolong_spectral(wc.plan, wf.plan, x.data_ptr(), ncomp, out.data_ptr(), _lib.stream())
    _lib.check(rc, "vr_prolong_spectral")
    return ScalarField(target, out) if ncomp == 1 else VectorField(target, out)
