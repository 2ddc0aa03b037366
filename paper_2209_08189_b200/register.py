"""`register(m0, m1, params)` -- the north star's drop-in entry point.

The reference has no single call for this; it is the composition used by its
CLI and experiment driver: gauss_newton_register (optim.py:275) -> solve_state
of the template (cli.py:134-141) -> relative_residual (optim.py:364) ->
optional transport_labels + dice_averages (experiment.py:132-135).  Everything
stays on the device; host <-> device traffic is the two input images (and
label maps) in, and whatever the caller pulls out of the result.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import GridError
from .grid import Grid, LabelMap, ScalarField, VectorField
from .metrics import DiceReport, dice_averages
from .optim import RegistrationConfig, SolverDiagnostics, gauss_newton_solve
from .synth import transport_labels


@dataclass
class RegistrationResult:
    velocity: VectorField
    deformed: ScalarField
    relative_residual: float
    diagnostics: SolverDiagnostics
    dice: DiceReport | None = None
    dice_pre: DiceReport | None = None

    @property
    def mismatch(self) -> float:
        return self.relative_residual


def _as_field(x, grid: Grid | None) -> ScalarField:
    if isinstance(x, ScalarField):
        return x
    if grid is None:
        grid = Grid(tuple(x.shape))
    return ScalarField(grid, x)


_side = {}


def _upload_async(items, pending: list) -> list:
    """Copy pinned host tensors to the device on a side stream (overlapping the
    Gauss-Newton solve); the caller's stream waits on the returned events
    before first use.  Anything else is returned unchanged."""
    out = []
    for x in items:
        if isinstance(x, torch.Tensor) and x.device.type == "cpu" and x.is_pinned() and x.dtype == torch.int32:
            dev = torch.cuda.current_device()
            st = _side.get(dev)
            if st is None:
                st = _side[dev] = torch.cuda.Stream()
            d = torch.empty(x.shape, dtype=torch.int32, device="cuda")
            st.wait_stream(torch.cuda.current_stream())   # d's allocation is ordered on the current stream
            with torch.cuda.stream(st):
                d.copy_(x, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(st)
            pending.append(ev)
            out.append(d)
        else:
            out.append(x)
    return out


def _download_async(pairs) -> torch.cuda.Event:
    """Device -> host copies (pinned destinations) on the side stream, ordered
    after the current stream's work; returns the completion event."""
    dev = torch.cuda.current_device()
    st = _side.get(dev)
    if st is None:
        st = _side[dev] = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for host, d in pairs:
            host.copy_(d, non_blocking=True)
            d.record_stream(st)
        ev = torch.cuda.Event()
        ev.record(st)
    return ev


def register(m0, m1, params: RegistrationConfig | dict | None = None, labels0=None, labels1=None,
             v0: VectorField | None = None, pre_dice: bool = False, grid: Grid | None = None,
             out_host: tuple | None = None) -> RegistrationResult:
    """Register template m0 to reference m1 (arrays, tensors or ScalarFields;
    pinned host tensors are uploaded asynchronously).  `grid` names the lattice
    when m0 is a bare array that is only this rank's x1 slab.  `out_host` =
    (velocity, deformed) pinned host tensors: the final velocity and deformed
    template are copied into them while the labels are transported and scored
    (complete when this call's stream work is)."""
    if params is None:
        cfg = RegistrationConfig()
    elif isinstance(params, dict):
        cfg = RegistrationConfig(**params)
    else:
        cfg = params
    m0 = _as_field(m0, grid)
    m1 = _as_field(m1, m0.grid)
    if out_host is not None:
        shp = tuple(m0.values.shape)
        if tuple(out_host[0].shape) != (3,) + shp or tuple(out_host[1].shape) != shp:
            raise GridError("out_host buffers do not match the velocity / deformed template shapes")
    # host label maps (pinned) upload on a side stream while the solver runs
    pending = []
    if labels0 is not None and labels1 is not None:
        labels0, labels1 = _upload_async([labels0, labels1], pending)
    v, diag, state = gauss_newton_solve(m0, m1, cfg, v0)
    res = RegistrationResult(v, state.deformed, diag.relative_residual, diag)
    copied = None
    if out_host is not None:
        copied = _download_async([(out_host[0], v.data), (out_host[1], state.deformed.values)])
    if labels0 is not None and labels1 is not None:
        for ev in pending:
            torch.cuda.current_stream().wait_event(ev)
        l0 = labels0 if isinstance(labels0, LabelMap) else LabelMap(m0.grid, labels0)
        l1 = labels1 if isinstance(labels1, LabelMap) else LabelMap(m0.grid, labels1)
        moved = transport_labels(l0, v, cfg.transport(), state.transport_ops)
        res.dice = dice_averages(moved, l1)
        if pre_dice:
            res.dice_pre = dice_averages(l0, l1)
    if copied is not None:
        torch.cuda.current_stream().wait_event(copied)
    return res
