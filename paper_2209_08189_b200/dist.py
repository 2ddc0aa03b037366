"""x1-slab domain decomposition across the GPUs of one node.

Rank r of P owns x1 planes [r*L1, (r+1)*L1), L1 = N1/P, of every voxel field
(the paper's slab axis).  Three exchange steps exist, all issued
through torch.distributed (NCCL on GPUs, gloo for the CPU tests of the host
logic):

* halo      -- ghost x1 planes for the FD8 stencil (4) and the semi-Lagrangian
               gathers (ceil(max |x1 displacement|) + stencil, from an
               allreduce-max of the velocity), one batched send/recv pair per
               neighbour;
* transpose -- one all-to-all per component before and after the x1 pass of
               every spectral operator (x1 slabs <-> x2 slabs);
* allreduce -- the f64 scalars of every reduction (dots, norms, extrema,
               non-finite counts, Dice counts).

`activate(ctx)` installs the context process-wide; the operator modules
(diffops, transport, reductions, synth) consult `current()` and switch to the
slab kernels, so optim.py's Gauss-Newton / PCG control flow runs unchanged.
"""
from __future__ import annotations

import contextlib
import math

import numpy as np
import torch
import torch.distributed as tdist

from . import _lib

_CTX = None


def current():
    return _CTX


def for_grid(dims):
    """The active context if it decomposes a lattice of `dims`, else None (a
    field on another grid is single-domain even while a context is active)."""
    ctx = _CTX
    if ctx is not None and tuple(ctx.dims) == tuple(int(n) for n in dims):
        return ctx
    return None


def for_shape(shape):
    """The active context if a tensor of `shape` (..., L1, N2, N3) is one of its
    local slabs, else None.  Every slab-aware operator and reduction routes
    through this (or `for_grid`), so one call never mixes slab kernels with a
    replicated field."""
    ctx = _CTX
    if ctx is not None and len(shape) >= 3 and tuple(shape[-3:]) == tuple(ctx.local_dims):
        return ctx
    return None


@contextlib.contextmanager
def activate(ctx):
    global _CTX
    prev = _CTX
    _CTX = ctx
    try:
        yield ctx
    finally:
        _CTX = prev


class SlabContext:
    """Decomposition of a global (N1, N2, N3) lattice into x1 slabs."""

    def __init__(self, dims, group=None, rank: int | None = None, world: int | None = None):
        self.dims = tuple(int(n) for n in dims)
        self.group = group
        self.rank = tdist.get_rank(group) if rank is None else rank
        self.world = tdist.get_world_size(group) if world is None else world
        n1, n2, n3 = self.dims
        if n1 % self.world or n2 % self.world:
            raise ValueError(f"N1={n1} and N2={n2} must be divisible by the number of ranks {self.world}")
        self.L1 = n1 // self.world
        self.L2 = n2 // self.world
        self.x0 = self.rank * self.L1
        self.local_dims = (self.L1, n2, n3)
        self.left = (self.rank - 1) % self.world
        self.right = (self.rank + 1) % self.world

    # ---- collectives on small host arrays ---------------------------------------
    def _dev(self):
        return torch.device("cuda", torch.cuda.current_device()) if tdist.get_backend(self.group) == "nccl" \
            else torch.device("cpu")

    def allreduce(self, values, op: str = "sum") -> np.ndarray:
        t = torch.as_tensor(np.asarray(values, dtype=np.float64).reshape(-1), device=self._dev())
        rop = {"sum": tdist.ReduceOp.SUM, "max": tdist.ReduceOp.MAX, "min": tdist.ReduceOp.MIN}[op]
        tdist.all_reduce(t, op=rop, group=self.group)
        return t.cpu().numpy()

    def allreduce_(self, t: torch.Tensor, op: str = "sum") -> torch.Tensor:
        """In-place allreduce of a device tensor (no host round trip)."""
        rop = {"sum": tdist.ReduceOp.SUM, "max": tdist.ReduceOp.MAX, "min": tdist.ReduceOp.MIN}[op]
        with _lib.timed("dist.allreduce"):
            tdist.all_reduce(t, op=rop, group=self.group)
        return t

    def barrier(self) -> None:
        if self.world > 1:
            tdist.barrier(group=self.group)

    # ---- ghost planes --------------------------------------------------------------
    def ghosts(self, x: torch.Tensor, w: int) -> tuple:
        """(lo, hi) ghost blocks (..., w, N2, N3) of the local slab x (..., L1, N2, N3):
        lo = the w periodic planes preceding this slab, hi = the w following it.
        The slab itself is not copied; kernels read lo / x / hi by plane."""
        L1 = x.shape[-3]
        if w > L1:
            raise ValueError(f"ghost width {w} exceeds the slab depth {L1}; use fewer ranks")
        send_lo = x[..., :w, :, :]            # -> left neighbour's hi ghost
        send_hi = x[..., L1 - w:, :, :]       # -> right neighbour's lo ghost
        if self.world == 1:
            return send_hi.contiguous(), send_lo.contiguous()
        with _lib.timed("dist.ghosts"):
            lo, hi, works = self.ghosts_async(x, w)
            self.finish(works)
        return lo, hi

    def ghosts_async(self, x: torch.Tensor, w: int) -> tuple:
        """Post the ghost exchange and return (lo, hi, works) without waiting, so
        the interior planes can be swept meanwhile; `finish(works)` makes the
        current stream wait for the ghosts."""
        L1 = x.shape[-3]
        if w > L1:
            raise ValueError(f"ghost width {w} exceeds the slab depth {L1}; use fewer ranks")
        send_lo = x[..., :w, :, :]
        send_hi = x[..., L1 - w:, :, :]
        if self.world == 1:
            return send_hi.contiguous(), send_lo.contiguous(), []
        send_lo = send_lo.contiguous()
        send_hi = send_hi.contiguous()
        hi = torch.empty_like(send_lo)        # <- right neighbour's first planes
        lo = torch.empty_like(send_hi)        # <- left neighbour's last planes
        ops = [tdist.P2POp(tdist.isend, send_lo, self.left, self.group),
               tdist.P2POp(tdist.isend, send_hi, self.right, self.group),
               tdist.P2POp(tdist.irecv, hi, self.right, self.group),
               tdist.P2POp(tdist.irecv, lo, self.left, self.group)]
        return lo, hi, tdist.batch_isend_irecv(ops)

    @staticmethod
    def finish(works) -> None:
        for req in works:
            req.wait()

    def halo(self, x: torch.Tensor, w: int) -> torch.Tensor:
        """(..., L1, N2, N3) -> (..., L1 + 2w, N2, N3) extended copy (tests / tools)."""
        lo, hi = self.ghosts(x, w)
        return torch.cat([lo, x, hi], dim=-3)

    # ---- transposes -------------------------------------------------------------
    def alltoall(self, out: torch.Tensor, inp: torch.Tensor, async_op: bool = False):
        """Equal-split all-to-all along dim 0 of flat views (x1 slabs <-> x2 slabs);
        async_op returns the work handle (wait() = stream wait)."""
        if self.world == 1:
            out.copy_(inp)
            return None
        if async_op:
            return tdist.all_to_all_single(out, inp, group=self.group, async_op=True)
        with _lib.timed("dist.alltoall"):
            tdist.all_to_all_single(out, inp, group=self.group)
        return None

    # ---- synthetic-input helpers -------------------------------------------------
    def local_coords(self) -> np.ndarray:
        """(3, L1, N2, N3) lattice coordinates of this rank's planes."""
        n1, n2, n3 = self.dims
        ax = [np.arange(self.x0, self.x0 + self.L1) * (2 * np.pi / n1), np.arange(n2) * (2 * np.pi / n2),
              np.arange(n3) * (2 * np.pi / n3)]
        return np.stack(np.meshgrid(*ax, indexing="ij"))


def ghost_width(vmax1: float, dt: float, n1: int, order: str) -> int:
    """x1 ghost planes covering every departure point plus the stencil."""
    h1 = 2 * math.pi / n1
    return max(4, int(math.ceil(dt * vmax1 / h1)) + (3 if order == "cubic" else 2))


def ghost_width_for_displacement(dmax1: float, order: str) -> int:
    """Smallest ghost width whose planes hold every departure stencil of x1
    displacement |d1| <= dmax1: the slab gathers accept base indices in
    [1 - w, L1 + w - 3] (cubic) / [-w, L1 + w - 2] (linear)."""
    return int(math.ceil(dmax1)) + (1 if order == "cubic" else 0)
