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
import os

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


class _DevPtr:
    """Zero-copy torch view of raw device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                          "version": 3}


def _view(ptr: int, nbytes: int, dtype: torch.dtype, shape) -> torch.Tensor:
    t = torch.as_tensor(_DevPtr(ptr, nbytes), device=_lib.device())
    return t.view(dtype).view(shape)


class _PeerWork:
    """Completion of one peer exchange: wait() makes the current stream wait
    for the senders' epoch flags (cuStreamWaitValue64, no host round trip)."""

    def __init__(self, mesh, flags):
        self.mesh = mesh
        self.flags = flags          # [(local flag address, epoch)]

    def wait(self) -> None:
        st = _lib.stream()
        by_epoch = {}
        for addr, e in self.flags:
            by_epoch.setdefault(e, []).append(addr)
        for e, addrs in by_epoch.items():
            self.mesh.wait_many(addrs, e, st)


class PeerMesh:
    """Peer-memory transport of one SlabContext (csrc/peer.cu): symmetric
    IPC-mapped receive buffers on every rank, copy-engine copies on a side
    stream, and per-(source, channel) uint64 epoch flags in the receiver's
    memory (written by the sender behind its data, awaited on the receiver's
    stream).  Replaces NCCL for the ghost planes and the spectral transposes;
    NCCL keeps the scalar allreduces.  Buffer creation and growth are
    collective (every rank makes the same calls in the same order)."""

    GHOST_LO, GHOST_HI, A2A = 0, 1, 2
    NCH = 4

    def __init__(self, ctx):
        import ctypes as C
        self.C = C
        self.ctx = ctx
        self.lib = _lib.lib()
        self.P, self.me = ctx.world, ctx.rank
        self.hbytes = int(self.lib.vr_peer_handle_bytes())
        self.side = torch.cuda.Stream()
        self.epoch = {}
        self._arrays = {}                # flag-address tuples -> ctypes arrays
        self.bufs = {}                   # name -> (local ptr, [ptr on rank q], nbytes)
        self._opened = []
        self.flags, self.flags_remote = self._symmetric(self.P * self.NCH * 8)

    # ---- symmetric buffers --------------------------------------------------------
    def _symmetric(self, nbytes: int):
        C = self.C
        ptr = C.c_void_p()
        handle = C.create_string_buffer(self.hbytes)
        _lib.check(self.lib.vr_peer_malloc(int(nbytes), C.byref(ptr), handle), "vr_peer_malloc")
        handles = [None] * self.P
        tdist.all_gather_object(handles, bytes(handle.raw), group=self.ctx.group)
        remote = []
        for q in range(self.P):
            if q == self.me:
                remote.append(ptr.value)
                continue
            rp = C.c_void_p()
            _lib.check(self.lib.vr_peer_open(C.create_string_buffer(handles[q], self.hbytes), C.byref(rp)),
                       "vr_peer_open")
            self._opened.append(rp.value)
            remote.append(rp.value)
        return ptr.value, remote

    def buffer(self, name: str, nbytes: int):
        """(local ptr, per-rank ptrs) of a symmetric buffer of >= nbytes (grown collectively)."""
        cur = self.bufs.get(name)
        if cur is None or cur[2] < nbytes:
            local, remote = self._symmetric(nbytes)
            self.bufs[name] = (local, remote, nbytes)   # the old mapping stays valid until teardown
        return self.bufs[name]

    def tensor(self, name: str, dtype: torch.dtype, numel: int) -> torch.Tensor:
        esz = torch.empty((), dtype=dtype).element_size()
        local, _, _ = self.buffer(name, numel * esz)
        return _view(local, numel * esz, dtype, (numel,))

    def remote_of(self, t: torch.Tensor, q: int) -> int:
        """Address on rank q of the element t[0] of a view into a symmetric buffer."""
        p = t.data_ptr()
        for local, remote, nbytes in self.bufs.values():
            if local <= p < local + nbytes:
                return remote[q] + (p - local)
        raise ValueError("tensor does not live in a symmetric peer buffer")

    def _flag_local(self, src: int, ch: int) -> int:
        return self.flags + (src * self.NCH + ch) * 8

    def _flag_remote(self, q: int, src: int, ch: int) -> int:
        return self.flags_remote[q] + (src * self.NCH + ch) * 8

    def _addr_array(self, addrs):
        key = tuple(addrs)
        arr = self._arrays.get(key)
        if arr is None:
            arr = (self.C.c_void_p * len(key))(*key)
            self._arrays[key] = arr
        return arr

    def signal_many(self, addrs, e: int, st) -> None:
        """Set the (peer) flags `addrs` to epoch e behind the stream's work: one launch."""
        _lib.check(self.lib.vr_peer_signal_many(self._addr_array(addrs), len(addrs), e, st), "vr_peer_signal_many")

    def wait_many(self, addrs, e: int, st) -> None:
        """The stream waits until every local flag in `addrs` reaches epoch e (one batched op)."""
        _lib.check(self.lib.vr_peer_wait_many(self._addr_array(addrs), len(addrs), e, st), "vr_peer_wait_many")

    def _next(self, key: str) -> int:
        e = self.epoch.get(key, 0) + 1
        self.epoch[key] = e
        return e

    def _on_side(self, *tensors):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.side.wait_event(ev)
        for t in tensors:
            t.record_stream(self.side)

    # ---- ghost planes ---------------------------------------------------------------
    def ghosts_post(self, x: torch.Tensor, w: int) -> tuple:
        """Copy-engine ghost exchange of x (..., L1, N2, N3): my first w planes
        into the left neighbour's hi ghost block, my last w planes into the right
        neighbour's lo block (double-buffered by epoch parity)."""
        L1, n2, n3 = x.shape[-3:]
        lead = tuple(x.shape[:-3])
        ncomp = int(np.prod(lead)) if lead else 1
        plane = n2 * n3 * x.element_size()
        blk = ncomp * w * plane
        xs = x.reshape((ncomp, L1, n2, n3))
        if not xs.is_contiguous():
            xs = xs.contiguous()
        local, remote, cap = self.buffer("ghost", 4 * blk)
        cap = (cap // 4) & ~255
        e = self._next("ghost")
        par = e % 2
        off_lo, off_hi = (2 * par) * cap, (2 * par + 1) * cap
        left, right = self.ctx.left, self.ctx.right
        # one SM copy kernel on the current stream (ordered behind the producer
        # of x), then the two completion flags
        st = _lib.stream()
        _lib.check(self.lib.vr_peer_halo_put(xs.data_ptr(), ncomp, L1, n2 * n3, w, remote[left] + off_hi,
                                             remote[right] + off_lo, st), "vr_peer_halo_put")
        self.signal_many((self._flag_remote(left, self.me, self.GHOST_HI),
                          self._flag_remote(right, self.me, self.GHOST_LO)), e, st)
        shape = lead + (w, n2, n3)
        lo = _view(local + off_lo, blk, x.dtype, shape)
        hi = _view(local + off_hi, blk, x.dtype, shape)
        work = _PeerWork(self, [(self._flag_local(left, self.GHOST_LO), e),
                                (self._flag_local(right, self.GHOST_HI), e)])
        return lo, hi, [work]

    # ---- all-to-all ------------------------------------------------------------------
    def alltoall_post(self, out: torch.Tensor, inp: torch.Tensor) -> _PeerWork:
        """Equal-split all-to-all of flat views: block q of `inp` lands in rank
        q's `out` (a symmetric buffer view) at block `me`."""
        nb = inp.numel() * inp.element_size() // self.P
        self._on_side(inp)
        st = self.side.cuda_stream
        e = self._next("a2a")
        base = inp.data_ptr()
        for k in range(self.P):
            q = (self.me + k) % self.P                     # stagger the destinations
            _lib.check(self.lib.vr_peer_copy(self.remote_of(out, q) + self.me * nb, base + q * nb, nb, st),
                       "vr_peer_copy")
        self.signal_many([self._flag_remote(q, self.me, self.A2A) for q in range(self.P)], e, st)
        return _PeerWork(self, [(self._flag_local(q, self.A2A), e) for q in range(self.P)])


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
        self._mesh = None

    @property
    def mesh(self):
        """PeerMesh for NCCL (GPU) groups with > 1 rank unless VR_PEER=0; None otherwise."""
        if self._mesh is None and self.world > 1 and os.environ.get("VR_PEER", "1") != "0" \
                and tdist.get_backend(self.group) == "nccl":
            self._mesh = PeerMesh(self)
        return self._mesh

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
        if self.mesh is not None:
            return self.mesh.ghosts_post(x, w)
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
        if self.mesh is not None and self._symmetric_view(out):
            with _lib.timed("dist.alltoall"):
                work = self.mesh.alltoall_post(out, inp)
                if async_op:
                    return work
                work.wait()
            return None
        if async_op:
            return tdist.all_to_all_single(out, inp, group=self.group, async_op=True)
        with _lib.timed("dist.alltoall"):
            tdist.all_to_all_single(out, inp, group=self.group)
        return None

    def _symmetric_view(self, t: torch.Tensor) -> bool:
        try:
            self.mesh.remote_of(t, self.rank)
            return True
        except ValueError:
            return False

    def buffer(self, name: str, dtype: torch.dtype, numel: int) -> torch.Tensor:
        """A receive buffer other ranks can write into (symmetric peer buffer
        when the mesh is active, else a plain device tensor)."""
        if self.mesh is not None:
            return self.mesh.tensor(name, dtype, numel)
        return torch.empty(numel, dtype=dtype, device=_lib.device())

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
