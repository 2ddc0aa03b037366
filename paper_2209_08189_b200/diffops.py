"""Differential and spectral regularization operators (drop-in for
/root/reference/pkg/src/velreg/diffops.py).

FD8 gradient / divergence run the fp32 stencil kernel (bit-identical to the
reference's numpy evaluation for float32 input).  A, its shifted inverse, the
Leray blend K and the H1 energy run on the hand-written FFT engine
(csrc/spectral.cu); `SpectralWorkspace` owns its plan (device buffers and
twiddle tables) and, like the reference's, must not be shared by concurrent
callers.
"""
from __future__ import annotations

import os
import weakref
from dataclasses import dataclass

import ctypes as C
import numpy as np
import torch

from . import _lib
from .errors import GridError
from .grid import Grid, ScalarField, VectorField, TWO_PI

FD8_COEFFS = (4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0)   # diffops.py:20
FD8_MIN_DIM = 9


def _destroy_plan(handle):
    lib = _lib.load_library()
    lib.vr_spec_plan_destroy(handle)


class SpectralWorkspace:
    """Plan + scratch spectra for one grid (diffops.py:24-55).  The wavenumber
    tables of the reference are exposed lazily as host arrays for inspection;
    the device kernels regenerate wavenumbers from indices."""

    def __init__(self, grid: Grid):
        self.grid = grid
        lib = _lib.lib()
        handle = C.c_void_p()
        _lib.check(lib.vr_spec_plan_create(_lib.dims_arg(grid.dims), C.byref(handle)), "vr_spec_plan_create")
        self._plan = handle
        self._finalizer = weakref.finalize(self, _destroy_plan, handle)
        self.device = torch.cuda.current_device()

    @property
    def plan(self):
        return self._plan

    # host-side views of the reference's tables (diffops.py:34-49)
    @property
    def k(self):
        n1, n2, n3 = self.grid.dims
        return ((np.fft.fftfreq(n1) * n1).reshape(n1, 1, 1), (np.fft.fftfreq(n2) * n2).reshape(1, n2, 1),
                np.arange(n3 // 2 + 1, dtype=np.float64).reshape(1, 1, n3 // 2 + 1))

    @property
    def ksq(self):
        k1, k2, k3 = self.k
        return k1 ** 2 + k2 ** 2 + k3 ** 2

    @property
    def mode_multiplicity(self):
        n3 = self.grid.dims[2]
        mult = np.full(self.ksq.shape, 2.0)
        mult[:, :, 0] = 1.0
        if n3 % 2 == 0:
            mult[:, :, -1] = 1.0
        return mult

    def apply(self, kind: int, x: torch.Tensor, out: torch.Tensor | None = None, add: torch.Tensor | None = None,
              beta_v: float = 0.0, beta_w: float = 0.0, shift: float = 0.0, sigma: float = 0.0,
              alpha: float = 1.0) -> torch.Tensor:
        ncomp = 3 if x.dim() == 4 else 1
        if out is None:
            out = torch.empty_like(x)
        rc = _lib.lib().vr_spec_apply(self._plan, int(kind), x.data_ptr(), ncomp, float(beta_v), float(beta_w),
                                      float(shift), float(sigma), float(alpha), _lib.ptr(add), out.data_ptr(),
                                      _lib.stream())
        _lib.check(rc, "vr_spec_apply")
        return out

    def h1_energy(self, f: torch.Tensor) -> float:
        out = _lib.out_buf(1)
        _lib.check(_lib.lib().vr_h1_energy(self._plan, f.data_ptr(), out.data_ptr(), _lib.stream()),
                   "vr_h1_energy")
        return float(out.cpu()[0])


# distributed separable A: x2 pass fused with the final (after the x1
# exchange, VR_SEP_A_FUSED=1) or overlapping the first exchange (0)
_SEP_A_FUSED_FINAL = os.environ.get("VR_SEP_A_FUSED", "1") != "0"


class DistSpectralWorkspace:
    """Spectral operators on x1 slabs (see csrc/spectral.cu "Distributed"):
    local x3/x2 passes + pack -> one all-to-all per component -> x1 pass with
    the symbol on complete x1 lines -> all-to-all back -> local x2/x3 inverse."""

    def __init__(self, grid: Grid, ctx):
        self.grid = grid
        self.ctx = ctx
        lib = _lib.lib()
        n1, n2, n3 = grid.dims
        self.n3h = n3 // 2 + 1
        self._pl = C.c_void_p()
        self._px = C.c_void_p()
        _lib.check(lib.vr_spec_plan_create(_lib.dims_arg(ctx.local_dims), C.byref(self._pl)), "vr_spec_plan_create")
        self._fin1 = weakref.finalize(self, _destroy_plan, self._pl)
        _lib.check(lib.vr_spec_plan_create(_lib.dims_arg((n1, ctx.L2, n3)), C.byref(self._px)), "vr_spec_plan_create")
        self._fin2 = weakref.finalize(self, _destroy_plan, self._px)
        # power-of-two sizes run the fast engines (and the fused peer
        # transposes); any other even size (e.g. the CLARITY shape) the generic
        # mixed-radix engine, whose forward half is always f64
        self.generic = not (lib.vr_spec_plan_is_fast(self._pl) and lib.vr_spec_plan_is_fast(self._px))
        nc = 3 * ctx.L1 * n2 * self.n3h          # complex elements per 3-component slab spectrum
        self._nc = nc
        self._send = self._xout = None   # staging of the packed (non-fused) path, allocated on first use
        self.recv = ctx.buffer(f"spec_recv_{n1}x{n2}x{n3}", torch.float64, 2 * nc)     # peers write here
        self.irecv = ctx.buffer(f"spec_irecv_{n1}x{n2}x{n3}", torch.float32, 2 * nc)
        self.per_comp = ctx.L1 * n2 * self.n3h   # complex elements per component
        self.device = torch.cuda.current_device()
        # transposes fused into the passes over peer memory (csrc/spectral.cu
        # vr_dspec_*_peer) when the peer mesh is active and the shapes allow
        P = ctx.world
        self.peer = (ctx.mesh is not None and not self.generic and n2 == 256 and 1 < P <= 8 and (P & (P - 1)) == 0
                     and os.environ.get("VR_PEER_FUSED", "1") != "0")
        # A through the separable line engine with the transposes as pass
        # outputs (csrc/spectral.cu vr_dspec_a_*): f32 rows over NVLink instead
        # of f64 half spectra, no 3-D transform
        self.sep_a = (ctx.mesh is not None and 1 < P <= 8 and os.environ.get("VR_DIST_SEP_A", "1") != "0"
                      and bool(lib.vr_dspec_a_ok(self._pl, self._px, P)))
        self._dst_cache = {}

    @property
    def send(self) -> torch.Tensor:
        if self._send is None:
            self._send = torch.empty(2 * self._nc, dtype=torch.float64, device=_lib.device())
        return self._send

    @property
    def xout(self) -> torch.Tensor:
        if self._xout is None:
            self._xout = torch.empty(2 * self._nc, dtype=torch.float32, device=_lib.device())
        return self._xout

    # ---- peer (fused-transpose) path ---------------------------------------------
    def _dst(self, view: torch.Tensor):
        """Host array of the P device addresses of `view` (a symmetric buffer region)."""
        key = view.data_ptr()
        arr = self._dst_cache.get(key)
        if arr is None:
            mesh = self.ctx.mesh
            arr = (C.c_void_p * self.ctx.world)(*[mesh.remote_of(view, q) for q in range(self.ctx.world)])
            self._dst_cache[key] = arr
        return arr

    def _signal(self) -> int:
        mesh, st = self.ctx.mesh, _lib.stream()
        e = mesh._next("a2a")
        mesh.signal_many([mesh._flag_remote(q, self.ctx.rank, mesh.A2A) for q in range(self.ctx.world)], e, st)
        return e

    def _wait(self, e: int) -> None:
        mesh, st = self.ctx.mesh, _lib.stream()
        mesh.wait_many([mesh._flag_local(q, mesh.A2A) for q in range(self.ctx.world)], e, st)

    def _regions(self, c: int, ncomp: int, f64: bool):
        """(recv, irecv) views of component c's regions (or all ncomp from 0)."""
        rv = self.recv if f64 else self.recv.view(torch.float32)   # 2 reals per complex either way
        off, n = c * self.per_comp * 2, self.per_comp * 2 * ncomp
        return rv[off:off + n], self.irecv[off:off + n]

    def _apply_peer(self, kind, x, out, add, f64, beta_v, beta_w, shift, sigma, alpha, comps) -> bool:
        lib, st, ctx = _lib.lib(), _lib.stream(), self.ctx
        P, me = ctx.world, ctx.rank
        n1, n2, n3 = self.grid.dims
        nvox = x[0].numel() if x.dim() == 4 else x.numel()
        groups = [(c, 1) for c in range(3)] if comps == "pipelined" else [(0, 3 if x.dim() == 4 else 1)]
        ef, ei = [], []
        with _lib.timed("dist.spectral"):
            for c, nc in groups:
                rv, _ = self._regions(c, nc, f64)
                rc = lib.vr_dspec_forward_peer(self._pl, x.data_ptr() + 4 * c * nvox, nc, int(f64), P, me,
                                               self._dst(rv), st)
                if rc == -5:
                    if ef:
                        raise RuntimeError("fused-transpose path became unsupported mid-operator")
                    self.peer = False
                    return False
                _lib.check(rc, "vr_dspec_forward_peer")
                ef.append(self._signal())
            for (c, nc), e in zip(groups, ef):
                rv, iv = self._regions(c, nc, f64)
                self._wait(e)
                _lib.check(lib.vr_dspec_xpass_peer(self._px, int(kind), nc, int(f64), float(beta_v), float(beta_w),
                                                   float(shift), float(sigma), float(alpha), n1 * n2 * n3,
                                                   ctx.rank * ctx.L2, n2, ctx.L1, rv.data_ptr(), P, me,
                                                   self._dst(iv), st), "vr_dspec_xpass_peer")
                ei.append(self._signal())
            for (c, nc), e in zip(groups, ei):
                _, iv = self._regions(c, nc, f64)
                self._wait(e)
                a = None if add is None else add.data_ptr() + 4 * c * nvox
                _lib.check(lib.vr_dspec_inverse_peer(self._pl, iv.data_ptr(), nc, P, a, out.data_ptr() + 4 * c * nvox,
                                                     st), "vr_dspec_inverse_peer")
        return True

    def _apply_sep_a(self, x, out, add, alpha) -> None:
        """out = alpha A x (+ add) on the slab: local x3 / x2 line passes, the
        slab rows stored into the x2-chunk owners' block buffers by the x3
        pass, the x1 pass on this rank's block storing D11 x back to the slab
        owners, then alpha (acc + back) (+ add) -- the single-domain
        operator's arithmetic (spectral_d2.cuh)."""
        lib, st, ctx = _lib.lib(), _lib.stream(), self.ctx
        P, me = ctx.world, ctx.rank
        ncomp = 3 if x.dim() == 4 else 1
        n = ncomp * (x[0].numel() if ncomp == 3 else x.numel())
        blk = self.recv.view(torch.float32)[:n]     # [c][N1][L2][N3] -- peers write here
        back = self.irecv[:n]                       # [c][L1][N2][N3]
        fused = _SEP_A_FUSED_FINAL
        with _lib.timed("dist.spectral"):
            _lib.check(lib.vr_dspec_a_rows(self._pl, self._px, x.data_ptr(), ncomp, P, me, self._dst(blk), st),
                       "vr_dspec_a_rows")
            e1 = self._signal()
            if not fused:   # the local x2 pass covers the exchange
                _lib.check(lib.vr_dspec_a_x2(self._pl, x.data_ptr(), ncomp, st), "vr_dspec_a_x2")
            self._wait(e1)
            _lib.check(lib.vr_dspec_a_x1_peer(self._pl, self._px, blk.data_ptr(), ncomp, P, me, self._dst(back), st),
                       "vr_dspec_a_x1_peer")
            self._wait(self._signal())
            if fused:
                _lib.check(lib.vr_dspec_a_x2_final(self._pl, x.data_ptr(), back.data_ptr(), ncomp, float(alpha),
                                                   _lib.ptr(add), out.data_ptr(), st), "vr_dspec_a_x2_final")
            else:
                _lib.check(lib.vr_dspec_a_final(self._pl, back.data_ptr(), ncomp, float(alpha), _lib.ptr(add),
                                                out.data_ptr(), st), "vr_dspec_a_final")

    def _exchange(self, dst: torch.Tensor, src: torch.Tensor, ncomp: int, cplx_words: int) -> None:
        """One all-to-all for all components: blocks are [rank][component][...]."""
        m = self.per_comp * cplx_words * ncomp
        self.ctx.alltoall(dst[:m], src[:m])

    def apply(self, kind: int, x: torch.Tensor, out: torch.Tensor | None = None, add: torch.Tensor | None = None,
              beta_v: float = 0.0, beta_w: float = 0.0, shift: float = 0.0, sigma: float = 0.0,
              alpha: float = 1.0) -> torch.Tensor:
        lib = _lib.lib()
        st = _lib.stream()
        ncomp = 3 if x.dim() == 4 else 1
        if out is None:
            out = torch.empty_like(x)
        f64 = kind in (_lib.SPEC_A, _lib.SPEC_A2) or self.generic
        P = self.ctx.world
        if kind == _lib.SPEC_A and self.sep_a:
            self._apply_sep_a(x, out, add, alpha)
            return out
        if self.peer:
            comps = "pipelined" if (ncomp == 3 and kind != _lib.SPEC_K) else "fused"
            if self._apply_peer(kind, x, out, add, f64, beta_v, beta_w, shift, sigma, alpha, comps):
                return out
        if ncomp == 3 and kind != _lib.SPEC_K and P > 1:
            return self._apply_pipelined(kind, x, out, add, f64, beta_v, beta_w, shift, sigma, alpha)
        _lib.check(lib.vr_dspec_forward(self._pl, x.data_ptr(), ncomp, int(f64), P, self.send.data_ptr(), st),
                   "vr_dspec_forward")
        snd = self.send if f64 else self.send.view(torch.float32)
        rcv = self.recv if f64 else self.recv.view(torch.float32)
        self._exchange(rcv, snd, ncomp, 2)
        n1, n2, n3 = self.grid.dims
        _lib.check(lib.vr_dspec_xpass(self._px, int(kind), ncomp, int(f64), float(beta_v), float(beta_w),
                                      float(shift), float(sigma), float(alpha), n1 * n2 * n3,
                                      self.ctx.rank * self.ctx.L2, n2, self.ctx.L1, self.recv.data_ptr(),
                                      self.xout.data_ptr(), st), "vr_dspec_xpass")
        self._exchange(self.irecv, self.xout, ncomp, 2)
        _lib.check(lib.vr_dspec_inverse(self._pl, self.irecv.data_ptr(), ncomp, P, _lib.ptr(add), out.data_ptr(),
                                        st), "vr_dspec_inverse")
        return out

    def _apply_pipelined(self, kind, x, out, add, f64, beta_v, beta_w, shift, sigma, alpha) -> torch.Tensor:
        """Component-wise software pipeline: the all-to-all of one component is in
        flight while the local passes / x1 pass of another run (K couples the
        components inside the x1 pass and uses the fused path instead)."""
        lib = _lib.lib()
        st = _lib.stream()
        P = self.ctx.world
        n1, n2, n3 = self.grid.dims
        nvox = x[0].numel()
        esz = 16 if f64 else 8
        blk = self.per_comp * esz                       # bytes of one component's spectrum
        snd = self.send if f64 else self.send.view(torch.float32)
        rcv = self.recv if f64 else self.recv.view(torch.float32)
        words = blk // snd.element_size()
        xwords = self.per_comp * 2                      # complex64 words per component

        def fwd(c):
            _lib.check(lib.vr_dspec_forward(self._pl, x.data_ptr() + 4 * c * nvox, 1, int(f64), P,
                                            self.send.data_ptr() + c * blk, st), "vr_dspec_forward")
            return self.ctx.alltoall(rcv[c * words:(c + 1) * words], snd[c * words:(c + 1) * words], async_op=True)

        def xpass(c):
            _lib.check(lib.vr_dspec_xpass(self._px, int(kind), 1, int(f64), float(beta_v), float(beta_w), float(shift),
                                          float(sigma), float(alpha), n1 * n2 * n3, self.ctx.rank * self.ctx.L2, n2,
                                          self.ctx.L1, self.recv.data_ptr() + c * blk,
                                          self.xout.data_ptr() + 8 * c * self.per_comp, st), "vr_dspec_xpass")
            return self.ctx.alltoall(self.irecv[c * xwords:(c + 1) * xwords], self.xout[c * xwords:(c + 1) * xwords],
                                     async_op=True)

        def inv(c):
            a = None if add is None else add.data_ptr() + 4 * c * nvox
            _lib.check(lib.vr_dspec_inverse(self._pl, self.irecv.data_ptr() + 8 * c * self.per_comp, 1, P, a,
                                            out.data_ptr() + 4 * c * nvox, st), "vr_dspec_inverse")

        with _lib.timed("dist.spectral"):
            a0 = fwd(0)
            a1 = fwd(1)
            a0.wait()
            b0 = xpass(0)
            a2 = fwd(2)
            a1.wait()
            b1 = xpass(1)
            b0.wait()
            inv(0)
            a2.wait()
            b2 = xpass(2)
            b1.wait()
            inv(1)
            b2.wait()
            inv(2)
        return out

    def h1_energy(self, f: torch.Tensor) -> float:
        lib = _lib.lib()
        st = _lib.stream()
        P = self.ctx.world
        done = False
        if self.peer:
            rv, _ = self._regions(0, 1, True)
            rc = lib.vr_dspec_forward_peer(self._pl, f.data_ptr(), 1, 1, P, self.ctx.rank, self._dst(rv), st)
            if rc == 0:
                self._wait(self._signal())
                done = True
            elif rc != -5:
                _lib.check(rc, "vr_dspec_forward_peer")
        if not done:
            _lib.check(lib.vr_dspec_forward(self._pl, f.data_ptr(), 1, 1, P, self.send.data_ptr(), st),
                       "vr_dspec_forward")
            self._exchange(self.recv, self.send, 1, 2)
        n = float(np.prod(self.grid.dims))
        out = _lib.out_buf(1)
        _lib.check(lib.vr_dspec_h1_partial(self._px, self.recv.data_ptr(), self.ctx.rank * self.ctx.L2,
                                           self.grid.dims[1], self.ctx.L1, TWO_PI ** 3 / (n * n), out.data_ptr(), st),
                   "vr_dspec_h1_partial")
        self.ctx.allreduce_(out, "sum")
        return float(out.cpu()[0])


_ws_cache: dict = {}


def workspace_for(grid: Grid):
    from . import dist
    ctx = dist.for_grid(grid.dims)
    key = (grid.dims, torch.cuda.current_device(), id(ctx) if ctx is not None else None)
    ws = _ws_cache.get(key)
    if ws is None:
        ws = DistSpectralWorkspace(grid, ctx) if ctx is not None else SpectralWorkspace(grid)
        _ws_cache[key] = ws
    return ws


@dataclass
class RegOperators:
    """Regularization weights plus the spectral workspace they act through
    (diffops.py:58-75)."""

    beta_v: float
    beta_w: float
    workspace: SpectralWorkspace = None

    def __post_init__(self):
        if not self.beta_v > 0:
            raise ValueError(f"beta_v must be positive, got {self.beta_v}")
        if self.beta_w < 0:
            raise ValueError(f"beta_w must be non-negative, got {self.beta_w}")

    @classmethod
    def for_grid(cls, grid: Grid, beta_v: float, beta_w: float) -> "RegOperators":
        return cls(beta_v, beta_w, workspace_for(grid))


def _require_fd8(grid: Grid) -> None:
    if min(grid.dims) < FD8_MIN_DIM:
        raise GridError(f"8th-order stencil needs dims >= {FD8_MIN_DIM}, got {grid.dims}")


# ---- FD8 (diffops.py:84-105) -------------------------------------------------
def fd8_gradient_t(f: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    from . import dist
    dims = tuple(f.shape[-3:])
    if out is None:
        out = torch.empty((3,) + dims, dtype=torch.float32, device=f.device)
    ctx = dist.for_shape(f.shape)
    if ctx is not None:   # x1 slab: 4 ghost planes from the neighbours
        lo, hi = ctx.ghosts(f, 4)
        _lib.check(_lib.lib().vr_fd8_grad_slab(f.data_ptr(), lo.data_ptr(), hi.data_ptr(), _lib.dims_arg(dims),
                                               ctx.dims[0], out.data_ptr(), _lib.stream()), "vr_fd8_grad_slab")
        return out
    _lib.check(_lib.lib().vr_fd8_grad(f.data_ptr(), _lib.dims_arg(dims), out.data_ptr(), _lib.stream()),
               "vr_fd8_grad")
    return out


def fd8_divergence_t(v: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    from . import dist
    dims = tuple(v.shape[-3:])
    if out is None:
        out = torch.empty(dims, dtype=torch.float32, device=v.device)
    ctx = dist.for_shape(v.shape)
    if ctx is not None:   # only v1 is differentiated along x1
        lo, hi = ctx.ghosts(v[0], 4)
        _lib.check(_lib.lib().vr_fd8_div_slab(v.data_ptr(), lo.data_ptr(), hi.data_ptr(), _lib.dims_arg(dims),
                                              ctx.dims[0], out.data_ptr(), _lib.stream()), "vr_fd8_div_slab")
        return out
    _lib.check(_lib.lib().vr_fd8_div(v.data_ptr(), _lib.dims_arg(dims), out.data_ptr(), _lib.stream()),
               "vr_fd8_div")
    return out


def fd8_gradient(f: ScalarField) -> VectorField:
    _require_fd8(f.grid)
    return VectorField(f.grid, fd8_gradient_t(f.values))


def fd8_divergence(v: VectorField) -> ScalarField:
    _require_fd8(v.grid)
    return ScalarField(v.grid, fd8_divergence_t(v.data))


# ---- spectral operators (diffops.py:108-154) -------------------------------------
def apply_A(v: VectorField, ops: RegOperators) -> VectorField:
    """Negative vector Laplacian (symbol |k|^2); kills constants."""
    return VectorField(v.grid, ops.workspace.apply(_lib.SPEC_A, v.data))


def apply_inv_shifted_A(v: VectorField, ops: RegOperators, shift: float) -> VectorField:
    """Spectral inverse of (beta_v*A + shift*I); preconditioner support."""
    if not shift > 0:
        raise ValueError(f"shift must be positive, got {shift}")
    return VectorField(v.grid, ops.workspace.apply(_lib.SPEC_INVSHIFT, v.data, beta_v=ops.beta_v, shift=shift))


def apply_K(g: VectorField, ops: RegOperators) -> VectorField:
    """Blend toward the Leray projection (diffops.py:129-146); beta_w = 0 is the
    identity (a copy, as in the reference)."""
    if ops.beta_w == 0.0:
        return g.copy()
    return VectorField(g.grid, ops.workspace.apply(_lib.SPEC_K, g.data, beta_v=ops.beta_v, beta_w=ops.beta_w))


def h1_energy(f: ScalarField, ws: SpectralWorkspace) -> float:
    """Spectral H1 norm squared: integral of f^2 + |grad f|^2 over the box."""
    return ws.h1_energy(f.values)


# ---- north-star extras without a reference counterpart (flags default off) -------
def gaussian_smooth(v, ws: SpectralWorkspace, sigma: float):
    """Spectral Gaussian smoothing exp(-sigma^2 |k|^2 / 2) (sigma in voxels of the
    unit-wavenumber lattice); pinned analytically by eigenfunction tests."""
    data = v.data if isinstance(v, VectorField) else v.values
    out = ws.apply(_lib.SPEC_GAUSS, data, sigma=sigma)
    return VectorField(v.grid, out) if isinstance(v, VectorField) else ScalarField(v.grid, out)


def apply_A2(v: VectorField, ops: RegOperators) -> VectorField:
    """H2-seminorm operator (bi-Laplacian, symbol |k|^4)."""
    return VectorField(v.grid, ops.workspace.apply(_lib.SPEC_A2, v.data))


def apply_inv_shifted_A2(v: VectorField, ops: RegOperators, shift: float) -> VectorField:
    if not shift > 0:
        raise ValueError(f"shift must be positive, got {shift}")
    return VectorField(v.grid, ops.workspace.apply(_lib.SPEC_INVSHIFT2, v.data, beta_v=ops.beta_v, shift=shift))
