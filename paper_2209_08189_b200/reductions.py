"""Host wrappers of the deterministic f64 reductions and fused vector updates
(csrc/reduce.cu).  Each reduction is one device pass plus a single-CTA fold;
results come back to the host in one small copy (the only host sync points of
the solver, matching where the reference needs a Python float)."""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from . import dist as _dist


def _n(t: torch.Tensor) -> int:
    return t.numel()


def _ctx(t: torch.Tensor):
    """The slab context `t` belongs to (dist.for_shape), or None."""
    return _dist.for_shape(t.shape)


def dots_dev(pairs) -> torch.Tensor:
    """[sum(a*b) for a, b in pairs] as a device f64 vector (summed across ranks
    on the device under a slab decomposition) -- no host read."""
    lib = _lib.lib()
    k = len(pairs)
    assert 1 <= k <= 4
    n = _n(pairs[0][0])
    out = _lib.out_buf(k)
    a = _lib.ptr_array([p[0] for p in pairs])
    b = _lib.ptr_array([p[1] for p in pairs])
    _lib.check(lib.vr_dots(k, a, b, n, _lib.scratch().data_ptr(), out.data_ptr(), _lib.stream()), "vr_dots")
    ctx = _ctx(pairs[0][0])
    if ctx is not None:
        ctx.allreduce_(out, "sum")
    return out


def host(*devs: torch.Tensor) -> list:
    """One device->host read for several device result vectors (the solver's
    sync points), then the deferred non-finite checks; returns numpy arrays."""
    flat = torch.cat([d.reshape(-1) for d in devs]).cpu().numpy()
    _lib.run_deferred()
    res, o = [], 0
    for d in devs:
        res.append(flat[o:o + d.numel()])
        o += d.numel()
    return res


def dots(pairs) -> np.ndarray:
    """[sum(a*b) for a, b in pairs] (<= 4 pairs, same length) -> float64 array."""
    return host(dots_dev(pairs))[0]


def dot(a: torch.Tensor, b: torch.Tensor) -> float:
    return float(dots([(a, b)])[0])


def sqdiff_dev(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor | None = None) -> torch.Tensor:
    lib = _lib.lib()
    out = _lib.out_buf(2)
    _lib.check(lib.vr_sqdiff(a.data_ptr(), b.data_ptr(), _lib.ptr(c), _n(a), _lib.scratch().data_ptr(),
                             out.data_ptr(), _lib.stream()), "vr_sqdiff")
    ctx = _ctx(a)
    if ctx is not None:
        ctx.allreduce_(out, "sum")
    return out


def sqdiff(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor | None = None) -> np.ndarray:
    return host(sqdiff_dev(a, b, c))[0]


def minmax(a: torch.Tensor, b: torch.Tensor | None = None) -> np.ndarray:
    lib = _lib.lib()
    out = _lib.out_buf(4)
    _lib.check(lib.vr_minmax(a.data_ptr(), _lib.ptr(b), _n(a), _lib.scratch().data_ptr(), out.data_ptr(),
                             _lib.stream()), "vr_minmax")
    ctx = _ctx(a)
    if ctx is not None:
        out[0::2].neg_()
        ctx.allreduce_(out, "max")
        out[0::2].neg_()
    return out.cpu().numpy()


def local_absmax(x: torch.Tensor) -> float:
    """max |x| over this rank's data (host-side sizing of ghost widths)."""
    mn, mx, _, _ = minmax_local(x)
    return max(abs(mn), abs(mx))


def minmax_local(a: torch.Tensor, b: torch.Tensor | None = None) -> np.ndarray:
    """(min a, max a, min b, max b) over this rank's data only (no allreduce)."""
    lib = _lib.lib()
    out = _lib.out_buf(4)
    _lib.check(lib.vr_minmax(a.data_ptr(), _lib.ptr(b), _n(a), _lib.scratch().data_ptr(), out.data_ptr(),
                             _lib.stream()), "vr_minmax")
    return out.cpu().numpy()


def vecstats_dev(v: torch.Tensor) -> torch.Tensor:
    """device f64 [-, max |v|^2, #non-finite, #non-zero] (no host read)"""
    lib = _lib.lib()
    out = _lib.out_buf(4)
    _lib.check(lib.vr_vecstats(v.data_ptr(), _n(v) // 3, _lib.scratch().data_ptr(), out.data_ptr(),
                               _lib.stream()), "vr_vecstats")
    ctx = _ctx(v)
    if ctx is not None:
        ctx.allreduce_(out[1:2], "max")
        ctx.allreduce_(out[2:4], "sum")
    return out


def vecstats(v: torch.Tensor) -> tuple:
    """(max_x |v(x)|^2, number of non-finite entries, number of non-zero entries)"""
    o = vecstats_dev(v).cpu().numpy()
    return float(o[1]), int(o[2]), int(o[3])


def axpby(a: float, x: torch.Tensor, b: float = 0.0, y: torch.Tensor | None = None,
          out: torch.Tensor | None = None) -> torch.Tensor:
    """out = a*x + b*y (f64 arithmetic, f32 storage)."""
    if out is None:
        out = torch.empty_like(x)
    _lib.check(_lib.lib().vr_axpby(_n(x), float(a), x.data_ptr(), float(b), _lib.ptr(y), out.data_ptr(),
                                   _lib.stream()), "vr_axpby")
    return out


def pcg_update2(rz_dev: torch.Tensor, php_dev: torch.Tensor, p: torch.Tensor, hp: torch.Tensor, x: torch.Tensor,
                r: torch.Tensor, x_out: torch.Tensor, r_out: torch.Tensor) -> None:
    """x_out = x + alpha p, r_out = r - alpha hp with alpha = rz / php formed on the device."""
    _lib.check(_lib.lib().vr_pcg_update2(_n(x), rz_dev.data_ptr(), php_dev.data_ptr(), p.data_ptr(), hp.data_ptr(),
                                         x.data_ptr(), r.data_ptr(), x_out.data_ptr(), r_out.data_ptr(),
                                         _lib.stream()), "vr_pcg_update2")


def pcg_update(alpha: float, p: torch.Tensor, hp: torch.Tensor, x: torch.Tensor, r: torch.Tensor) -> None:
    _lib.check(_lib.lib().vr_pcg_update(_n(x), float(alpha), p.data_ptr(), hp.data_ptr(), x.data_ptr(),
                                        r.data_ptr(), _lib.stream()), "vr_pcg_update")


def fill(out: torch.Tensor, value: float) -> torch.Tensor:
    _lib.check(_lib.lib().vr_fill(_n(out), float(value), out.data_ptr(), _lib.stream()), "vr_fill")
    return out


def label_range(l0: torch.Tensor, l1: torch.Tensor | None = None) -> np.ndarray:
    """(min l0, max l0, min l1, max l1) over the whole decomposed field (one
    device pass, one host read); int32 extremes for an absent / empty map."""
    out = torch.empty(4, dtype=torch.int32, device=l0.device)
    _lib.check(_lib.lib().vr_label_range(l0.data_ptr(), _lib.ptr(l1), _n(l0), out.data_ptr(), _lib.stream()),
               "vr_label_range")
    ctx = _ctx(l0)
    if ctx is not None:
        o = out.to(torch.float64)
        o[0::2].neg_()
        ctx.allreduce_(o, "max")
        o[0::2].neg_()
        return o.cpu().numpy().astype(np.int64)
    return out.cpu().numpy().astype(np.int64)


def label_histogram(l0: torch.Tensor, l1: torch.Tensor, max_id: int | None = None) -> np.ndarray:
    """counts[id] = (|l0==id|, |l1==id|, |l0==id & l1==id|) as exact int64."""
    ctx = _ctx(l0)
    if max_id is None:
        r = label_range(l0, l1)
        max_id = max(int(r[1]), int(r[3]), 0) if l0.numel() else 0
    counts = torch.empty(3 * (max_id + 1), dtype=torch.int64, device=l0.device)
    _lib.check(_lib.lib().vr_label_counts(l0.data_ptr(), l1.data_ptr(), _n(l0), int(max_id), counts.data_ptr(),
                                          _lib.stream()), "vr_label_counts")
    c = counts.cpu().numpy().reshape(max_id + 1, 3)
    if ctx is not None:
        c = np.rint(ctx.allreduce(c.reshape(-1).astype(np.float64), "sum")).astype(np.int64).reshape(max_id + 1, 3)
    return c
