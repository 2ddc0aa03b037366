"""CPU ORACLE -- test infrastructure only.

A functional numpy (+ numba for the scattered gathers) restatement of the
reference algorithm in /root/reference/pkg/src/velreg (velreg 0.1.0; numpy
2.3.5 pocketfft FFTs; numba 0.65.0 gathers).  Every function cites the
reference file:line it restates.

Who may use this module: tests/ (as the parity checker), __graft_entry__.smoke()
and bench.py's cpu_baseline / `--impl reference` leg.  The product package
(paper_2209_08189_b200) never imports it; there is no CPU fallback.

Pinning: tests/test_oracle_golden.py checks this restatement against golden
vectors produced by the LIVE reference (tests/golden/make_golden.py, committed
fixtures), including full Gauss-Newton trajectories.

Conventions: arrays are numpy, C order (N1,N2,N3); vectors (3,N1,N2,N3);
velocity-space arithmetic in float64 like the reference (grid.py:112-114).
"""
from __future__ import annotations

import math

import numpy as np

try:  # numba is a dependency of the reference itself (pkg/pyproject.toml:10)
    from numba import njit, prange
    HAVE_NUMBA = True
except Exception:  # pragma: no cover - fallback keeps the oracle usable
    HAVE_NUMBA = False

    def njit(*a, **k):
        def deco(f):
            return f
        return deco if not (a and callable(a[0])) else a[0]

    prange = range

TWO_PI = 2.0 * np.pi
FD8 = (4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0)   # diffops.py:20


def spacing(dims):
    """grid.py:35-37"""
    return tuple(TWO_PI / n for n in dims)


def lattice(dims) -> np.ndarray:
    """grid.py:53-56: (3, N1, N2, N3) voxel coordinates i*h."""
    ax = [np.arange(n) * (TWO_PI / n) for n in dims]
    return np.stack(np.meshgrid(*ax, indexing="ij"))


# ---------------------------------------------------------------------------
# scattered interpolation -- interp.py:19-128
# ---------------------------------------------------------------------------
@njit(parallel=True, cache=False)
def _lin_kernel(f, q, out):
    n1, n2, n3 = f.shape
    npts = q.shape[1]
    for p in prange(npts):
        b0 = math.floor(q[0, p])
        b1 = math.floor(q[1, p])
        b2 = math.floor(q[2, p])
        t0 = q[0, p] - b0
        t1 = q[1, p] - b1
        t2 = q[2, p] - b2
        ia, ib = int(b0) % n1, (int(b0) + 1) % n1
        ja, jb = int(b1) % n2, (int(b1) + 1) % n2
        ka, kb = int(b2) % n3, (int(b2) + 1) % n3
        lo = (f[ia, ja, ka] * (1.0 - t2) + f[ia, ja, kb] * t2) * (1.0 - t1) \
            + (f[ia, jb, ka] * (1.0 - t2) + f[ia, jb, kb] * t2) * t1
        hi = (f[ib, ja, ka] * (1.0 - t2) + f[ib, ja, kb] * t2) * (1.0 - t1) \
            + (f[ib, jb, ka] * (1.0 - t2) + f[ib, jb, kb] * t2) * t1
        out[p] = lo * (1.0 - t0) + hi * t0


@njit(cache=False, inline="always")
def _lag4(t):
    # interp.py:61-72 (Lagrange cubic on offsets -1, 0, 1, 2)
    return (-t * (t - 1.0) * (t - 2.0) / 6.0, (t * t - 1.0) * (t - 2.0) / 2.0,
            -t * (t + 1.0) * (t - 2.0) / 2.0, t * (t * t - 1.0) / 6.0)


@njit(parallel=True, cache=False)
def _cub_kernel(f, q, out):
    n1, n2, n3 = f.shape
    npts = q.shape[1]
    for p in prange(npts):
        b0 = int(math.floor(q[0, p]))
        b1 = int(math.floor(q[1, p]))
        b2 = int(math.floor(q[2, p]))
        wx = _lag4(q[0, p] - b0)
        wy = _lag4(q[1, p] - b1)
        wz = _lag4(q[2, p] - b2)
        k0, k1, k2, k3 = (b2 - 1) % n3, b2 % n3, (b2 + 1) % n3, (b2 + 2) % n3
        acc = 0.0
        for a in range(4):
            ia = (b0 - 1 + a) % n1
            sa = 0.0
            for c in range(4):
                jc = (b1 - 1 + c) % n2
                row = f[ia, jc]
                sa += wy[c] * (wz[0] * row[k0] + wz[1] * row[k1] + wz[2] * row[k2] + wz[3] * row[k3])
            acc += wx[a] * sa
        out[p] = acc


def interp(values: np.ndarray, points: np.ndarray, order: str) -> np.ndarray:
    """interp.py:112-128: periodic interpolant of `values` at radian `points`
    (3, ...); f64 arithmetic, result cast to values.dtype."""
    dims = values.shape
    h = spacing(dims)
    q = np.empty((3, points[0].size))
    for a in range(3):
        q[a] = np.asarray(points[a], dtype=np.float64).ravel() / h[a]   # interp.py:23-25
    out = np.empty(q.shape[1])
    f = np.ascontiguousarray(values, dtype=np.float64)
    if order == "linear":
        _lin_kernel(f, q, out)
    elif order == "cubic":
        _cub_kernel(f, q, out)
    else:
        raise ValueError(order)
    return out.reshape(points.shape[1:]).astype(values.dtype, copy=False)


# ---------------------------------------------------------------------------
# FD8 -- diffops.py:84-105 (periodic shifts via index arrays)
# ---------------------------------------------------------------------------
def _shift(f: np.ndarray, axis: int, o: int) -> np.ndarray:
    """g[i] = f[i + o] with periodic wrap along `axis`."""
    n = f.shape[axis]
    idx = (np.arange(n) + o) % n
    return np.take(f, idx, axis=axis)


def d_axis(f: np.ndarray, axis: int) -> np.ndarray:
    h = spacing(f.shape)[axis]
    out = np.zeros_like(f)
    for o, c in enumerate(FD8, start=1):
        out += c * (_shift(f, axis, o) - _shift(f, axis, -o))
    out /= h
    return out


def grad(f: np.ndarray) -> np.ndarray:
    return np.stack([d_axis(f, a) for a in range(3)])


def div(v: np.ndarray) -> np.ndarray:
    out = d_axis(v[0], 0)
    out += d_axis(v[1], 1)
    out += d_axis(v[2], 2)
    return out


# ---------------------------------------------------------------------------
# spectral -- diffops.py:24-55, 108-154 (numpy pocketfft, like the reference)
# ---------------------------------------------------------------------------
def wavenumbers(dims):
    n1, n2, n3 = dims
    k1 = (np.fft.fftfreq(n1) * n1).reshape(n1, 1, 1)
    k2 = (np.fft.fftfreq(n2) * n2).reshape(1, n2, 1)
    k3 = np.arange(n3 // 2 + 1, dtype=np.float64).reshape(1, 1, n3 // 2 + 1)
    return k1, k2, k3, k1 ** 2 + k2 ** 2 + k3 ** 2


def _per_comp(v: np.ndarray, mult: np.ndarray) -> np.ndarray:
    dims = v.shape[1:]
    return np.stack([np.fft.irfftn(mult * np.fft.rfftn(v[i]), s=dims, axes=(0, 1, 2)).astype(v.dtype) for i in range(3)])


def op_A(v):
    return _per_comp(v, wavenumbers(v.shape[1:])[3])


def op_inv_shifted(v, beta_v, shift):
    return _per_comp(v, 1.0 / (beta_v * wavenumbers(v.shape[1:])[3] + shift))


def op_K(g, beta_v, beta_w):
    if beta_w == 0.0:
        return g.copy()
    dims = g.shape[1:]
    k1, k2, k3, ksq = wavenumbers(dims)
    with np.errstate(divide="ignore"):
        inv = np.where(ksq > 0, 1.0 / np.where(ksq > 0, ksq, 1.0), 0.0)
    c = beta_w * (1.0 + ksq) / (beta_v * ksq + beta_w * (1.0 + ksq))
    spec = [np.fft.rfftn(g[i]) for i in range(3)]
    kd = k1 * spec[0] + k2 * spec[1] + k3 * spec[2]
    sc = c * inv * kd
    ks = (k1, k2, k3)
    return np.stack([np.fft.irfftn(spec[i] - ks[i] * sc, s=dims, axes=(0, 1, 2)).astype(g.dtype) for i in range(3)])


def h1(f: np.ndarray) -> float:
    dims = f.shape
    n = f.size
    spec = np.fft.rfftn(f) / n
    ksq = wavenumbers(dims)[3]
    mult = np.full(ksq.shape, 2.0)
    mult[:, :, 0] = 1.0
    if dims[2] % 2 == 0:
        mult[:, :, -1] = 1.0
    return float(TWO_PI ** 3 * np.sum(mult * (1.0 + ksq) * (spec.real ** 2 + spec.imag ** 2)))


# ---------------------------------------------------------------------------
# transport -- transport.py:66-197
# ---------------------------------------------------------------------------
def trace(v: np.ndarray, dt: float, order: str) -> np.ndarray:
    """RK2 Heun (transport.py:66-76): x* = x - dt v; X = mod(x - dt/2 (v + v(x*)), 2pi)."""
    x = lattice(v.shape[1:])
    xs = x - dt * v
    vs = np.stack([interp(v[i], xs, order) for i in range(3)])
    return np.mod(x - 0.5 * dt * (v + vs), TWO_PI)


class Transport:
    """transport.py:89-116"""

    def __init__(self, v: np.ndarray, n_t: int, order: str):
        self.n_t, self.order, self.dt = n_t, order, 1.0 / n_t
        self.fwd = trace(v, self.dt, order)
        self.bwd = trace(-v, self.dt, order)
        d = div(v)
        half = 0.5 * self.dt
        self.jac_numer = 1.0 + half * interp(d, self.fwd, order)
        self.jac_denom = 1.0 - half * d
        self.adj_numer = 1.0 + half * interp(d, self.bwd, order)
        self.adj_denom = 1.0 - half * d

    def state_series(self, m0):
        s = np.empty((self.n_t + 1,) + m0.shape, dtype=m0.dtype)
        s[0] = m0
        for j in range(self.n_t):
            s[j + 1] = interp(s[j], self.fwd, self.order)
        return s

    def adjoint_series(self, lam_final):
        s = np.empty((self.n_t + 1,) + lam_final.shape, dtype=lam_final.dtype)
        s[self.n_t] = lam_final
        for j in range(self.n_t - 1, -1, -1):
            s[j] = interp(s[j + 1], self.bwd, self.order) * self.adj_numer / self.adj_denom
        return s

    def incremental(self, grad_series, vt):
        half = 0.5 * self.dt
        src = [-(vt[0] * g[0] + vt[1] * g[1] + vt[2] * g[2]) for g in grad_series]
        cur = np.zeros(vt.shape[1:], dtype=vt.dtype)
        for j in range(self.n_t):
            cur = interp(cur + half * src[j], self.fwd, self.order) + half * src[j + 1]
        return cur

    def jacobian(self, like):
        cur = np.ones(like.shape[1:], dtype=like.dtype)
        for _ in range(self.n_t):
            cur = interp(cur, self.fwd, self.order) * self.jac_numer / self.jac_denom
        return cur


def transport_labels(labels: np.ndarray, tr: Transport) -> np.ndarray:
    """synth.py:121-131"""
    out = np.zeros(labels.shape, dtype=np.int32)
    for lab in [int(i) for i in np.unique(labels) if i != 0]:
        moved = tr.state_series((labels == lab).astype(np.float64))[-1]
        out[moved >= 0.5] = lab
    return out


def dice_counts(l0: np.ndarray, l1: np.ndarray, lab: int):
    a, b = l0 == lab, l1 == lab
    return int(a.sum()), int(b.sum()), int((a & b).sum())


def dice_average(l0: np.ndarray, l1: np.ndarray) -> float:
    """metrics.py:60-87 (arithmetic average D_a over the union of labels)."""
    labs = sorted((set(np.unique(l0).tolist()) | set(np.unique(l1).tolist())) - {0})
    sc = []
    for lab in labs:
        na, nb, ov = dice_counts(l0, l1, lab)
        sc.append(1.0 if na + nb == 0 else 2.0 * ov / (na + nb))
    return float(np.mean(sc))


# ---------------------------------------------------------------------------
# objective / gradient / GN matvec / PCG / GN -- optim.py:80-367
# ---------------------------------------------------------------------------
class Problem:
    """Per-velocity state (optim.py:88-182) for images m0, m1 (any float dtype)."""

    def __init__(self, m0, m1, v, beta_v=1e-2, beta_w=0.0, n_t=4, order="cubic"):
        self.m0, self.m1, self.v = m0, m1, v
        self.beta_v, self.beta_w, self.n_t, self.order = beta_v, beta_w, n_t, order
        self.hvol = float(np.prod(spacing(m0.shape)))
        self.tr = Transport(v, n_t, order)
        self.m = self.tr.state_series(m0)
        self._gm = None
        self._g = None

    @property
    def grad_m(self):
        if self._gm is None:
            self._gm = np.stack([grad(self.m[j]) for j in range(self.n_t + 1)])
        return self._gm

    def objective(self) -> float:
        mis = self.m[-1] - self.m1
        val = 0.5 * float(np.dot(mis.ravel(), mis.ravel())) * self.hvol
        val += 0.5 * self.beta_v * float(np.dot(op_A(self.v).ravel(), self.v.ravel())) * self.hvol
        if self.beta_w > 0:
            val += 0.5 * self.beta_w * h1(div(self.v))
        return val

    def body(self, lam):
        dt = 1.0 / self.n_t
        acc = np.zeros((3,) + self.m0.shape)
        for j in range(self.n_t + 1):
            w = 0.5 * dt if j in (0, self.n_t) else dt
            acc += w * lam[j] * self.grad_m[j]
        return acc

    def gradient(self):
        if self._g is None:
            lam = self.tr.adjoint_series(self.m1 - self.m[-1])
            self._g = self.beta_v * op_A(self.v) + op_K(self.body(lam), self.beta_v, self.beta_w)
        return self._g

    def matvec(self, vt):
        mt = self.tr.incremental(self.grad_m, vt)
        lam = self.tr.adjoint_series(-mt)
        return self.beta_v * op_A(vt) + op_K(self.body(lam), self.beta_v, self.beta_w)


def pcg(matvec, rhs, precond, tol, max_iters):
    """optim.py:220-249 -> (x, iterations)"""
    x = np.zeros_like(rhs)
    if not np.any(rhs):
        return x, 0
    r = rhs.copy()
    z = precond(r)
    p = z.copy()
    rz = float(np.dot(r.ravel(), z.ravel()))
    z0 = float(np.linalg.norm(z))
    if z0 == 0.0:
        return x, 0
    for it in range(1, max_iters + 1):
        hp = matvec(p)
        php = float(np.dot(p.ravel(), hp.ravel()))
        if php <= 0.0:
            return x, it - 1
        a = rz / php
        x += a * p
        r -= a * hp
        z = precond(r)
        if float(np.linalg.norm(z)) / z0 <= tol:
            return x, it
        rzn = float(np.dot(r.ravel(), z.ravel()))
        p = z + (rzn / rz) * p
        rz = rzn
    return x, max_iters


def gauss_newton(m0, m1, beta_v=1e-2, beta_w=0.0, n_t=4, order="cubic", gtol=5e-2, max_gn=50, max_pcg=50,
                 c1=1e-4, backtrack=0.5, max_trials=20, v0=None):
    """optim.py:275-367 -> (v, record dict)"""
    hvol = float(np.prod(spacing(m0.shape)))
    lo = min(float(m0.min()), float(m1.min()))
    hi = max(float(m0.max()), float(m1.max()))
    shift = (hi - lo) ** 2 if hi > lo else 1.0
    kw = dict(beta_v=beta_v, beta_w=beta_w, n_t=n_t, order=order)
    v = np.zeros((3,) + m0.shape) if v0 is None else v0.astype(np.float64).copy()
    st = Problem(m0, m1, v, **kw)
    J = st.objective()
    g = st.gradient()
    gn = math.sqrt(max(float(np.dot(g.ravel(), g.ravel())) * hvol, 0.0))
    gn0 = gn
    rec = {"objective": [J], "pcg": [0], "rel_grad": [1.0 if gn0 > 0 else 0.0], "step": [0.0],
           "matvecs": 0}
    reason = "max-iterations"
    stagnant = 0

    def mv(w):
        rec["matvecs"] += 1
        return st.matvec(w)

    def prec(w):
        return op_inv_shifted(w, beta_v, shift)

    if gn0 == 0.0:
        reason = "zero-gradient"
    else:
        for _k in range(1, max_gn + 1):
            rel = gn / gn0
            if rel <= gtol:
                reason = "gradient-tolerance"
                break
            d, its = pcg(mv, -g, prec, min(0.5, math.sqrt(rel)), max_pcg)
            gd = float(np.dot(g.ravel(), d.ravel())) * hvol
            if gd >= 0.0 or not np.any(d):
                d = prec(-g)
                gd = float(np.dot(g.ravel(), d.ravel())) * hvol
            alpha, ok = 1.0, False
            for _ in range(max_trials):
                trial = Problem(m0, m1, v + alpha * d, **kw)
                Jt = trial.objective()
                if not math.isfinite(Jt):
                    alpha *= backtrack
                    continue
                if Jt <= J + c1 * alpha * gd:
                    ok = True
                    break
                alpha *= backtrack
            if not ok:
                reason = "line-search-failure"
                break
            step = alpha * math.sqrt(max(float(np.dot(d.ravel(), d.ravel())) * hvol, 0.0))
            Jp, J = J, Jt
            v, st = v + alpha * d, trial
            g = st.gradient()
            gn = math.sqrt(max(float(np.dot(g.ravel(), g.ravel())) * hvol, 0.0))
            rec["objective"].append(J)
            rec["pcg"].append(its)
            rec["rel_grad"].append(gn / gn0)
            rec["step"].append(alpha)
            stagnant = stagnant + 1 if (Jp - J) / max(abs(Jp), 1e-300) < 1e-6 else 0
            if stagnant >= 2:
                reason = "objective-stagnation"
                break
            if step < 1e-10:
                reason = "step-stagnation"
                break
        if gn0 > 0 and gn / gn0 <= gtol and reason == "max-iterations":
            reason = "gradient-tolerance"
    jac = st.tr.jacobian(v)
    rec["j_min"], rec["j_max"] = float(jac.min()), float(jac.max())
    num = float(np.sum((st.m[-1] - m1) ** 2))
    den = float(np.sum((m0 - m1) ** 2))
    rec["relative_residual"] = 0.0 if den == 0.0 else num / den
    rec["reason"] = reason
    rec["deformed"] = st.m[-1]
    return v, rec


# ---------------------------------------------------------------------------
# synthetic inputs -- identical definitions to the package's
# ---------------------------------------------------------------------------
def velocity(K: int, dims) -> np.ndarray:
    """synth.py:104-118"""
    x, y, z = lattice(dims) - math.pi
    out = np.zeros((3,) + tuple(dims))
    for k in range(1, K + 1):
        a = k ** -0.5
        out[0] += a * np.cos(k * y) * np.cos(k * x)
        out[1] += a * np.sin(k * z) * np.sin(k * y)
        out[2] += a * np.cos(k * x) * np.cos(k * z)
    return out
