"""Per-operator parity at the bench sizes.

256^3 (C2's grid): every operator against the CPU oracle (oracle/, pinned to
the live reference by test_oracle_golden.py) on IDENTICAL float32 inputs --
the spectral operators A (both engines), shifted inverse and K, FD8 gradient
and divergence (bit-exact), both RK2 traces, and the state / adjoint /
incremental-state / Jacobian sweeps.  Tolerance: the north star's 1e-5
relative L2 per operator (FD8: bit-exact; traces: 1e-5 rad).

1024^3 (C3's grid): the oracle cannot hold 1024^3 f64 transport arrays on the
host, so the gathers, traces and FD8 are checked at 2^17 sampled voxels with
the oracle's own formulas (interp.py / diffops.py restatements) on the full
float32 fields, and the spectral operators against cuFFT in float64
(torch.fft -- test-only cross-check, like the reference's f64 pocketfft).
"""
import math

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    import paper_2209_08189_b200 as P
    assert torch.cuda.is_available()
    return P


def _np(t):
    return t.detach().cpu().numpy()


def _periodic_maxdiff(a, b):
    d = np.abs(a - b)
    return float(np.minimum(d, 2 * math.pi - d).max())


# ---------------------------------------------------------------------------- 256^3
@pytest.fixture(scope="module")
def c2(P):
    from oracle import velreg_oracle as O
    n = 256
    g = P.make_grid((n, n, n))
    v = (0.2 * O.velocity(2, g.dims)).astype(np.float32)
    x = O.lattice(g.dims)
    r = np.sqrt(sum((x[i] - math.pi) ** 2 for i in range(3)))
    f = (0.5 * (1.0 - np.tanh((r - 1.2) / 0.19635))).astype(np.float32)
    del x, r
    w = np.random.default_rng(5).standard_normal((3,) + g.dims).astype(np.float32)
    return {"g": g, "v": v, "f": f, "w": w}


def test_256_spectral_vs_oracle(P, c2):
    """A (separable f64 line engine and the 3-D f64 path), shifted inverse and
    K at 256^3 -- the precision case SURVEY §7 flags (an f32 3-D FFT gives
    3-5e-5 for A here)."""
    from oracle import velreg_oracle as O
    from paper_2209_08189_b200 import _lib
    g = c2["g"]
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    lib = _lib.lib()
    for name in ("v", "w"):
        x = c2[name]
        X = P.VectorField(g, x)
        x64 = x.astype(np.float64)
        refA = O.op_A(x64)
        for mode in (1, 0):
            prev = lib.vr_set_spec_a_mode(mode)
            try:
                err = rel_l2(_np(P.apply_A(X, ops).data), refA)
            finally:
                lib.vr_set_spec_a_mode(prev)
            assert err < TOL, (name, mode, err)
        assert rel_l2(_np(P.apply_inv_shifted_A(X, ops, 1.0).data), O.op_inv_shifted(x64, 1e-2, 1.0)) < TOL
        assert rel_l2(_np(P.apply_K(X, ops).data), O.op_K(x64, 1e-2, 1e-4)) < TOL


def test_256_fd8_bit_exact(P, c2):
    from oracle import velreg_oracle as O
    g = c2["g"]
    np.testing.assert_array_equal(_np(P.fd8_gradient(P.ScalarField(g, c2["f"])).data), O.grad(c2["f"]))
    np.testing.assert_array_equal(_np(P.fd8_divergence(P.VectorField(g, c2["v"])).values), O.div(c2["v"]))


@pytest.mark.parametrize("order", ["cubic", "linear"])
def test_256_transport_vs_oracle(P, c2, order):
    from oracle import velreg_oracle as O
    g, v, f = c2["g"], c2["v"], c2["f"]
    v64 = v.astype(np.float64)
    tr = O.Transport(v64, 4, order)
    V = P.VectorField(g, v)
    cfg = P.TransportConfig(4, order)
    tops = P.TransportOperators(V, cfg)
    # traces (radians, periodic) and source factors
    assert _periodic_maxdiff(_np(tops.forward.points), tr.fwd) < 1e-5
    assert _periodic_maxdiff(_np(tops.backward.points), tr.bwd) < 1e-5
    assert rel_l2(_np(tops.jac_factor), tr.jac_numer / tr.jac_denom) < TOL
    assert rel_l2(_np(tops.adj_factor), tr.adj_numer / tr.adj_denom) < TOL
    # state series
    ms = P.solve_state_series(P.ScalarField(g, f), V, cfg, tops)
    ref = tr.state_series(f)
    for j in range(1, 5):
        assert rel_l2(_np(ms[j]), ref[j]) < TOL, j
    # adjoint from the final condition m(1) - m0 (an image-shaped f32 field)
    lam1 = (ref[-1] - f).astype(np.float32)
    lam = P.solve_adjoint(P.ScalarField(g, lam1), V, cfg, tops)
    lref = tr.adjoint_series(lam1)
    for j in range(4):
        assert rel_l2(_np(lam[j]), lref[j]) < TOL, j
    # incremental state along the device state series (identical f32 inputs)
    vt = c2["w"] * 0.1
    ms_np = _np(ms)
    inc = P.solve_incremental_state(ms, V, P.VectorField(g, vt), cfg, tops)
    iref = tr.incremental([O.grad(ms_np[j]) for j in range(5)], vt.astype(np.float64))
    assert rel_l2(_np(inc.values), iref) < TOL
    # Jacobian determinant
    jac = P.jacobian_determinant(V, cfg, tops)
    assert rel_l2(_np(jac.values), tr.jacobian(v64)) < TOL


# --------------------------------------------------------------------------- 1024^3
N_SAMPLE = 1 << 17


@pytest.fixture(scope="module")
def c3(P):
    from paper_2209_08189_b200.synth import velocity_tensor
    n = 1024
    g = P.make_grid((n, n, n))
    v = velocity_tensor(2, g, 0.2)
    rng = np.random.default_rng(11)
    idx = np.sort(rng.choice(n ** 3, N_SAMPLE, replace=False))
    ijk = np.stack(np.unravel_index(idx, g.dims))
    return {"g": g, "v": v, "idx": idx, "ijk": ijk}


def _take(t, idx):
    """values of a device field at flat voxel indices (host f32)."""
    return t.reshape(-1)[torch.from_numpy(idx).to(t.device)].cpu().numpy()


@pytest.mark.parametrize("order", ["linear", "cubic"])
def test_1024_trace_and_sweep_sampled(P, c3, order):
    """RK2 trace and one semi-Lagrangian step at 1024^3, checked at sampled
    voxels with the oracle's interpolation (interp.py:112-128) on the full
    float32 fields: x* = x - dt v(x), X = x - dt/2 (v(x) + v(x*))."""
    from oracle import velreg_oracle as O
    g, v, idx, ijk = c3["g"], c3["v"], c3["idx"], c3["ijk"]
    dt = 1.0 / 16
    h = np.array(g.spacing).reshape(3, 1)
    tops = P.TransportOperators(P.VectorField(g, v), P.TransportConfig(16, order))
    got = np.stack([_take(tops.forward.displacement[c], idx) for c in range(3)])
    x = ijk * h
    v_np = v.cpu().numpy()
    vx = np.stack([v_np[c].reshape(-1)[idx].astype(np.float64) for c in range(3)])
    xs = x - dt * vx
    vs = np.stack([O.interp(v_np[c], xs, order).astype(np.float64) for c in range(3)])
    X = x - 0.5 * dt * (vx + vs)
    Xgot = x - got.astype(np.float64) * h     # displacement (index units) -> radians
    assert float(np.abs(Xgot - X).max()) < 1e-5
    # one state step at the device departure points
    f = (torch.sin(torch.arange(g.dims[0], device="cuda", dtype=torch.float32) * 0.05).view(-1, 1, 1)
         * torch.cos(torch.arange(g.dims[1], device="cuda", dtype=torch.float32) * 0.03).view(1, -1, 1)
         + torch.arange(g.dims[2], device="cuda", dtype=torch.float32).view(1, 1, -1) * 1e-3)
    out = tops.advect_step(f)
    ref = O.interp(f.cpu().numpy(), Xgot, order)
    assert rel_l2(_take(out, idx), ref) < TOL


def test_1024_fd8_sampled_bit_exact(P, c3):
    """FD8 gradient at 1024^3 against the oracle's evaluation order
    (diffops.py:84-105: out += c_o (f[i+o] - f[i-o]) in f32, then / h)."""
    from oracle import velreg_oracle as O
    g, v, idx, ijk = c3["g"], c3["v"], c3["idx"], c3["ijk"]
    f = v[0]
    gr = P.fd8_gradient(P.ScalarField(g, f)).data
    fn = f.cpu().numpy()
    n = g.dims
    for a in range(3):
        out = np.zeros(len(idx), dtype=np.float32)
        for o, c in enumerate(O.FD8, start=1):
            ip = ijk.copy()
            im = ijk.copy()
            ip[a] = (ip[a] + o) % n[a]
            im[a] = (im[a] - o) % n[a]
            out += c * (fn[tuple(ip)] - fn[tuple(im)])
        out /= g.spacing[a]
        np.testing.assert_array_equal(_take(gr[a], idx), out)


def test_1024_spectral_vs_cufft_f64(P, c3):
    """A, shifted inverse and K at 1024^3 against torch.fft (cuFFT) in float64
    on the identical float32 input (test-only cross-check), one f64 component
    at a time (a 1024^3 complex128 half spectrum is 8.6 GB)."""
    g, v = c3["g"], c3["v"]
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    V = P.VectorField(g, v)
    dims = tuple(g.dims)
    n1, n2, n3 = dims
    dev = v.device
    k1 = torch.fft.fftfreq(n1, d=1.0 / n1, dtype=torch.float64, device=dev).view(n1, 1, 1)
    k2 = torch.fft.fftfreq(n2, d=1.0 / n2, dtype=torch.float64, device=dev).view(1, n2, 1)
    k3 = torch.arange(n3 // 2 + 1, dtype=torch.float64, device=dev).view(1, 1, -1)
    ksq = k1 ** 2 + k2 ** 2 + k3 ** 2
    ks = (k1, k2, k3)

    def rfft(c):
        return torch.fft.rfftn(v[c].double())

    def irfft(F):
        return torch.fft.irfftn(F, s=dims)

    def check(got, refs):
        num = den = 0.0
        for c in range(3):
            r = refs(c)
            num += float(torch.sum((got[c].double() - r) ** 2))
            den += float(torch.sum(r ** 2))
            del r
        return math.sqrt(num / den)

    got = P.apply_A(V, ops).data
    assert check(got, lambda c: irfft(rfft(c) * ksq)) < TOL
    got = P.apply_inv_shifted_A(V, ops, 1.0).data
    assert check(got, lambda c: irfft(rfft(c) / (1e-2 * ksq + 1.0))) < TOL
    got = P.apply_K(V, ops).data
    cb = 1e-4 * (1 + ksq) / (1e-2 * ksq + 1e-4 * (1 + ksq))
    f = torch.where(ksq > 0, cb / torch.where(ksq > 0, ksq, torch.ones_like(ksq)), torch.zeros_like(ksq))
    kd = None
    for c in range(3):
        t = ks[c] * rfft(c)
        kd = t if kd is None else kd + t
        del t
    kd *= f
    del f, cb
    assert check(got, lambda c: irfft(rfft(c) - ks[c] * kd)) < TOL
    del kd, got
    torch.cuda.empty_cache()


def test_clarity_shape_ops_vs_oracle(P):
    """C5's CLARITY shape reduced with its odd prime factors kept (88 x 104 x
    166: 11, 13, 83 -- radix-11/13 butterflies and a direct radix-83 stage in
    the generic engine): spectral operators, FD8 and a linear SL step against
    the oracle at 1e-5 (FD8 bit-exact)."""
    from oracle import velreg_oracle as O
    dims = (88, 104, 166)
    g = P.make_grid(dims)
    rng = np.random.default_rng(21)
    w = rng.standard_normal((3,) + dims).astype(np.float32)
    f = rng.random(dims).astype(np.float32)
    v = (0.2 * O.velocity(2, dims)).astype(np.float32)
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-5)
    W = P.VectorField(g, w)
    w64 = w.astype(np.float64)
    assert rel_l2(_np(P.apply_A(W, ops).data), O.op_A(w64)) < TOL
    assert rel_l2(_np(P.apply_inv_shifted_A(W, ops, 1.0).data), O.op_inv_shifted(w64, 1e-2, 1.0)) < TOL
    assert rel_l2(_np(P.apply_K(W, ops).data), O.op_K(w64, 1e-2, 1e-5)) < TOL
    np.testing.assert_array_equal(_np(P.fd8_gradient(P.ScalarField(g, f)).data), O.grad(f))
    tr = O.Transport(v.astype(np.float64), 4, "linear")
    tops = P.TransportOperators(P.VectorField(g, v), P.TransportConfig(4, "linear"))
    got = _np(P.solve_state(P.ScalarField(g, f), tops.v, tops.cfg, tops).values)
    assert rel_l2(got, tr.state_series(f.astype(np.float64))[-1]) < TOL
