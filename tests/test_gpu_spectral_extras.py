"""North-star spectral extras without a reference counterpart: the H2 operator
(symbol |k|^4), its shifted inverse 1/(beta_v |k|^4 + shift) and the Gaussian
smoothing exp(-sigma^2 |k|^2 / 2) -- pinned analytically by eigenfunctions.

A plane wave cos(k.x + phi) with integer k is an eigenfunction of every
Fourier multiplier s(|k|^2): the operator returns s * cos(k.x + phi).  Each
component carries its own wave, including Nyquist and mixed-sign modes, on a
power-of-two grid (fast engine) and a non-power-of-two grid (generic
mixed-radix engine).  Tolerance 1e-5 relative L2 (the north star's operator
bar); A and the shifted inverse are checked the same way as a control.
"""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    import paper_2209_08189_b200 as P
    assert torch.cuda.is_available()
    return P


def _waves(dims):
    """(3, N1, N2, N3) field: component c = cos(k_c . x + phi_c), and |k_c|^2."""
    n1, n2, n3 = dims
    ks = [(1, 2, 3), (-(n1 // 2) + 1, 3, n3 // 2 - 1), (2, -(n2 // 2 - 2), 1)]
    phis = [0.3, -1.1, 2.0]
    x = [np.arange(n) * (2 * math.pi / n) for n in dims]
    X = np.meshgrid(*x, indexing="ij")
    field = np.stack([np.cos(k[0] * X[0] + k[1] * X[1] + k[2] * X[2] + ph) for k, ph in zip(ks, phis)])
    ksq = np.array([k[0] ** 2 + k[1] ** 2 + k[2] ** 2 for k in ks], dtype=np.float64)
    return field.astype(np.float32), field, ksq


def _check(got, exact_f64, mult):
    ref = exact_f64 * mult.reshape(3, 1, 1, 1)
    got = got.detach().cpu().numpy().astype(np.float64)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err < TOL, err


@pytest.mark.parametrize("dims", [(32, 32, 32), (64, 32, 48), (20, 24, 30)])
def test_eigenfunctions(P, dims):
    from paper_2209_08189_b200.diffops import apply_A2, apply_inv_shifted_A2, gaussian_smooth
    g = P.make_grid(dims)
    f32, f64, ksq = _waves(dims)
    V = P.VectorField(g, f32)
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    beta, shift, sigma = 1e-2, 3.0, 0.7
    _check(apply_A2(V, ops).data, f64, ksq ** 2)
    _check(apply_inv_shifted_A2(V, ops, shift).data, f64, 1.0 / (beta * ksq ** 2 + shift))
    _check(gaussian_smooth(V, ops.workspace, sigma).data, f64, np.exp(-0.5 * sigma ** 2 * ksq))
    # scalar Gaussian (one component; the low mode: exp(-sigma^2 |k|^2 / 2) of
    # the Nyquist-side waves is below f32 rounding noise of the transform)
    Sf = P.ScalarField(g, f32[0])
    got = gaussian_smooth(Sf, ops.workspace, sigma).values
    ref = f64[0] * math.exp(-0.5 * sigma ** 2 * ksq[0])
    err = np.linalg.norm(got.cpu().numpy() - ref) / np.linalg.norm(ref)
    assert err < TOL, err
    # controls: A and its shifted inverse on the same eigenfunctions
    _check(P.apply_A(V, ops).data, f64, ksq)
    _check(P.apply_inv_shifted_A(V, ops, shift).data, f64, 1.0 / (beta * ksq + shift))


def test_inverse_pairs(P):
    """apply_inv_shifted_A2 inverts (beta_v A2 + shift): a round trip returns
    the input on a random smooth field."""
    from paper_2209_08189_b200.diffops import apply_A2, apply_inv_shifted_A2
    dims = (32, 32, 32)
    g = P.make_grid(dims)
    rng = np.random.default_rng(4)
    f = rng.standard_normal((3,) + dims).astype(np.float32)
    V = P.VectorField(g, f)
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    shift = 2.0
    a2 = apply_A2(V, ops).data
    lhs = (1e-2 * a2 + shift * V.data)
    back = apply_inv_shifted_A2(P.VectorField(g, lhs), ops, shift).data
    err = float(torch.linalg.vector_norm(back - V.data) / torch.linalg.vector_norm(V.data))
    assert err < 1e-5, err


@pytest.mark.parametrize("dims", [(512, 128, 128), (1024, 128, 256), (2048, 128, 128)])
def test_separable_A_long_x1(P, dims):
    """A on the separable line engine with x1 lines of 512 / 1024 / 2048 (the
    three-step long_kernel; the same kernels run the x1 pass of the distributed
    A): plane-wave eigenfunctions at 1e-5 and the 3-D f64 engine at 1e-6."""
    from paper_2209_08189_b200 import _lib
    g = P.make_grid(dims)
    ops = P.RegOperators.for_grid(g, 1e-2, 0.0)
    if dims[0] == 512:
        f32, f64, ksq = _waves(dims)
        _check(P.apply_A(P.VectorField(g, f32), ops).data, f64, ksq)
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((3,) + dims, device="cuda", generator=gen)
    sep = P.apply_A(P.VectorField(g, x), ops).data.clone()
    lib = _lib.lib()
    prev = lib.vr_set_spec_a_mode(0)
    try:
        full = P.apply_A(P.VectorField(g, x), ops).data
    finally:
        lib.vr_set_spec_a_mode(prev)
    err = float(torch.linalg.vector_norm((sep - full).double()) / torch.linalg.vector_norm(full.double()))
    assert err < 1e-6, err
