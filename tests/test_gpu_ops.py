"""Per-operator parity of the CUDA path against the reference.

Inputs are the float32 arrays of the golden fixture (tests/golden/ops_16x20x24,
made by the LIVE reference); larger sizes compare against the CPU oracle
(pinned to the same fixtures by test_oracle_golden.py) on identical float32
inputs.  Tolerance: the north star's <= 1e-5 relative L2 per operator; FD8 is
bit-exact for float32 input.
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


def _grid(P, fx):
    return P.make_grid(tuple(int(n) for n in fx["dims"]))


def _np(t):
    return t.detach().cpu().numpy()


def test_interpolate_values(P, ops_fx):
    g = _grid(P, ops_fx)
    for order in ("linear", "cubic"):
        for src in ("smooth", "rand"):
            vals = ops_fx[f"f_{src}"]
            got = P.interpolate_values(vals, ops_fx[f"trace_fwd_{order}"].astype(np.float64), order, g.spacing)
            assert rel_l2(_np(got), ops_fx[f"interp_{order}_{src}_trace"]) < TOL
            got = P.interpolate_values(vals, ops_fx["pts_rand"], order, g.spacing)   # f32 points, out of box
            assert rel_l2(_np(got), ops_fx[f"interp_{order}_{src}_rand"]) < TOL


def test_trace_characteristics(P, ops_fx):
    g = _grid(P, ops_fx)
    v = P.VectorField(g, ops_fx["v"])
    for order in ("linear", "cubic"):
        for sign, key in ((1, "fwd"), (-1, "bwd")):
            vv = v if sign > 0 else P.VectorField(g, -ops_fx["v"])
            pts = _np(P.trace_characteristics(vv, 0.25, order).points)
            d = np.abs(pts - ops_fx[f"trace_{key}_{order}"])
            d = np.minimum(d, 2 * math.pi - d)   # periodic
            assert d.max() < 1e-5


def test_fd8_bit_exact(P, ops_fx):
    g = _grid(P, ops_fx)
    got = _np(P.fd8_gradient(P.ScalarField(g, ops_fx["f_rand"])).data)
    np.testing.assert_array_equal(got, ops_fx["fd8_grad_f32"])
    got = _np(P.fd8_divergence(P.VectorField(g, ops_fx["w"])).values)
    np.testing.assert_array_equal(got, ops_fx["fd8_div_f32"])
    assert rel_l2(got, ops_fx["fd8_div"]) < TOL


@pytest.mark.parametrize("dims", [(10, 14, 10), (40, 72, 96), (64, 64, 64), (24, 16, 128), (16, 24, 256),
                                  (10, 12, 512)])
def test_fd8_bit_exact_sizes(P, dims):
    """Ragged tiles, the minimum stencil size and magnitudes from 1e-38 to 1e30
    (the reciprocal division must reproduce IEEE division bit for bit)."""
    from oracle import velreg_oracle as O
    rng = np.random.default_rng(7)
    g = P.make_grid(dims)
    scale = 10.0 ** rng.uniform(-38, 30, size=dims)
    f = (rng.standard_normal(dims) * scale).astype(np.float32)
    f[rng.random(dims) < 0.05] = 0.0
    np.testing.assert_array_equal(_np(P.fd8_gradient(P.ScalarField(g, f)).data), O.grad(f))
    w = (rng.standard_normal((3,) + dims)).astype(np.float32)
    np.testing.assert_array_equal(_np(P.fd8_divergence(P.VectorField(g, w)).values), O.div(w))


@pytest.mark.parametrize("dims", [(64, 64, 64), (16, 24, 256)])
def test_fd8_bit_exact_tiny_band(P, dims):
    """Sums between 2^-124 and 2^-100 (far-field values of transported
    templates) take the inline scaled reciprocal path: still IEEE bits, in both
    the tile and the row-tile kernels."""
    from oracle import velreg_oracle as O
    from paper_2209_08189_b200 import _lib
    rng = np.random.default_rng(11)
    g = P.make_grid(dims)
    f = (rng.standard_normal(dims) * 10.0 ** rng.uniform(-37, -29, size=dims)).astype(np.float32)
    ref = O.grad(f)
    lib = _lib.lib()
    for mode in (0, 1):
        prev = lib.vr_set_fd8_mode(mode)
        try:
            np.testing.assert_array_equal(_np(P.fd8_gradient(P.ScalarField(g, f)).data), ref)
        finally:
            lib.vr_set_fd8_mode(prev)


@pytest.mark.parametrize("dims", [(32, 40, 128), (20, 32, 256)])
def test_fd8_row_kernel_matches_tile_kernel(P, dims):
    """vr_set_fd8_mode A/B: the bulk-copy row-tile kernel and the cp.async tile
    kernel give identical bits (gradient and divergence)."""
    from paper_2209_08189_b200 import _lib
    lib = _lib.lib()
    g = P.make_grid(dims)
    gen = torch.Generator(device="cuda").manual_seed(1)
    f = torch.randn(dims, device="cuda", generator=gen) * 10.0
    v = torch.randn((3,) + dims, device="cuda", generator=gen)
    outs = {}
    for mode in (0, 1):
        prev = lib.vr_set_fd8_mode(mode)
        try:
            outs[mode] = (P.fd8_gradient(P.ScalarField(g, f)).data.clone(),
                          P.fd8_divergence(P.VectorField(g, v)).values.clone())
        finally:
            lib.vr_set_fd8_mode(prev)
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_fd8_requires_nine(P):
    g = P.make_grid((8, 16, 16))
    with pytest.raises(P.GridError):
        P.fd8_gradient(P.ScalarField.zeros(g))


def test_spectral_operators(P, ops_fx):
    g = _grid(P, ops_fx)
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    v = P.VectorField(g, ops_fx["v"])
    w = P.VectorField(g, ops_fx["w"])
    assert rel_l2(_np(P.apply_A(v, ops).data), ops_fx["apply_A_v"]) < TOL
    assert rel_l2(_np(P.apply_A(w, ops).data), ops_fx["apply_A_w"]) < TOL
    assert rel_l2(_np(P.apply_inv_shifted_A(w, ops, 1.0).data), ops_fx["inv_shifted_A_w_1"]) < TOL
    assert rel_l2(_np(P.apply_inv_shifted_A(w, ops, 0.37).data), ops_fx["inv_shifted_A_w_037"]) < TOL
    assert rel_l2(_np(P.apply_K(w, ops).data), ops_fx["apply_K_w"]) < TOL
    assert rel_l2(_np(P.apply_K(v, ops).data), ops_fx["apply_K_v"]) < TOL
    ops3 = P.RegOperators.for_grid(g, 1e-2, 3.0)
    assert rel_l2(_np(P.apply_K(w, ops3).data), ops_fx["apply_K_w_bw3"]) < TOL
    ops0 = P.RegOperators.for_grid(g, 1e-2, 0.0)
    assert torch.equal(P.apply_K(w, ops0).data, w.data)   # beta_w = 0 -> identity copy
    div = P.fd8_divergence(v)
    assert abs(P.h1_energy(div, ops.workspace) / float(ops_fx["h1_energy_divv"]) - 1) < TOL
    fr = P.ScalarField(g, ops_fx["f_rand"])
    assert abs(P.h1_energy(fr, ops.workspace) / float(ops_fx["h1_energy_frand"]) - 1) < TOL


def test_transport_sweeps(P, ops_fx):
    g = _grid(P, ops_fx)
    v = P.VectorField(g, ops_fx["v"])
    vt = P.VectorField(g, ops_fx["vt"])
    f = P.ScalarField(g, ops_fx["f_smooth"])
    lam = P.ScalarField(g, ops_fx["f_rand"] - 0.5)
    for order in ("linear", "cubic"):
        cfg = P.TransportConfig(4, order)
        tops = P.TransportOperators(v, cfg)
        jac = ops_fx[f"jac_numer_{order}"].astype(np.float64) / ops_fx[f"jac_denom_{order}"]
        adj = ops_fx[f"adj_numer_{order}"].astype(np.float64) / ops_fx[f"adj_denom_{order}"]
        assert rel_l2(_np(tops.jac_factor), jac) < TOL
        assert rel_l2(_np(tops.adj_factor), adj) < TOL
        series = P.solve_state_series(f, v, cfg, tops)
        assert rel_l2(_np(series), ops_fx[f"state_series_{order}"]) < TOL
        assert rel_l2(_np(P.solve_state(f, v, cfg, tops).values), ops_fx[f"state_series_{order}"][-1]) < TOL
        assert rel_l2(_np(P.solve_adjoint(lam, v, cfg, tops)), ops_fx[f"adjoint_series_{order}"]) < TOL
        inc = P.solve_incremental_state(series, v, vt, cfg, tops)
        assert rel_l2(_np(inc.values), ops_fx[f"incstate_{order}"]) < TOL
        assert rel_l2(_np(P.jacobian_determinant(v, cfg, tops).values), ops_fx[f"jacobian_{order}"]) < TOL


def test_objective_gradient_matvec(P, ops_fx):
    g = _grid(P, ops_fx)
    v = P.VectorField(g, 0.5 * ops_fx["v"].astype(np.float64))
    w = P.VectorField(g, ops_fx["w"])
    for order in ("cubic", "linear"):
        m0 = P.ScalarField(g, ops_fx[f"obj_m0_{order}"])
        m1 = P.ScalarField(g, ops_fx[f"obj_m1_{order}"])
        for bw in (0.0, 1e-4):
            tag = f"{order}_bw{bw:g}"
            cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=bw, n_t=4, interp_order=order)
            st = P.ObjectiveState(m0, m1, v, cfg, P.RegOperators.for_grid(g, 1e-2, bw))
            assert abs(st.objective / float(ops_fx[f"objective_{tag}"]) - 1) < TOL
            assert rel_l2(_np(st.deformed.values), ops_fx[f"deformed_{tag}"]) < TOL
            assert rel_l2(_np(st.gradient.data), ops_fx[f"gradient_{tag}"]) < TOL
            assert rel_l2(_np(P.hessian_matvec(w, st).data), ops_fx[f"matvec_{tag}"]) < TOL


def test_labels_and_dice(P, ops_fx):
    g = _grid(P, ops_fx)
    v = P.VectorField(g, ops_fx["v"])
    lab0 = P.LabelMap(g, ops_fx["labels0"])
    for order in ("cubic", "linear"):
        moved = P.transport_labels(lab0, v, P.TransportConfig(4, order))
        ref = ops_fx[f"labels_moved_{order}"]
        assert int((_np(moved.labels) != ref).sum()) == 0
        rep = P.dice_averages(moved, lab0)
        np.testing.assert_allclose([rep.d_a, rep.d_vw, rep.d_ivw], ops_fx[f"dice_avgs_{order}"], rtol=1e-6)
        assert rep.label_ids == [int(i) for i in ops_fx[f"dice_ids_{order}"]]


def test_restrict(P, ops_fx):
    g = _grid(P, ops_fx)
    got = P.restrict(P.ScalarField(g, ops_fx["f_rand"]), 2)
    np.testing.assert_array_equal(_np(got.values), ops_fx["restrict2_f"])


def test_prolong_spectral(P, ops_fx):
    g = _grid(P, ops_fx)
    coarse = P.make_grid(tuple(n // 2 for n in g.dims))
    got = P.prolong_spectral(P.VectorField(coarse, ops_fx["prolong_in"]), g)
    assert rel_l2(_np(got.data), ops_fx["prolong_out"]) < TOL


# ---- larger grids against the oracle (identical float32 inputs) ----------------
@pytest.mark.parametrize("n", [64, 96])
def test_ops_vs_oracle(P, n):
    from oracle import velreg_oracle as O
    dims = (n, n, n)
    g = P.make_grid(dims)
    rng = np.random.default_rng(n)
    v = (0.2 * O.velocity(2, dims)).astype(np.float32)
    f = rng.random(dims).astype(np.float32)
    w = rng.standard_normal((3,) + dims).astype(np.float32)
    v64 = v.astype(np.float64)
    for order in ("linear", "cubic"):
        tr = O.Transport(v64, 4, order)
        tops = P.TransportOperators(P.VectorField(g, v), P.TransportConfig(4, order))
        fs = P.ScalarField(g, f)
        got = _np(P.solve_state(fs, tops.v, tops.cfg, tops).values)
        assert rel_l2(got, tr.state_series(f.astype(np.float64))[-1]) < TOL
        assert rel_l2(_np(tops.jac_factor), tr.jac_numer / tr.jac_denom) < TOL
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    W = P.VectorField(g, w)
    assert rel_l2(_np(P.apply_A(W, ops).data), O.op_A(w.astype(np.float64))) < TOL
    assert rel_l2(_np(P.apply_K(W, ops).data), O.op_K(w.astype(np.float64), 1e-2, 1e-4)) < TOL
    assert rel_l2(_np(P.apply_inv_shifted_A(W, ops, 1.0).data),
                  O.op_inv_shifted(w.astype(np.float64), 1e-2, 1.0)) < TOL
    np.testing.assert_array_equal(_np(P.fd8_gradient(P.ScalarField(g, f)).data), O.grad(f))


@pytest.mark.parametrize("dims,scale", [((256, 256, 256), 0.2), ((32, 32, 32), 1.0), ((16, 20, 32), 0.5),
                                        ((36, 40, 64), 2.0), ((12, 12, 32), 0.3), ((20, 16, 96), 4.0)])
def test_staged_gather_matches_direct(P, dims, scale):
    """The shared-memory-staged sweeps (stage_tma.cuh: per-tile source box copied
    with cp.async.bulk, taps from shared memory) return the direct per-point
    gather's floats to the ulp -- smooth fields, large displacements (boxes over
    budget -> direct fallback inside the same launch) and random displacements
    -- for the state/adjoint sweep (with factor) and the incremental state
    step, trilinear and tricubic."""
    from paper_2209_08189_b200 import _lib, transport
    from paper_2209_08189_b200.synth import velocity_array
    g = P.make_grid(dims)
    gen = torch.Generator(device="cuda").manual_seed(3)
    f = torch.rand(dims, device="cuda", generator=gen)
    v = P.VectorField(g, scale * velocity_array(2, g))
    rnd = (torch.rand((3,) + dims, device="cuda", generator=gen) - 0.5) * (2 * min(dims))
    vt = torch.randn((3,) + dims, device="cuda", generator=gen)
    gm = torch.randn((3,) + dims, device="cuda", generator=gen)
    lib = _lib.lib()
    for order in ("cubic", "linear"):
        tops = P.TransportOperators(v, P.TransportConfig(4, order))
        for disp in (tops.forward.displacement, tops.backward.displacement, rnd):
            outs = {}
            for mode in (0, 1, 5):
                prev = lib.vr_set_gather_mode(mode)
                try:
                    res = [transport.advect(f, disp, order, factor=tops.adj_factor), transport.advect(f, disp, order)]
                    b = torch.empty_like(f)
                    for last in (0, 1, 2):
                        rc = lib.vr_incstate_step(f.data_ptr(), _lib.dims_arg(dims), disp.data_ptr(), vt.data_ptr(),
                                                  gm.data_ptr(), 0.25, _lib.ORDER[order], last, b.data_ptr(), None,
                                                  _lib.stream())
                        _lib.check(rc, "vr_incstate_step")
                        res.append(b.clone())
                    outs[mode] = res
                finally:
                    lib.vr_set_gather_mode(prev)
            torch.cuda.synchronize()
            for mode in (1, 5):
                for x, y in zip(outs[0], outs[mode]):
                    # same taps and arithmetic order; FMA contraction may differ by an ulp
                    assert float((x - y).abs().max()) <= 4e-6 * float(x.abs().max()), (order, dims, mode)


@pytest.mark.parametrize("dims", [(2048, 8, 16), (1024, 16, 16), (512, 16, 32), (256, 256, 32)])
def test_spectral_long_x1_lines(P, dims):
    """Power-of-two x1 lines up to 2048 (the transposed x1 pass of an 8-rank
    weak-scaling run has N1 = 2048): A and the shifted inverse against the
    oracle, and the coupled K (three-pass long-line path for 512-2048)."""
    from oracle import velreg_oracle as O
    g = P.make_grid(dims)
    w = np.random.default_rng(7).standard_normal((3,) + dims).astype(np.float32)
    ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    W = P.VectorField(g, w)
    assert rel_l2(_np(P.apply_A(W, ops).data), O.op_A(w.astype(np.float64))) < TOL
    assert rel_l2(_np(P.apply_inv_shifted_A(W, ops, 1.0).data),
                  O.op_inv_shifted(w.astype(np.float64), 1e-2, 1.0)) < TOL
    # K on 512-2048-point x1 lines: forward / 3-component symbol / inverse passes
    assert rel_l2(_np(P.apply_K(W, ops).data), O.op_K(w.astype(np.float64), 1e-2, 1e-4)) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(32, 32, 32), (16, 20, 24)])
def test_trace_lean_matches_general(dims):
    """vr_set_trace_mode A/B: the float4-velocity trace (default) against the
    general flat-index trace and the lean periodic trace, both orders, with source factors,
    including displacements beyond one period (scaled velocity)."""
    import torch
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import _lib
    from paper_2209_08189_b200.synth import velocity_array
    g = P.make_grid(dims)
    lib = _lib.lib()
    for scale in (0.25, 40.0):
        v = P.VectorField(g, scale * velocity_array(2, g))
        for order in ("cubic", "linear"):
            outs = {}
            for mode in (0, 1, 2):
                prev = lib.vr_set_trace_mode(mode)
                try:
                    t = P.TransportOperators(v, P.TransportConfig(4, order))
                    outs[mode] = [t.forward.displacement.clone(), t.backward.displacement.clone(),
                                  t.jac_factor.clone(), t.adj_factor.clone()]
                finally:
                    lib.vr_set_trace_mode(prev)
            torch.cuda.synchronize()
            for other in (1, 2):
                for x, y in zip(outs[0], outs[other]):
                    assert float((x - y).abs().max()) <= 4e-6 * max(float(x.abs().max()), 1.0), (order, scale, other)
