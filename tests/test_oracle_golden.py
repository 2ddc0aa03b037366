"""Pin the CPU oracle (oracle/velreg_oracle.py) against golden vectors produced
by the LIVE reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import golden_json, golden_npz, rel_l2
from oracle import velreg_oracle as O

TOL = 1e-6   # oracle vs reference, both f64 (fixtures stored as f32 -> ~6e-8)


def test_interp(ops_fx):
    fx = ops_fx
    for order in ("linear", "cubic"):
        pts = fx[f"trace_fwd_{order}"].astype(np.float64)
        for src in ("smooth", "rand"):
            vals = fx[f"f_{src}"].astype(np.float64)
            got = O.interp(vals, pts, order)
            assert rel_l2(got, fx[f"interp_{order}_{src}_trace"]) < TOL
            got = O.interp(vals, fx["pts_rand"].astype(np.float64), order)
            assert rel_l2(got, fx[f"interp_{order}_{src}_rand"]) < TOL


def test_trace(ops_fx):
    v = ops_fx["v"].astype(np.float64)
    for order in ("linear", "cubic"):
        assert np.abs(O.trace(v, 0.25, order) - ops_fx[f"trace_fwd_{order}"]).max() < 2e-6
        assert np.abs(O.trace(-v, 0.25, order) - ops_fx[f"trace_bwd_{order}"]).max() < 2e-6


def test_fd8(ops_fx):
    f = ops_fx["f_rand"]
    assert rel_l2(O.grad(f.astype(np.float64)), ops_fx["fd8_grad"]) < TOL
    # float32 evaluation is bit-identical to the reference's float32 evaluation
    np.testing.assert_array_equal(O.grad(f), ops_fx["fd8_grad_f32"])
    w = ops_fx["w"]
    np.testing.assert_array_equal(O.div(w), ops_fx["fd8_div_f32"])
    assert rel_l2(O.div(w.astype(np.float64)), ops_fx["fd8_div"]) < TOL


def test_spectral(ops_fx):
    v = ops_fx["v"].astype(np.float64)
    w = ops_fx["w"].astype(np.float64)
    assert rel_l2(O.op_A(v), ops_fx["apply_A_v"]) < TOL
    assert rel_l2(O.op_A(w), ops_fx["apply_A_w"]) < TOL
    assert rel_l2(O.op_inv_shifted(w, 1e-2, 1.0), ops_fx["inv_shifted_A_w_1"]) < TOL
    assert rel_l2(O.op_inv_shifted(w, 1e-2, 0.37), ops_fx["inv_shifted_A_w_037"]) < TOL
    assert rel_l2(O.op_K(w, 1e-2, 1e-4), ops_fx["apply_K_w"]) < TOL
    assert rel_l2(O.op_K(w, 1e-2, 3.0), ops_fx["apply_K_w_bw3"]) < TOL
    assert abs(O.h1(O.div(v)) / float(ops_fx["h1_energy_divv"]) - 1) < 1e-12
    assert abs(O.h1(ops_fx["f_rand"].astype(np.float64)) / float(ops_fx["h1_energy_frand"]) - 1) < 1e-12


def test_transport(ops_fx):
    v = ops_fx["v"].astype(np.float64)
    vt = ops_fx["vt"].astype(np.float64)
    f = ops_fx["f_smooth"].astype(np.float64)
    lam = ops_fx["f_rand"].astype(np.float64) - 0.5
    for order in ("linear", "cubic"):
        tr = O.Transport(v, 4, order)
        assert rel_l2(tr.jac_numer / tr.jac_denom,
                      ops_fx[f"jac_numer_{order}"] / ops_fx[f"jac_denom_{order}"]) < TOL
        assert rel_l2(tr.adj_numer / tr.adj_denom,
                      ops_fx[f"adj_numer_{order}"] / ops_fx[f"adj_denom_{order}"]) < TOL
        s = tr.state_series(f)
        assert rel_l2(s, ops_fx[f"state_series_{order}"]) < TOL
        assert rel_l2(tr.adjoint_series(lam), ops_fx[f"adjoint_series_{order}"]) < TOL
        gs = np.stack([O.grad(s[j]) for j in range(5)])
        assert rel_l2(tr.incremental(gs, vt), ops_fx[f"incstate_{order}"]) < TOL
        assert rel_l2(tr.jacobian(v), ops_fx[f"jacobian_{order}"]) < TOL


def test_objective_gradient_matvec(ops_fx):
    v = 0.5 * ops_fx["v"].astype(np.float64)
    w = ops_fx["w"].astype(np.float64)
    for order in ("cubic", "linear"):
        m0, m1 = ops_fx[f"obj_m0_{order}"], ops_fx[f"obj_m1_{order}"]
        for bw in (0.0, 1e-4):
            tag = f"{order}_bw{bw:g}"
            pb = O.Problem(m0, m1, v, beta_v=1e-2, beta_w=bw, n_t=4, order=order)
            assert abs(pb.objective() / float(ops_fx[f"objective_{tag}"]) - 1) < 1e-6
            assert rel_l2(pb.gradient(), ops_fx[f"gradient_{tag}"]) < TOL
            assert rel_l2(pb.matvec(w), ops_fx[f"matvec_{tag}"]) < TOL


def test_labels(ops_fx):
    v = ops_fx["v"].astype(np.float64)
    lab0 = ops_fx["labels0"]
    for order in ("cubic", "linear"):
        moved = O.transport_labels(lab0, O.Transport(v, 4, order))
        np.testing.assert_array_equal(moved, ops_fx[f"labels_moved_{order}"])
        assert abs(O.dice_average(moved, lab0) - float(ops_fx[f"dice_avgs_{order}"][0])) < 1e-6


@pytest.mark.parametrize("name,tag", [("32", "cubic_bw0"), ("32", "linear_bw0.0001"),
                                      ("16x20x24", "linear_bw0.0001")])
def test_gn_trajectory(name, tag):
    """Full Gauss-Newton solves: objective per iteration, PCG counts, residual."""
    gold = golden_json(f"gn_{name}.json")["runs"][tag]
    arr = golden_npz(f"gn_{name}.npz")
    order = tag.split("_")[0]
    bw = float(tag.split("bw")[1])
    v, rec = O.gauss_newton(arr[f"m0_{order}"], arr[f"m1_{order}"], beta_w=bw, order=order)
    assert rec["pcg"] == gold["pcg"]
    np.testing.assert_allclose(rec["objective"], gold["objective"], rtol=1e-8)
    assert abs(rec["relative_residual"] / gold["relative_residual"] - 1) < 1e-6
    assert rec["reason"] == gold["reason"]
