"""x1-slab decomposition on the GPU (NCCL).

* world 1 (any box): the slab kernels, self-halo and distributed-FFT path must
  reproduce the single-domain path and the reference trajectories;
* world 2 (boxes with >= 2 GPUs, e.g. `gpurun --gpus 2`): a real two-rank
  registration against the live-reference golden trajectory and Dice.
"""
import os
import socket

import numpy as np
import pytest
import torch

from conftest import golden_json, golden_npz

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    tdist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        globals()[case](rank, world)
        q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        tdist.destroy_process_group()


def spawn(case, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, "\n".join(r[1] for r in bad)


def _check(diag, gold, rtol=1e-3):
    assert [r.pcg_iterations for r in diag.iterations] == gold["pcg"]
    np.testing.assert_allclose([r.objective for r in diag.iterations], gold["objective"], rtol=rtol)
    assert abs(diag.relative_residual / gold["relative_residual"] - 1) < rtol
    assert abs(diag.j_min / gold["j_min"] - 1) < rtol and abs(diag.j_max / gold["j_max"] - 1) < rtol
    assert diag.termination_reason == gold["reason"]


def case_ops_match_single(rank, world):
    """slab operators (world=1: self halo, P=1 transposes) == single-domain operators"""
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import dist, _lib
    from paper_2209_08189_b200.synth import velocity_array
    n = 64
    g = P.make_grid((n, n, n))
    rng = np.random.default_rng(0)
    f = rng.random((n, n, n)).astype(np.float32)
    w = rng.standard_normal((3, n, n, n)).astype(np.float32)
    v = (0.3 * velocity_array(2, g)).astype(np.float32)
    outs = {}
    for tag in ("single", "slab"):
        ctxm = dist.activate(dist.SlabContext(g.dims)) if tag == "slab" else dist.activate(None)
        with ctxm:
            ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
            tops = P.TransportOperators(P.VectorField(g, v), P.TransportConfig(4, "cubic"))
            outs[tag] = [P.apply_A(P.VectorField(g, w), ops).numpy(),
                         P.apply_K(P.VectorField(g, w), ops).numpy(),
                         P.apply_inv_shifted_A(P.VectorField(g, w), ops, 1.0).numpy(),
                         P.fd8_gradient(P.ScalarField(g, f)).numpy(),
                         P.solve_state(P.ScalarField(g, f), tops.v, tops.cfg, tops).numpy(),
                         tops.adj_factor.cpu().numpy(),
                         np.array([P.h1_energy(P.ScalarField(g, f), ops.workspace)])]
    for a, b in zip(outs["single"], outs["slab"]):
        np.testing.assert_allclose(a, b, rtol=2e-6, atol=2e-6 * np.abs(a).max())


def case_gn32(rank, world):
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import dist
    gold = golden_json("gn_32.json")["runs"]["cubic_bw0.0001"]
    arr = golden_npz("gn_32.npz")
    g = P.make_grid((32, 32, 32))
    ctx = dist.SlabContext(g.dims)
    sl = slice(ctx.x0, ctx.x0 + ctx.L1)
    with dist.activate(ctx):
        cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=1e-4, n_t=4, interp_order="cubic")
        v, diag = P.gauss_newton_register(P.ScalarField(g, arr["m0_cubic"][sl]), P.ScalarField(g, arr["m1_cubic"][sl]),
                                          cfg)
    _check(diag, gold)


def case_c2_64(rank, world):
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import dist
    from paper_2209_08189_b200.synth import c2_problem
    gold = golden_json("c2_64.json")
    g = P.make_grid((64, 64, 64))
    with dist.activate(dist.SlabContext(g.dims)):
        m0, m1, l0, l1, _ = c2_problem(g)
        res = P.register(m0, m1, P.RegistrationConfig(beta_v=1e-2, n_t=4, interp_order="cubic"), labels0=l0,
                         labels1=l1, pre_dice=True)
    assert [r.pcg_iterations for r in res.diagnostics.iterations] == gold["run"]["pcg"]
    assert abs(res.relative_residual / gold["run"]["relative_residual"] - 1) < 1e-3
    assert abs(res.dice_pre.d_a - gold["dice_pre"]) < 0.005
    assert abs(res.dice.d_a - gold["dice_post"]) < 0.005


def _dist_vs_single(rank, world, n, order):
    _dist_vs_single_dims(rank, world, (n, n, n), order, 1e-4)


def _dist_vs_single_dims(rank, world, dims, order, beta_w):
    """Every operator and a full C2 registration on x1 slabs against the
    single-domain result on the same GPU (identical float32 inputs, made on
    the device): global relative L2 <= 1e-6 per operator (allreduced), PCG
    counts identical, objective / residual / J extrema / Dice within 1e-6."""
    import torch.distributed as tdist
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import dist
    from paper_2209_08189_b200.synth import c2_problem_device
    g = P.make_grid(dims)
    n = "x".join(map(str, dims))
    cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=beta_w, n_t=4, interp_order=order)
    m0, m1, l0, l1, vtrue = c2_problem_device(g, order, 4)
    gen = torch.Generator(device="cuda").manual_seed(9)
    w = 0.1 * torch.randn((3,) + g.dims, device="cuda", generator=gen)
    v = P.VectorField(g, 0.5 * vtrue.data)

    def ops_list(vv, ww, mm0, mm1, ctx):
        ops = P.RegOperators.for_grid(g, cfg.beta_v, cfg.beta_w)
        W = P.VectorField(g, ww)
        st = P.ObjectiveState(mm0, mm1, vv, cfg, ops)
        return {"A": P.apply_A(W, ops).data, "K": P.apply_K(W, ops).data,
                "invshift": P.apply_inv_shifted_A(W, ops, 1.0).data,
                "grad_m0": P.fd8_gradient(mm0).data, "div_v": P.fd8_divergence(vv).values,
                "disp_fwd": st.transport_ops.forward.displacement, "disp_bwd": st.transport_ops.backward.displacement,
                "state": st.m_series[-1], "adjoint": st.lambda_series[0], "gradient": st.gradient.data,
                "matvec": P.hessian_matvec(W, st).data, "objective": torch.tensor([st.objective], device="cuda")}

    single = ops_list(v, w, m0, m1, None)
    ref = P.register(m0, m1, cfg, labels0=l0, labels1=l1)
    ctx = dist.SlabContext(g.dims)
    sl = slice(ctx.x0, ctx.x0 + ctx.L1)
    with dist.activate(ctx):
        def loc(x):
            return x[..., sl, :, :].contiguous()
        V = P.VectorField(g, loc(v.data))
        M0, M1 = P.ScalarField(g, loc(m0.values)), P.ScalarField(g, loc(m1.values))
        slab = ops_list(V, loc(w), M0, M1, ctx)
        res = P.register(M0, M1, cfg, labels0=P.LabelMap(g, loc(l0.labels)), labels1=P.LabelMap(g, loc(l1.labels)))
    errs = {}
    for k, a in slab.items():
        b = single[k] if k == "objective" else single[k][..., sl, :, :]
        nd = torch.tensor([float(torch.sum((a.double() - b.double()) ** 2)), float(torch.sum(b.double() ** 2))],
                          dtype=torch.float64, device="cuda")
        if k != "objective":
            tdist.all_reduce(nd)
        errs[k] = float((nd[0] / nd[1]).sqrt())
    bad = {k: e for k, e in errs.items() if not e <= 1e-6}
    assert not bad, (rank, errs)
    d0, d1 = ref.diagnostics, res.diagnostics
    assert [r.pcg_iterations for r in d0.iterations] == [r.pcg_iterations for r in d1.iterations]
    assert d0.termination_reason == d1.termination_reason
    for a, b in ((d0.relative_residual, d1.relative_residual), (d0.j_min, d1.j_min), (d0.j_max, d1.j_max),
                 (d0.iterations[-1].objective, d1.iterations[-1].objective), (ref.dice.d_a, res.dice.d_a)):
        assert abs(a / b - 1) < 1e-6, (a, b)
    if rank == 0:
        print(f"dist-vs-single n={n} {order} world={world}: max operator rel L2 {max(errs.values()):.2e} "
              f"({max(errs, key=errs.get)}); PCG {[r.pcg_iterations for r in d1.iterations]}; residual "
              f"{d1.relative_residual:.9e} vs {d0.relative_residual:.9e}; Dice {res.dice.d_a:.9f}", flush=True)


def case_parity_512(rank, world):
    _dist_vs_single(rank, world, 512, "linear")


def case_parity_clarity(rank, world):
    """C5's CLARITY shape reduced with its prime factors kept: 88 x 104 x 166
    (2816 = 2^8 11, 3016 = 2^3 13 29, 1162 = 2 7 83 -> 11, 13, 83 here): the
    generic mixed-radix engine on x1 slabs, linear interpolation and
    beta_w = 1e-5 as C5."""
    _dist_vs_single_dims(rank, world, (88, 104, 166), "linear", 1e-5)


def case_parity_256(rank, world):
    _dist_vs_single(rank, world, 256, "cubic")


def case_sep_a_bitwise(rank, world):
    """A on the distributed separable engine (vr_dspec_a_*) equals the
    single-GPU separable operator bit for bit (same line transforms, same
    roundings of the partial sums), at 256^3 (block x1 lines of 256) and on
    the weak-scaling shape (x1 lines of 256 world)."""
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import dist, _lib
    for dims in ((256, 256, 256), (256 * world, 256, 256)):
        g = P.make_grid(dims)
        gen = torch.Generator(device="cuda").manual_seed(3)
        w = torch.randn((3,) + dims, device="cuda", generator=gen)
        add = torch.randn((3,) + dims, device="cuda", generator=gen)
        ops = P.RegOperators.for_grid(g, 1e-2, 0.0)
        ref = ops.workspace.apply(_lib.SPEC_A, w, add=add, alpha=1e-2)
        ctx = dist.SlabContext(g.dims)
        sl = slice(ctx.x0, ctx.x0 + ctx.L1)
        with dist.activate(ctx):
            ops_s = P.RegOperators.for_grid(g, 1e-2, 0.0)
            ws = ops_s.workspace
            assert ws.sep_a, "distributed separable A not selected"
            got = ws.apply(_lib.SPEC_A, w[:, sl].contiguous(), add=add[:, sl].contiguous(), alpha=1e-2)
        assert torch.equal(got, ref[:, sl]), (dims, float((got - ref[:, sl]).abs().max()))


def case_parity_weak(rank, world):
    """The weak-scaling bench shape (256 world, 256, 256): x1 lines of 512 /
    1024 on the transposed block (separable A's long x1 pass, xdiag_long)."""
    _dist_vs_single_dims(rank, world, (256 * world, 256, 256), "cubic", 1e-4)


@pytest.mark.parametrize("case", ["case_ops_match_single", "case_gn32", "case_c2_64"])
def test_slab_world1(case):
    spawn(case, 1)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (gpurun --gpus 2)")
@pytest.mark.parametrize("case", ["case_gn32", "case_c2_64"])
def test_slab_world2(case):
    spawn(case, 2)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (gpurun --gpus 2)")
@pytest.mark.parametrize("case", ["case_parity_256", "case_parity_512", "case_parity_clarity", "case_parity_weak",
                                  "case_sep_a_bitwise"])
def test_dist_vs_single_world2(case):
    spawn(case, 2)


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs (gpurun --gpus 4)")
@pytest.mark.parametrize("case", ["case_parity_256", "case_parity_512", "case_parity_clarity", "case_parity_weak",
                                  "case_sep_a_bitwise"])
def test_dist_vs_single_world4(case):
    spawn(case, 4)
