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


@pytest.mark.parametrize("case", ["case_ops_match_single", "case_gn32", "case_c2_64"])
def test_slab_world1(case):
    spawn(case, 1)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (gpurun --gpus 2)")
@pytest.mark.parametrize("case", ["case_gn32", "case_c2_64"])
def test_slab_world2(case):
    spawn(case, 2)
