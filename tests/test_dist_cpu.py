"""Host-side logic of the x1-slab decomposition (dist.py) with the gloo
backend on CPU, world size 2 (and 4): ghost-plane exchange, the transpose
layout contract of the distributed FFT, and the cross-rank reductions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        tdist.destroy_process_group()


def spawn(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, bad


DIMS = (16, 8, 6)


def _global():
    return np.arange(np.prod(DIMS), dtype=np.float32).reshape(DIMS)


def _halo_case(rank, world):
    from paper_2209_08189_b200.dist import SlabContext
    ctx = SlabContext(DIMS)
    g = _global()
    loc = torch.from_numpy(g[ctx.x0:ctx.x0 + ctx.L1].copy())
    for w in (1, 3, ctx.L1):
        ext = ctx.halo(loc, w).numpy()
        idx = np.arange(ctx.x0 - w, ctx.x0 + ctx.L1 + w) % DIMS[0]
        np.testing.assert_array_equal(ext, g[idx])
    vec = torch.from_numpy(np.stack([g, 2 * g, -g])[:, ctx.x0:ctx.x0 + ctx.L1].copy())
    ext = ctx.halo(vec, 2).numpy()
    idx = np.arange(ctx.x0 - 2, ctx.x0 + ctx.L1 + 2) % DIMS[0]
    np.testing.assert_array_equal(ext, np.stack([g, 2 * g, -g])[:, idx])


def _transpose_case(rank, world):
    """pack([q][c][i][jl][kz]) -> ONE all-to-all -> [p][c][il][jl][kz], i.e. complete
    x1 lines x1 = p*L1 + il (the contract of vr_dspec_forward / vr_dspec_xpass /
    vr_dspec_inverse)."""
    from paper_2209_08189_b200.dist import SlabContext
    ctx = SlabContext(DIMS)
    n1, n2, n3h = DIMS
    spec = np.random.default_rng(0).standard_normal((3, n1, n2, n3h)).astype(np.float32)
    loc = spec[:, ctx.x0:ctx.x0 + ctx.L1]
    send = np.stack([loc[:, :, q * ctx.L2:(q + 1) * ctx.L2] for q in range(world)], axis=0)  # [q][c][i][jl][kz]
    send = torch.from_numpy(np.ascontiguousarray(send)).reshape(-1)
    recv = torch.empty_like(send)
    ctx.alltoall(recv, send)
    got = recv.reshape(world, 3, ctx.L1, ctx.L2, n3h).numpy()      # [p][c][il][jl][kz]
    want = spec[:, :, rank * ctx.L2:(rank + 1) * ctx.L2].reshape(3, world, ctx.L1, ctx.L2, n3h).transpose(1, 0, 2, 3, 4)
    np.testing.assert_array_equal(got, want)
    # inverse direction: the X pass output keeps that layout; blocks go back to their owners
    back = torch.empty_like(recv)
    ctx.alltoall(back, recv)
    got = back.reshape(world, 3, ctx.L1, ctx.L2, n3h).numpy()      # [q][c][i][jl][kz]
    np.testing.assert_array_equal(got, send.reshape(world, 3, ctx.L1, ctx.L2, n3h).numpy())


def _reduce_case(rank, world):
    from paper_2209_08189_b200.dist import SlabContext, ghost_width
    ctx = SlabContext(DIMS)
    np.testing.assert_allclose(ctx.allreduce([rank + 1.0, 2.0]), [world * (world + 1) / 2, 2.0 * world])
    assert ctx.allreduce([rank], "max")[0] == world - 1
    assert ctx.allreduce([rank], "min")[0] == 0
    # ghost width covers the largest x1 displacement plus the stencil
    assert ghost_width(0.0, 0.25, 256, "cubic") == 4
    assert ghost_width(0.341, 0.25, 256, "cubic") == int(np.ceil(0.25 * 0.341 / (2 * np.pi / 256))) + 3


@pytest.mark.parametrize("world", [2, 4])
def test_halo_gloo(world):
    spawn(_halo_case, world)


def test_transpose_gloo():
    spawn(_transpose_case, 2)


def test_reductions_gloo():
    spawn(_reduce_case, 2)


def test_slab_context_validation():
    from paper_2209_08189_b200.dist import SlabContext
    with pytest.raises(ValueError):
        SlabContext((10, 8, 8), rank=0, world=4)
    ctx = SlabContext((16, 8, 8), rank=1, world=2)
    assert ctx.local_dims == (8, 8, 8) and ctx.x0 == 8 and ctx.left == 0 and ctx.right == 0
