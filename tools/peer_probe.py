"""2-rank timing of the peer transport pieces (torchrun --nproc-per-node 2):
ghost exchange (copy engine + flags), the fused-transpose spectral stages,
and the NCCL / copy-engine alternatives.  CUDA events on the launching stream."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as tdist


def tmed(fn, reps=20):
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        tdist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st); b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    rank = int(os.environ["RANK"]); torch.cuda.set_device(rank)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import dist, _lib
    n = int(os.environ.get("N", "256"))
    world = tdist.get_world_size()
    g = P.make_grid((n * world, n, n))
    ctx = dist.SlabContext(g.dims)
    res = {}
    x = torch.randn((3,) + ctx.local_dims, device="cuda")
    with dist.activate(ctx):
        for w in (4, 6):
            def ex():
                lo, hi, works = ctx.ghosts_async(x[0], w)
                ctx.finish(works)
            res[f"ghost_w{w}_peer"] = tmed(ex)
            mesh = ctx._mesh
            ctx._mesh = None
            os.environ["VR_PEER"] = "0"
            res[f"ghost_w{w}_nccl"] = tmed(ex)
            os.environ["VR_PEER"] = "1"
            ctx._mesh = mesh
        ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
        ws = ops.workspace
        W = x
        for kind, name in ((_lib.SPEC_A, "A"), (_lib.SPEC_INVSHIFT, "invshift")):
            kw = {} if name == "A" else {"beta_v": 1e-2, "shift": 1.0}
            ws.peer = True
            res[f"{name}_fused"] = tmed(lambda: ws.apply(kind, W, **kw))
            ws.peer = False
            res[f"{name}_copyengine_a2a"] = tmed(lambda: ws.apply(kind, W, **kw))
            ws.peer = True
        # the stages of one fused apply (invshift, component 0)
        lib, st = _lib.lib(), _lib.stream()
        rv, iv = ws._regions(0, 1, False)
        P_, me = ctx.world, ctx.rank
        n1, n2, n3 = g.dims
        res["stage_forward_peer"] = tmed(lambda: lib.vr_dspec_forward_peer(ws._pl, x.data_ptr(), 1, 0, P_, me,
                                                                           ws._dst(rv), st))
        res["stage_signal_wait"] = tmed(lambda: ws._wait(ws._signal()))
        res["stage_xpass_peer"] = tmed(lambda: lib.vr_dspec_xpass_peer(ws._px, _lib.SPEC_INVSHIFT, 1, 0, 1e-2, 0.0, 1.0,
                                                                       0.0, 1.0, n1 * n2 * n3, me * ctx.L2, n2,
                                                                       ctx.L1, rv.data_ptr(), P_, me, ws._dst(iv), st))
        res["stage_inverse_peer"] = tmed(lambda: lib.vr_dspec_inverse_peer(ws._pl, iv.data_ptr(), 1, P_, None,
                                                                           x.data_ptr(), st))
        res["stage_forward_packed"] = tmed(lambda: lib.vr_dspec_forward(ws._pl, x.data_ptr(), 1, 0, P_,
                                                                        ws.send.data_ptr(), st))
    if rank == 0:
        print(json.dumps({k: round(v, 4) for k, v in res.items()}), flush=True)
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
