"""2-rank debug of the fused-transpose spectral path (torchrun --nproc-per-node 2)."""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as tdist


def main():
    rank = int(os.environ["RANK"]); torch.cuda.set_device(rank)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200 import dist
    n = int(os.environ.get("N", "256"))
    g = P.make_grid((n, n, n))
    ctx = dist.SlabContext(g.dims)
    gen = torch.Generator(device="cuda").manual_seed(1)
    w = torch.randn((3,) + g.dims, device="cuda", generator=gen)
    ref = {}
    ops1 = P.RegOperators.for_grid(g, 1e-2, 1e-4)
    sl = slice(ctx.x0, ctx.x0 + ctx.L1)
    for name, fn in (("A", lambda o, W: P.apply_A(W, o).data), ("inv", lambda o, W: P.apply_inv_shifted_A(W, o, 1.0).data),
                     ("K", lambda o, W: P.apply_K(W, o).data)):
        ref[name] = fn(ops1, P.VectorField(g, w))[:, sl].clone()
    with dist.activate(ctx):
        ops = P.RegOperators.for_grid(g, 1e-2, 1e-4)
        W = P.VectorField(g, w[:, sl].contiguous())
        for name, fn in (("A", lambda o, W: P.apply_A(W, o).data), ("inv", lambda o, W: P.apply_inv_shifted_A(W, o, 1.0).data),
                         ("K", lambda o, W: P.apply_K(W, o).data)):
            try:
                out = fn(ops, W)
                torch.cuda.synchronize()
                err = float(torch.linalg.vector_norm(out - ref[name]) / torch.linalg.vector_norm(ref[name]))
                print(f"rank {rank} {name}: rel err {err:.3e}", flush=True)
            except Exception:
                print(f"rank {rank} {name}: FAILED\n{traceback.format_exc()}", flush=True)
                raise
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
