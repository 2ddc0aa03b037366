"""Measured HBM footprint per voxel of one registration.

    python tools/memory_plan.py [--size 256] [--nt 4] [--layout auto|stored|lean] [--order cubic]
    torchrun --nproc-per-node 2 ... tools/memory_plan.py --size 512      # x1 slabs

Runs C2's sphere problem (synth.c2_problem_device) through `register` and
reports, per rank, the torch allocator's peak (fields, PCG vectors, series)
and the device memory held outside it (spectral plans and scratch, peer
receive buffers, cuFFT-free engine workspaces) as
    device_used_after - device_used_before_torch - torch_reserved_after,
both in bytes per local voxel, then extrapolates them to C3 (1024^3 on 4
GPUs) and C5 (2816 x 3016 x 1162 on 8 GPUs) at the same bytes per voxel.
One JSON line per rank.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2209_08189_b200 as P  # noqa: E402
from paper_2209_08189_b200 import runtime  # noqa: E402
from paper_2209_08189_b200.synth import c2_problem_device  # noqa: E402

TARGETS = {"C3": ((1024, 1024, 1024), 4), "C5": ((2816, 3016, 1162), 8)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--nt", type=int, default=4)
    ap.add_argument("--order", default="cubic")
    ap.add_argument("--layout", default="auto")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    free0, total = torch.cuda.mem_get_info(dev)
    used0 = total - free0
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.distributed.init_process_group("nccl", device_id=dev)
    runtime.set_grad_layout(a.layout)
    from paper_2209_08189_b200 import dist as pdist
    g = P.make_grid((a.size,) * 3)
    act = pdist.activate(pdist.SlabContext(g.dims) if world > 1 else None)
    act.__enter__()
    m0, m1, l0, l1, vtrue = c2_problem_device(g, "linear", 16)
    del vtrue, l0, l1
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    base_alloc = torch.cuda.memory_allocated(dev)
    cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=1e-4, n_t=a.nt, interp_order=a.order)
    res = P.register(m0, m1, cfg)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated(dev) - base_alloc
    free1, _ = torch.cuda.mem_get_info(dev)
    outside = (total - free1) - used0 - torch.cuda.memory_reserved(dev)
    nloc = m0.values.numel()
    bpv_torch = peak / nloc
    bpv_lib = max(outside, 0) / nloc
    line = {"rank": rank, "world": world, "n": a.size, "n_t": a.nt, "order": a.order, "layout": a.layout,
            "local_voxels": nloc, "matvecs": res.diagnostics.matvecs,
            "torch_peak_gb": peak / 2 ** 30, "outside_torch_gb": outside / 2 ** 30,
            "bytes_per_voxel_torch": round(bpv_torch, 1), "bytes_per_voxel_outside": round(bpv_lib, 1),
            "device_total_gb": total / 2 ** 30}
    for name, (dims, gpus) in TARGETS.items():
        per = dims[0] * dims[1] * dims[2] / gpus
        line[f"{name}_per_gpu_gb"] = round(per * (bpv_torch + bpv_lib) / 2 ** 30, 1)
    print(json.dumps(line), flush=True)
    act.__exit__(None, None, None)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
