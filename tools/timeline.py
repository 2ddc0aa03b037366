"""GPU timeline of one C2 registration (torch.profiler / CUPTI): kernel-busy
time vs span, and the largest idle gaps (host-side launch or sync stalls).

    python tools/timeline.py [--n 256] [--top 15]
    torchrun --nproc-per-node N ... tools/timeline.py     # x1 slabs, (256 N, 256, 256); rank 0 reports
"""
from __future__ import annotations

import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--top", type=int, default=15)
    args = ap.parse_args()
    import paper_2209_08189_b200 as P
    from paper_2209_08189_b200.synth import c2_problem
    from paper_2209_08189_b200 import dist as pdist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    g = P.make_grid((args.n * world, args.n, args.n))
    act = pdist.activate(pdist.SlabContext(g.dims) if world > 1 else None)
    act.__enter__()
    m0, m1, _, _, _ = c2_problem(g)
    cfg = P.RegistrationConfig(beta_v=1e-2, beta_w=0.0, n_t=4, interp_order="cubic")
    for _ in range(2):
        P.gauss_newton_register(m0, m1, cfg)
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        P.gauss_newton_register(m0, m1, cfg)
        torch.cuda.synchronize()
    if rank != 0:
        return
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    t1 = max(e.time_range.end for e in ev)
    busy = 0.0
    cur_s, cur_e = None, None
    gaps = []
    prev_name = None
    for e in ev:
        s, en = e.time_range.start, e.time_range.end
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
                gaps.append((s - cur_e, prev_name, e.name))
            cur_s, cur_e = s, en
        else:
            cur_e = max(cur_e, en)
        prev_name = e.name
    busy += cur_e - cur_s
    span = t1 - t0
    print(f"span {span / 1e3:.2f} ms  kernel-busy {busy / 1e3:.2f} ms  idle {(span - busy) / 1e3:.2f} ms "
          f"({100 * (span - busy) / span:.1f} %)  kernels {len(ev)}")
    agg = collections.Counter()
    cnt = collections.Counter()
    for gsz, a, b in gaps:
        key = (a[:50], b[:50])
        agg[key] += gsz
        cnt[key] += 1
    print("largest idle totals by (previous kernel -> next kernel):")
    for (a, b), tot in agg.most_common(args.top):
        print(f"  {tot / 1e3:8.3f} ms  x{cnt[(a, b)]:4d}  {a}  ->  {b}")
    tot = collections.Counter()
    for e in ev:
        tot[e.name[:70]] += e.time_range.elapsed_us()
    print("kernel time:")
    for name, us in tot.most_common(args.top):
        print(f"  {us / 1e3:8.3f} ms  {name}")


if __name__ == "__main__":
    main()
