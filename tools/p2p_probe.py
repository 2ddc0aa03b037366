"""NVLink peer-copy bandwidth between GPU 0 and 1 (single process)."""
import torch
print("can_access_peer", torch.cuda.can_device_access_peer(0, 1), torch.cuda.can_device_access_peer(1, 0))
for mb in (1, 4, 16, 64, 256):
    a = torch.empty(mb * 2**20 // 4, device="cuda:0")
    b = torch.empty_like(a, device="cuda:1")
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    s = torch.cuda.Stream(device=0)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(10):
            b.copy_(a, non_blocking=True)
        e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{mb:4d} MB: {ms*1e3:8.1f} us  {mb*2**20/(ms*1e-3)/1e9:7.1f} GB/s", flush=True)
