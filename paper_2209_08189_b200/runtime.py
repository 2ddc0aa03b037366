"""Process-wide switches (reference: /root/reference/pkg/src/velreg/runtime.py:8-17).

The reference's reproducible mode swaps in serial numba kernels so that write
and reduction order is fixed.  Every kernel here is already deterministic: each
voxel is written by exactly one thread and every reduction uses a fixed tree
(per-CTA partials folded in index order, no floating-point atomics), so the flag
is kept for API compatibility and changes nothing numerically -- exactly the
reference's observed behaviour (parallel and serial kernels are
bitwise equal).
"""

_reproducible = False


def set_reproducible(flag: bool) -> None:
    global _reproducible
    _reproducible = bool(flag)


def reproducible() -> bool:
    return _reproducible


# Memory layout of the grad-m series (optim.py:127-135 keeps (n_t+1) x 3 fields).
# "auto": store it unless it would take more than a third of the device memory
# not yet allocated by torch, otherwise recompute grad m^j per use (transport.LazyGradientSeries;
# results are bit-identical, FD8 is deterministic).  "stored" / "lean" force one.
import os as _os

_grad_layout = _os.environ.get("VR_GRAD_LAYOUT", "auto")


def set_grad_layout(mode: str) -> None:
    global _grad_layout
    if mode not in ("auto", "stored", "lean"):
        raise ValueError(f"unknown grad-m layout {mode!r}")
    _grad_layout = mode


def lean_layout(series_bytes: int, device) -> bool:
    if _grad_layout != "auto":
        return _grad_layout == "lean"
    import torch
    if device.type != "cuda":
        return False
    # allocator statistics, not cudaMemGetInfo (a driver round trip that costs
    # ~4 ms per call on B200 -- measured as idle gaps in tools/timeline.py)
    total = torch.cuda.get_device_properties(device).total_memory
    free = total - torch.cuda.memory_allocated(device)
    return series_bytes > free // 3
