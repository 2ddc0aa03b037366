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
