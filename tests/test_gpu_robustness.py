"""Robustness fixes from the round-1 review: misaligned pointers on
the staged sweeps, deferred non-finite flags matched by storage, NaN-aware
min / max, single-pass label validation, and the slab-context routing."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2209_08189_b200 as P
    assert torch.cuda.is_available()
    return P


def test_staged_sweep_misaligned_pointer_falls_back(P):
    """A 4-byte-aligned (not 16-byte-aligned) source must not reach cp.async.bulk:
    the sweep falls back to the direct gather and gives the same values."""
    from paper_2209_08189_b200 import _lib
    from paper_2209_08189_b200.transport import TransportOperators, TransportConfig, advect
    g = P.make_grid((32, 32, 64))
    v = P.VectorField(g, 0.2 * P.synth.make_velocity(2, g).data)
    tops = TransportOperators(v, TransportConfig(4, "cubic"))
    f = torch.rand(g.dims, device="cuda", dtype=torch.float32)
    ref = advect(f, tops.forward.displacement, "cubic")
    buf = torch.empty(f.numel() + 1, device="cuda", dtype=torch.float32)
    mis = buf[1:].view(g.dims)          # base pointer 4 bytes past a 256-byte boundary
    mis.copy_(f)
    assert mis.data_ptr() % 16 == 4
    out = advect(mis, tops.forward.displacement, "cubic")
    torch.cuda.synchronize()
    assert torch.equal(out, ref) or float((out - ref).abs().max()) < 1e-6


def test_deferred_flag_matched_by_storage(P):
    from paper_2209_08189_b200 import _lib
    flags = torch.zeros((3, 1), dtype=torch.int32, device="cuda")
    _lib.defer_check(flags[1], RuntimeError("x"))
    try:
        assert _lib.is_deferred(flags[1])            # a fresh view of the same word
        assert not _lib.is_deferred(flags[2])
    finally:
        _lib._deferred.clear()


def test_minmax_propagates_nan(P):
    from paper_2209_08189_b200.reductions import minmax
    from paper_2209_08189_b200.autoparam import in_bounds
    g = P.make_grid((16, 16, 16))
    j = torch.ones(g.dims, device="cuda")
    j[3, 4, 5] = float("nan")
    mn, mx, _, _ = minmax(j)
    assert math.isnan(mn) and math.isnan(mx)
    assert not in_bounds(P.ScalarField(g, j), 0.5)           # numpy semantics: NaN extrema fail
    assert not in_bounds(P.ScalarField(g, torch.full(g.dims, float("nan"), device="cuda")), 0.5)
    assert in_bounds(P.ScalarField(g, torch.ones(g.dims, device="cuda")), 0.5)


def test_label_range_and_validation(P):
    from paper_2209_08189_b200.reductions import label_range
    g = P.make_grid((16, 16, 16))
    a = torch.zeros(g.dims, dtype=torch.int32, device="cuda")
    a[1, 2, 3] = 7
    b = torch.full(g.dims, 2, dtype=torch.int32, device="cuda")
    assert list(label_range(a, b)) == [0, 7, 2, 2]
    lm = P.LabelMap(g, a)
    assert lm.max_id == 7 and lm.label_ids() == [7]
    bad = a.clone()
    bad[0, 0, 0] = -1
    with pytest.raises(P.GridError):
        P.LabelMap(g, bad)


def test_register_from_pinned_host_buffers(P):
    """register() takes pinned host tensors (async uploads, labels on a side
    stream) and gives the same answer as device inputs."""
    g = P.make_grid((32, 32, 32))
    m0, m1, l0, l1, _ = P.synth.c2_problem(g, "cubic", 4)
    cfg = P.RegistrationConfig()
    ref = P.register(m0, m1, cfg, labels0=l0, labels1=l1)
    h = [torch.from_numpy(x.numpy()).pin_memory() for x in (m0, m1)]
    hl = [torch.from_numpy(x.numpy()).pin_memory() for x in (l0, l1)]
    got = P.register(h[0], h[1], cfg, labels0=hl[0], labels1=hl[1])
    assert got.relative_residual == ref.relative_residual
    assert got.dice.d_a == ref.dice.d_a
    assert torch.equal(got.velocity.data, ref.velocity.data)
    # results read back into caller-owned pinned buffers during the label scoring
    hv = torch.empty((3,) + g.dims, dtype=torch.float32).pin_memory()
    hd = torch.empty(g.dims, dtype=torch.float32).pin_memory()
    got = P.register(h[0], h[1], cfg, labels0=hl[0], labels1=hl[1], out_host=(hv, hd))
    torch.cuda.current_stream().synchronize()
    assert torch.equal(hv, ref.velocity.data.cpu()) and torch.equal(hd, ref.deformed.values.cpu())
    assert got.dice.d_a == ref.dice.d_a
    with pytest.raises(P.GridError):
        P.register(h[0], h[1], cfg, out_host=(hd, hv))
