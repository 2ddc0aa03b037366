"""Host-side logic added in round 2 (no GPU): slab-context routing, ghost
widths from departure displacements, SYN host utilities against the live
reference, and the volume container's header validation."""
import math

import numpy as np
import pytest

import paper_2209_08189_b200 as P
from paper_2209_08189_b200 import dist


def test_slab_routing_helpers():
    ctx = dist.SlabContext((32, 16, 8), rank=1, world=4)
    assert dist.for_grid((32, 16, 8)) is None           # nothing active
    with dist.activate(ctx):
        assert dist.for_grid((32, 16, 8)) is ctx
        assert dist.for_grid((16, 16, 8)) is None       # another grid stays single-domain
        assert dist.for_shape((3, 8, 16, 8)) is ctx      # a local slab (L1 = 8)
        assert dist.for_shape((8, 16, 8)) is ctx
        assert dist.for_shape((32, 16, 8)) is None       # a full field of the same grid
        assert dist.for_shape((4, 4)) is None


def test_ghost_width_for_displacement():
    # cubic stencil reaches base-1 .. base+2: |d| <= w - 1 keeps it inside w ghosts
    assert dist.ghost_width_for_displacement(3.0, "cubic") == 4
    assert dist.ghost_width_for_displacement(3.2, "cubic") == 5
    assert dist.ghost_width_for_displacement(3.2, "linear") == 4
    assert dist.ghost_width_for_displacement(0.0, "cubic") == 1


def test_synth_host_utilities_match_reference():
    from oracle import ref_arm
    V, _ = ref_arm.load()
    if V is None:
        pytest.skip("live reference not available")
    x = np.linspace(-1, 1, 41)
    for l, m in ((8, 6), (5, 2), (3, 0), (4, 4)):
        np.testing.assert_array_equal(P.assoc_legendre(l, m, x), V.assoc_legendre(l, m, x))
    phi = np.linspace(0, math.pi, 17)
    np.testing.assert_array_equal(P.spherical_harmonic_magnitude(8, 6, 0.3, phi),
                                  V.spherical_harmonic_magnitude(8, 6, 0.3, phi))
    with pytest.raises(ValueError):
        P.assoc_legendre(2, 3, 0.0)
    with pytest.raises(ValueError):
        P.SynthSpec(P.make_grid((8, 8, 8)), num_shapes=0)


def test_syn_random_stream_is_the_references():
    """_syn_shapes draws (centre, two quarter turns) per shape from
    default_rng(seed) in the reference's order (synth.py:88-92)."""
    from paper_2209_08189_b200.synth import _syn_shapes, OFFSET_BOUND, QUARTER_TURNS
    spec = P.SynthSpec(P.make_grid((8, 8, 8)), num_shapes=3, seed=11)
    rows = _syn_shapes(spec)
    rng = np.random.default_rng(11)
    for r in rows:
        c = rng.uniform(-OFFSET_BOUND, OFFSET_BOUND, size=3)
        rng.integers(0, 4)
        ph = QUARTER_TURNS[rng.integers(0, 4)]
        np.testing.assert_array_equal(r[:3], c)
        assert r[3] == ph


def test_volio_header_validation(tmp_path):
    with pytest.raises(P.VolumeIOError):
        P.load_volume(tmp_path / "missing")
    (tmp_path / "a.hdr").write_text("dims: 4 4 4\ndtype: f32\nkind: scalar\nlayout: col-major\n")
    (tmp_path / "a.raw").write_bytes(b"\0" * 256)
    with pytest.raises(P.VolumeIOError):
        P.load_volume(tmp_path / "a")
    (tmp_path / "b.hdr").write_text("dims: 4 4 4\ndtype: f16\nkind: scalar\nlayout: row-major-x1-outer\n")
    (tmp_path / "b.raw").write_bytes(b"\0" * 128)
    with pytest.raises(P.VolumeIOError):
        P.load_volume(tmp_path / "b")
    (tmp_path / "c.hdr").write_text("dims: 4 4 4\ndtype: f32\n")
    (tmp_path / "c.raw").write_bytes(b"\0" * 256)
    with pytest.raises(P.VolumeIOError):
        P.load_volume(tmp_path / "c")
    with pytest.raises(P.VolumeIOError):
        P.load_nifti(tmp_path / "nothing.nii")
    short = tmp_path / "short.nii"
    short.write_bytes(b"\0" * 100)
    with pytest.raises(P.VolumeIOError):
        P.load_nifti(short)
