"""Volume container / NIfTI I/O against files written by the
LIVE reference (tests/golden/make_golden_volio.py) and, both directions,
against the reference package installed in oracle/_ref (test infrastructure)."""
import os
import shutil

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
VOL = os.path.join(GOLDEN, "volio")


@pytest.fixture(scope="module")
def P():
    import paper_2209_08189_b200 as P
    assert torch.cuda.is_available()
    return P


@pytest.fixture(scope="module")
def exp():
    return np.load(os.path.join(VOL, "expected.npz"))


def test_load_reference_written_volumes(P, exp):
    s32 = P.load_volume(os.path.join(VOL, "scalar32"))
    np.testing.assert_array_equal(s32.values.cpu().numpy(), exp["scalar32"])
    s64 = P.load_volume(os.path.join(VOL, "scalar64.hdr"))
    np.testing.assert_array_equal(s64.values.cpu().numpy(), exp["scalar64"].astype(np.float32))
    vec = P.load_volume(os.path.join(VOL, "vector.raw"))
    np.testing.assert_array_equal(vec.data.cpu().numpy(), exp["vector"])
    lab = P.load_volume(os.path.join(VOL, "labels"))
    assert isinstance(lab, P.LabelMap)
    np.testing.assert_array_equal(lab.labels.cpu().numpy(), exp["labels"])


def test_load_nifti(P, exp):
    a = P.load_nifti(os.path.join(VOL, "vol_i16.nii"))
    np.testing.assert_array_equal(a.values.cpu().numpy(), exp["nii_i16"].astype(np.float32))
    b = P.load_nifti(os.path.join(VOL, "vol_f32.nii.gz"))
    np.testing.assert_array_equal(b.values.cpu().numpy(), exp["nii_f32"].astype(np.float32))
    c = P.load_nifti(os.path.join(VOL, "vol_u8.nii"), as_labels=True)
    np.testing.assert_array_equal(c.labels.cpu().numpy(), exp["nii_u8_labels"])
    with pytest.raises(P.VolumeIOError):
        P.load_nifti(os.path.join(VOL, "bad_magic.nii"))
    with pytest.raises(P.VolumeIOError):
        P.load_nifti(os.path.join(VOL, "missing.nii"))


def test_errors(P, tmp_path):
    with pytest.raises(P.VolumeIOError):
        P.load_volume(tmp_path / "nothing")
    shutil.copy(os.path.join(VOL, "scalar32.hdr"), tmp_path / "short.hdr")
    with open(tmp_path / "short.raw", "wb") as fh:
        fh.write(b"\0" * 100)
    with pytest.raises(P.VolumeIOError):
        P.load_volume(tmp_path / "short")
    (tmp_path / "lay.hdr").write_text("dims: 4 4 4\ndtype: f32\nkind: scalar\nlayout: col-major\n")
    (tmp_path / "lay.raw").write_bytes(b"\0" * 256)
    with pytest.raises(P.VolumeIOError):
        P.load_volume(tmp_path / "lay")


def test_round_trip_both_ways(P, tmp_path):
    """save_volume here -> the reference's load_volume, and a 128 MB field
    through the streamed (chunked) path."""
    from oracle import ref_arm
    V, _ = ref_arm.load()
    g = P.make_grid((12, 10, 8))
    gen = torch.Generator(device="cuda").manual_seed(2)
    v = P.VectorField(g, torch.randn((3, 12, 10, 8), device="cuda", generator=gen))
    P.save_volume(tmp_path / "v", v)
    if V is not None:
        back = V.load_volume(str(tmp_path / "v"))
        np.testing.assert_array_equal(back.data, v.data.cpu().numpy())
    lab = P.LabelMap(g, torch.randint(0, 9, (12, 10, 8), device="cuda", dtype=torch.int32, generator=gen))
    P.save_volume(tmp_path / "l", lab)
    assert torch.equal(P.load_volume(tmp_path / "l").labels, lab.labels)
    big = P.make_grid((128, 256, 256))   # 64 MB scalar > one 64 MB staging chunk with the vector below
    f = P.VectorField(big, torch.randn((3, 128, 256, 256), device="cuda", generator=gen))
    P.save_volume(tmp_path / "big", f)
    assert torch.equal(P.load_volume(tmp_path / "big").data, f.data)
