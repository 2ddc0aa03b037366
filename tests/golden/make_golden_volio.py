"""Volume-container fixtures written by the LIVE reference's volio
(velreg/volio.py:35-145): scalar (f32 and f64), vector and label volumes in the
native .hdr/.raw container, plus single-file NIfTI-1 volumes (int16, float32,
gzip) built from the format's header layout, with the voxel arrays the
reference reads back from each.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_volio.py
"""
import gzip
import os
import struct
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import velreg as V  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "volio")
DIMS = (12, 10, 8)


def nifti_bytes(arr_c: np.ndarray, code: int) -> bytes:
    """Single-file NIfTI-1: 348-byte header, 4 extension bytes, i-fastest voxels."""
    hdr = bytearray(348)
    struct.pack_into("<i", hdr, 0, 348)
    dim = [3, arr_c.shape[0], arr_c.shape[1], arr_c.shape[2], 1, 1, 1, 1]
    struct.pack_into("<8h", hdr, 40, *dim)
    struct.pack_into("<h", hdr, 70, code)
    struct.pack_into("<h", hdr, 72, arr_c.dtype.itemsize * 8)
    struct.pack_into("<f", hdr, 108, 352.0)
    hdr[344:348] = b"n+1\x00"
    return bytes(hdr) + b"\x00" * 4 + np.asfortranarray(arr_c).tobytes(order="F")


def main():
    os.makedirs(HERE, exist_ok=True)
    g = V.make_grid(DIMS)
    rng = np.random.default_rng(0)
    s32 = rng.standard_normal(DIMS).astype(np.float32)
    s64 = rng.standard_normal(DIMS)
    vec = rng.standard_normal((3,) + DIMS).astype(np.float32)
    lab = rng.integers(0, 6, DIMS).astype(np.int32)
    V.save_volume(os.path.join(HERE, "scalar32"), V.ScalarField(g, s32))
    V.save_volume(os.path.join(HERE, "scalar64"), V.ScalarField(g, s64))
    V.save_volume(os.path.join(HERE, "vector"), V.VectorField(g, vec))
    V.save_volume(os.path.join(HERE, "labels"), V.LabelMap(g, lab))
    i16 = rng.integers(-300, 300, DIMS).astype("<i2")
    f32 = rng.standard_normal(DIMS).astype("<f4")
    with open(os.path.join(HERE, "vol_i16.nii"), "wb") as fh:
        fh.write(nifti_bytes(i16, 4))
    with gzip.open(os.path.join(HERE, "vol_f32.nii.gz"), "wb") as fh:
        fh.write(nifti_bytes(f32, 16))
    u8 = rng.integers(0, 7, DIMS).astype("<u1")
    with open(os.path.join(HERE, "vol_u8.nii"), "wb") as fh:
        fh.write(nifti_bytes(u8, 2))
    with open(os.path.join(HERE, "bad_magic.nii"), "wb") as fh:
        b = bytearray(nifti_bytes(i16, 4))
        b[344:348] = b"xxxx"
        fh.write(bytes(b))
    # what the reference reads back (the expected arrays)
    exp = {
        "scalar32": V.load_volume(os.path.join(HERE, "scalar32")).values,
        "scalar64": V.load_volume(os.path.join(HERE, "scalar64")).values,
        "vector": V.load_volume(os.path.join(HERE, "vector")).data,
        "labels": V.load_volume(os.path.join(HERE, "labels")).labels,
        "nii_i16": V.load_nifti(os.path.join(HERE, "vol_i16.nii")).values,
        "nii_f32": V.load_nifti(os.path.join(HERE, "vol_f32.nii.gz")).values,
        "nii_u8_labels": V.load_nifti(os.path.join(HERE, "vol_u8.nii"), as_labels=True).labels,
    }
    np.savez_compressed(os.path.join(HERE, "expected.npz"), **exp)
    print({k: (v.dtype, v.shape) for k, v in exp.items()})


if __name__ == "__main__":
    main()
