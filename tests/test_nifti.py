"""NIfTI-1 / raw + JSON IO (nifti.hpp:24-303) of paper_2509_25044_b200.nifti against files
the reference itself wrote and parsed (tests/golden/make_golden.py: nifti_fixtures).
CPU only."""
import os

import numpy as np
import pytest

from paper_2509_25044_b200 import nifti as N

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "nifti")


@pytest.mark.parametrize("name", ["vol_f32", "vol_f64", "labels", "vol_be", "scaled_i16"])
def test_read_matches_reference_parse(golden, name):
    nv = N.read_nifti(os.path.join(GOLD, name + ".nii"))
    assert np.array_equal(nv.volume, golden[f"nii_{name}"])
    assert np.array_equal(np.array(nv.spacing), golden[f"nii_{name}_spacing"])
    assert np.array_equal(np.array(nv.origin), golden[f"nii_{name}_origin"])
    assert nv.header.big_endian == (name == "vol_be")


@pytest.mark.parametrize("f64", [False, True])
def test_write_is_byte_identical_to_reference(golden, f64, tmp_path):
    v = golden["nii_src"].astype(np.float64 if f64 else np.float32)
    fn = os.path.join(GOLD, "vol_f64.nii" if f64 else "vol_f32.nii")
    out = tmp_path / "v.nii"
    N.write_nifti(v, str(out), golden["nii_src_spacing"], golden["nii_src_origin"])
    assert out.read_bytes() == open(fn, "rb").read()


def test_labels_round_trip(golden, tmp_path):
    lab = golden["nii_labels_src"].astype(np.uint16)
    out = tmp_path / "l.nii"
    N.write_labels(lab, str(out), golden["nii_src_spacing"])
    assert out.read_bytes() == open(os.path.join(GOLD, "labels.nii"), "rb").read()
    assert np.array_equal(N.nifti_to_labels(N.read_nifti(str(out))), lab)
    with pytest.raises(N.FormatError):
        N.nifti_to_labels(N.read_nifti(os.path.join(GOLD, "vol_f32.nii")))


def test_warp_round_trip(golden, tmp_path):
    """The reference reads back what it wrote; ours reads the reference's files and writes
    files with the same payload and sidecar content."""
    assert np.array_equal(N.read_warp(os.path.join(GOLD, "warp")), golden["warp_read"])
    N.write_warp(golden["warp_src"], str(tmp_path / "w"), golden["nii_src_spacing"], golden["nii_src_origin"])
    assert (tmp_path / "w.raw").read_bytes() == open(os.path.join(GOLD, "warp.raw"), "rb").read()
    import json
    assert json.load(open(tmp_path / "w.json")) == json.load(open(os.path.join(GOLD, "warp.json")))
    assert np.array_equal(N.read_warp(str(tmp_path / "w")), golden["warp_read"])


def test_format_errors(tmp_path):
    """The reference's FormatError / IoError cases (nifti.hpp:100-166, 178-184)."""
    good = open(os.path.join(GOLD, "vol_f32.nii"), "rb").read()
    with pytest.raises(N.FormatError):
        N.read_nifti_bytes(good[:100])  # shorter than the header
    bad = bytearray(good)
    bad[0:4] = b"\x01\x02\x03\x04"
    with pytest.raises(N.FormatError):
        N.read_nifti_bytes(bytes(bad))  # sizeof_hdr
    bad = bytearray(good)
    bad[344:348] = b"ni1\0"
    with pytest.raises(N.FormatError, match="two-file"):
        N.read_nifti_bytes(bytes(bad))
    bad = bytearray(good)
    bad[344:348] = b"abc\0"
    with pytest.raises(N.FormatError, match="bad magic"):
        N.read_nifti_bytes(bytes(bad))
    bad = bytearray(good)
    bad[70:72] = (8).to_bytes(2, "little")
    with pytest.raises(N.FormatError, match="datatype"):
        N.read_nifti_bytes(bytes(bad))
    with pytest.raises(N.FormatError, match="truncated"):
        N.read_nifti_bytes(good[:-8])
    with pytest.raises(N.IoError):
        N.read_nifti(str(tmp_path / "missing.nii"))
    with pytest.raises(ValueError):
        N.write_nifti(np.zeros((2, 3, 40000), np.float32), str(tmp_path / "big.nii"))
