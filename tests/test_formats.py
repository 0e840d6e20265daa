"""PFM I/O (formats.py:17-66) against bytes written by the reference writer
(tests/golden/report.npz, oracle/make_golden.py)."""

import numpy as np

from conftest import load_golden


def test_pfm_bytes_match_reference(tmp_path):
    from paper_1909_07545_b200 import formats
    g = load_golden("report")
    formats.write_pfm(tmp_path / "a.pfm", g["d_gt"])
    formats.write_vector_pfm(tmp_path / "b.pfm", g["w_gt"], third=g["valid"])
    assert (tmp_path / "a.pfm").read_bytes() == g["pfm1"].tobytes()
    assert (tmp_path / "b.pfm").read_bytes() == g["pfm3"].tobytes()


def test_pfm_roundtrip(tmp_path):
    from paper_1909_07545_b200 import formats
    g = load_golden("report")
    (tmp_path / "r.pfm").write_bytes(g["pfm3"].tobytes())
    f, third = formats.read_vector_pfm(tmp_path / "r.pfm")
    np.testing.assert_array_equal(f, g["w_gt"].astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(third, g["valid"].astype(np.float64))
    (tmp_path / "s.pfm").write_bytes(g["pfm1"].tobytes())
    np.testing.assert_array_equal(formats.read_pfm(tmp_path / "s.pfm"),
                                  g["d_gt"].astype(np.float32))
