"""the VTK output format, byte for byte against files
written by the reference's own writer (tests/golden/make_golden.py case_vtk)."""

import os

import numpy as np

from paper_2109_01158_b200 import vtk_io

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read(path):
    with open(path, "rb") as fh:
        return fh.read()


def test_vtk_bytes_2d_with_data(tmp_path):
    with np.load(os.path.join(GOLDEN, "vtk_lshape1_data.npz")) as z:
        d = {k: z[k] for k in z.files}
    out = tmp_path / "l.vtk"
    vtk_io.write_vtk(out, d["coords"], d["conn"], point_data={"u": d["u"]},
                     cell_data={"density": d["density"]})
    assert _read(out) == _read(os.path.join(GOLDEN, "vtk_lshape1.vtk"))
    pts, cells, pdata, cdata = vtk_io.read_vtk(out)
    assert pts.shape == (d["coords"].shape[0], 3) and (pts[:, 2] == 0).all()
    np.testing.assert_array_equal(cells, d["conn"])
    np.testing.assert_array_equal(pdata["u"], d["u"])
    np.testing.assert_array_equal(cdata["density"], d["density"])


def test_vtk_bytes_3d(tmp_path, golden):
    g = golden("bar1_nh")
    out = tmp_path / "b.vtk"
    vtk_io.write_vtk(out, g["coords"], g["conn"])
    assert _read(out) == _read(os.path.join(GOLDEN, "vtk_bar1.vtk"))
    lines = _read(out).decode().splitlines()
    i = lines.index(f"CELL_TYPES {g['conn'].shape[0]}")
    assert set(lines[i + 1:i + 1 + g["conn"].shape[0]]) == {"10"}
