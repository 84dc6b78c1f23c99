"""the VTK output format, byte for byte against files
written by the reference's own writer (tests/golden/make_golden.py case_vtk)."""

import os

import numpy as np
import pytest

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


def test_report_csv_contract(tmp_path):
    """BenchmarkReport (reference bench.py:44-98): row-length check, exact
    float round trip through the CSV text and the file, table formatting."""
    from paper_2109_01158_b200.reports import BenchmarkReport
    rep = BenchmarkReport(benchmark="demo", columns=["level", "J", "name"])
    with pytest.raises(ValueError):
        rep.add_row(1)
    rep.add_row(1, 0.1 + 0.2, "run-a")
    rep.add_row(2, -8.16254321e7, "run-b")
    back = BenchmarkReport.from_csv_string("demo", rep.to_csv_string())
    assert back.columns == rep.columns and back.rows == rep.rows
    path = tmp_path / "r.csv"
    rep.to_csv(path)
    assert BenchmarkReport.from_csv("demo", path).rows == rep.rows
    assert rep.column("J") == [0.1 + 0.2, -8.16254321e7]
    table = rep.format_table()
    assert "level" in table and "run-b" in table and "0.3" in table


def test_report_csv_matches_reference_writer():
    """Same bytes as the reference's writer for the same rows."""
    import os
    import sys
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    sys.path.insert(0, ref)
    try:
        from femmin.bench import BenchmarkReport as RefReport
    finally:
        sys.path.remove(ref)
    from paper_2109_01158_b200.reports import BenchmarkReport
    rows = [(1, 0.1 + 0.2, "a"), (3, 6.425476e0, "b,c"), (7, float("inf"), "x")]
    a, b = BenchmarkReport("t", ["l", "J", "s"]), RefReport("t", ["l", "J", "s"])
    for r in rows:
        a.add_row(*r)
        b.add_row(*r)
    assert a.to_csv_string() == b.to_csv_string()
