"""CSV benchmark reports (reference bench.py:44-98) and the
reference's hot-path benchmarks 1-3 on the B200 engine (bench.py:208-296).

``BenchmarkReport`` keeps the reference's file format and contract: a header
row of column names, one CSV row per ``add_row`` (length checked), floats
written with ``repr`` so that reading the file back returns the identical
values, and cells parsed back as int, then float, then str.  ``bench1`` -
``bench3`` produce the same columns as the reference's: mesh / patch setup
sizes and times, the twisted-bar energy, and exact vs numeric gradient times
with their agreement; the times are the GPU path's (best of ``repeats``
wall-clock calls through the numpy drop-in API).
"""

from __future__ import annotations

import csv
import io
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

BAR_LX, BAR_LY, BAR_LZ = 0.4, 0.01, 0.01  # bench.py:37 (the paper's bar)


def _cell(token: str):
    for conv in (int, float):
        try:
            return conv(token)
        except ValueError:
            pass
    return token


def _short(v) -> str:
    return f"{v:.6g}" if isinstance(v, float) else str(v)


@dataclass
class BenchmarkReport:
    """One benchmark's table (bench.py:44-98)."""

    benchmark: str
    columns: list
    rows: list = field(default_factory=list)
    config: dict = field(default_factory=dict)

    def add_row(self, *values):
        if len(values) != len(self.columns):
            raise ValueError("row length does not match the report columns")
        self.rows.append(list(values))

    def to_csv_string(self) -> str:
        out = io.StringIO()
        w = csv.writer(out, lineterminator="\n")
        w.writerow(self.columns)
        w.writerows([[repr(c) if isinstance(c, float) else c for c in r] for r in self.rows])
        return out.getvalue()

    def to_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            fh.write(self.to_csv_string())

    @classmethod
    def from_csv_string(cls, benchmark: str, text: str) -> "BenchmarkReport":
        table = list(csv.reader(io.StringIO(text)))
        rep = cls(benchmark=benchmark, columns=table[0] if table else [])
        rep.rows = [[_cell(t) for t in r] for r in table[1:]]
        return rep

    @classmethod
    def from_csv(cls, benchmark: str, path) -> "BenchmarkReport":
        with open(path, newline="") as fh:
            return cls.from_csv_string(benchmark, fh.read())

    def column(self, name):
        k = self.columns.index(name)
        return [r[k] for r in self.rows]

    def format_table(self) -> str:
        cells = [[str(c) for c in self.columns]] + [[_short(v) for v in r] for r in self.rows]
        width = [max(len(row[k]) for row in cells) for k in range(len(self.columns))]
        return "\n".join("  ".join(t.rjust(wd) for t, wd in zip(row, width)) for row in cells)


def _config(**extra):
    cfg = {"threads": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
           "engine": "B200 (paper_2109_01158_b200)"}
    cfg.update(extra)
    return cfg


def _best(fn, repeats):
    t_best, out = math.inf, None
    for _ in range(max(1, repeats)):
        t0 = time.perf_counter()
        out = fn()
        t_best = min(t_best, time.perf_counter() - t0)
    return t_best, out


def bar_problem(level: int):
    """bench.py:126-132: the paper's bar, both end faces clamped (d = 3)."""
    from . import DirichletRegion, DirichletSpec, generate_bar_mesh_3d, mark_dirichlet
    mesh = generate_bar_mesh_3d(BAR_LX, BAR_LY, BAR_LZ, level)
    ends = DirichletSpec([DirichletRegion(where=lambda x: x[:, 0] < 1e-9),
                          DirichletRegion(where=lambda x: x[:, 0] > BAR_LX - 1e-9)])
    return mark_dirichlet(mesh, ends, d=3)


def twist_map(alpha: float, lx: float = BAR_LX):
    """The bar's torsion (bench.py:140-149): the (y, z) section rotated by
    the angle alpha x / lx, clockwise in the (y, z) plane."""
    def fn(pts):
        ang = alpha * pts[:, 0] / lx
        cs, sn = np.cos(ang), np.sin(ang)
        y, z = pts[:, 1], pts[:, 2]
        return np.stack([pts[:, 0], cs * y + sn * z, -sn * y + cs * z], axis=1)
    return fn


def _bar_model():
    from . import ElasticParams, NeoHookean
    return NeoHookean(ElasticParams(E=2e8, nu=0.3), dim=3)


def bench1(levels) -> BenchmarkReport:
    """Mesh and patch setup: sizes and (GPU) build times (bench.py:208-244)."""
    from . import build_patches
    rep = BenchmarkReport("bench1", ["level", "nodes", "elements", "free_dofs", "patch_rows",
                                     "mesh_time_s", "patches_time_s", "mesh_entries",
                                     "patches_entries"], config=_config())
    for level in levels:
        t0 = time.perf_counter()
        mesh = bar_problem(level)
        t_mesh = time.perf_counter() - t0
        t0 = time.perf_counter()
        pt = build_patches(mesh)
        t_pt = time.perf_counter() - t0
        mesh_entries = (mesh.nodes2coord.size + mesh.elems2nodes.size + mesh.volumes.size
                        + sum(g.size for g in mesh.dphi))
        pt_entries = (pt.lengths.size + pt.elems.size + pt.volumes.size + pt.elems2nodes.size
                      + sum(g.size for g in pt.dphi) + pt.logical.size + pt.prefix.size)
        rep.add_row(level, mesh.nn, mesh.ne, int(mesh.dofs_minim.size), int(pt.total_rows),
                    t_mesh, t_pt, int(mesh_entries), int(pt_entries))
    return rep


def bench2(levels, repeats=10, alpha=2 * np.pi) -> BenchmarkReport:
    """Energy of the twisted bar (bench.py:247-262)."""
    from . import energy, interpolate
    rep = BenchmarkReport("bench2", ["level", "free_dofs", "energy_time_s", "J_grad"],
                          config=_config(repeats=repeats, alpha=alpha))
    model = _bar_model()
    for level in levels:
        mesh = bar_problem(level)
        v = interpolate(twist_map(alpha), mesh, d=3)
        t, (J, _) = _best(lambda: energy(v, mesh, model), repeats)
        rep.add_row(level, int(mesh.dofs_minim.size), t, J)
    return rep


def bench3(levels, repeats=10, eps=1e-6, alpha=2 * np.pi) -> BenchmarkReport:
    """Exact vs nodal-patch FD gradient: times and agreement (bench.py:265-296)."""
    from . import build_patches, exact_gradient, interpolate, numeric_gradient
    rep = BenchmarkReport("bench3", ["level", "free_dofs", "exact_time_s", "numeric_time_s",
                                     "rel_agreement"],
                          config=_config(repeats=repeats, eps=eps, alpha=alpha))
    if repeats <= 0:
        return rep
    model = _bar_model()
    for level in levels:
        mesh = bar_problem(level)
        pt = build_patches(mesh)
        v = interpolate(twist_map(alpha), mesh, d=3)
        te, ge = _best(lambda: exact_gradient(v, mesh, pt, model), repeats)
        tn, gn = _best(lambda: numeric_gradient(v, mesh, pt, model, eps=eps), repeats)
        rel = float(np.abs(ge - gn).max() / max(np.abs(ge).max(), 1e-300))
        rep.add_row(level, int(mesh.dofs_minim.size), te, tn, rel)
    return rep


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser(description="hot-path benchmarks 1-3 as CSV reports")
    ap.add_argument("bench", choices=["bench1", "bench2", "bench3"])
    ap.add_argument("--levels", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--repeats", type=int, default=10)
    ap.add_argument("--csv", default="")
    a = ap.parse_args()
    fn = {"bench1": lambda: bench1(a.levels), "bench2": lambda: bench2(a.levels, a.repeats),
          "bench3": lambda: bench3(a.levels, a.repeats)}[a.bench]
    r = fn()
    print(r.format_table())
    if a.csv:
        r.to_csv(a.csv)
