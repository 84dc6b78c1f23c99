"""Legacy ASCII VTK output of meshes, fields and element densities
(vtk_io.py:1-96 of the reference).

``write_vtk`` / ``read_vtk`` keep the reference's signatures and write the
same bytes (DataFile Version 2.0, UNSTRUCTURED_GRID, 2D points padded with
z = 0, cell types 5 / 10, SCALARS ... double 1 with shortest round-trip
``repr`` values).  The rows are formatted with list joins instead of one
``fh.write`` per line.  ``write_solution_vtk`` is the device-side caller: it
takes CUDA tensors from the engine (the trial / solution field and the
per-element densities of ``fm_energy``) and writes the file the reference's
CLI writes for the benchmark solutions (cli.py:155-163, 188-196).
"""

from __future__ import annotations

import numpy as np

_CELL_TYPE = {3: 5, 4: 10}  # triangle, tetrahedron (vtk_io.py:7)


def _fmt(values) -> str:
    return "\n".join(map(repr, np.asarray(values, dtype=float).ravel().tolist()))


def write_vtk(path, points, cells, point_data=None, cell_data=None, title="femmin"):
    """Write an unstructured grid; 2D points are padded with z = 0
    (vtk_io.py:10-40)."""
    points = np.asarray(points, dtype=float)
    cells = np.asarray(cells, dtype=np.int64)
    if points.shape[1] == 2:
        points = np.column_stack([points, np.zeros(points.shape[0])])
    nv = cells.shape[1]
    if nv not in _CELL_TYPE:
        raise KeyError(nv)
    out = ["# vtk DataFile Version 2.0", f"{title}", "ASCII", "DATASET UNSTRUCTURED_GRID",
           f"POINTS {points.shape[0]} double"]
    out += [f"{x!r} {y!r} {z!r}" for x, y, z in points.tolist()]
    out.append(f"CELLS {cells.shape[0]} {cells.shape[0] * (nv + 1)}")
    pre = f"{nv} "
    out += [pre + " ".join(map(str, row)) for row in cells.tolist()]
    out.append(f"CELL_TYPES {cells.shape[0]}")
    ct = str(_CELL_TYPE[nv])
    out += [ct] * cells.shape[0]
    for kind, count, data in (("POINT_DATA", points.shape[0], point_data),
                              ("CELL_DATA", cells.shape[0], cell_data)):
        if data:
            out.append(f"{kind} {count}")
            for name, values in data.items():
                out += [f"SCALARS {name} double 1", "LOOKUP_TABLE default"]
                if np.asarray(values).size:
                    out.append(_fmt(values))
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")


def read_vtk(path):
    """Read back a legacy ASCII unstructured grid as written by
    :func:`write_vtk` (same contract as vtk_io.py:51-96: returns
    ``(points, cells, point_data, cell_data)``; 2D files come back with the
    z = 0 column).

    Token-stream parser: after the two header lines (version, title) the file
    is a sequence of keyword sections, each followed by a known number of
    numeric tokens, so the body is split once into tokens and walked with a
    cursor (sections may span or share lines)."""
    with open(path) as fh:
        fh.readline()  # "# vtk DataFile Version 2.0"
        fh.readline()  # title (free text)
        tok = fh.read().split()
    n_tok = len(tok)
    pos = 0
    points = np.zeros((0, 3))
    cells = np.zeros((0, 0), dtype=np.int64)
    data: dict[str, dict[str, np.ndarray]] = {"POINT_DATA": {}, "CELL_DATA": {}}
    section, count = None, 0

    def take(n):
        nonlocal pos
        if pos + n > n_tok:
            raise ValueError(f"{path}: truncated VTK file")
        out = tok[pos:pos + n]
        pos += n
        return out

    while pos < n_tok:
        key = take(1)[0]
        if key in ("ASCII", "DATASET"):
            if key == "DATASET":
                take(1)
        elif key == "POINTS":
            n, _ = take(2)
            points = np.asarray(take(3 * int(n)), dtype=float).reshape(int(n), 3)
        elif key == "CELLS":
            n, size = (int(x) for x in take(2))
            flat = np.asarray(take(size), dtype=np.int64)
            nv = int(flat[0]) if n else 0
            cells = flat.reshape(n, nv + 1)[:, 1:] if n else np.zeros((0, 0), dtype=np.int64)
        elif key == "CELL_TYPES":
            take(int(take(1)[0]))
        elif key in data:
            section, count = key, int(take(1)[0])
        elif key == "SCALARS":
            name, _dtype = take(2)
            ncomp = 1
            if pos < n_tok and tok[pos] != "LOOKUP_TABLE":
                ncomp = int(take(1)[0])
            if pos < n_tok and tok[pos] == "LOOKUP_TABLE":
                take(2)
            if section is None:
                raise ValueError(f"{path}: SCALARS outside POINT_DATA / CELL_DATA")
            vals = np.asarray(take(count * ncomp), dtype=float)
            data[section][name] = vals if ncomp == 1 else vals.reshape(count, ncomp)
        else:
            raise ValueError(f"{path}: unexpected VTK token {key!r}")
    return points, cells, data["POINT_DATA"], data["CELL_DATA"]


def write_solution_vtk(path, coords, conn, v, d, model=None, dm=None, b=None,
                       densities=None, point_fields=None, title="femmin"):
    """The benchmark solution files of the reference CLI (cli.py:155-163,
    188-196): points = the field reshaped (nn, d) when d = dim (deformed
    configuration), else the mesh coordinates with the field as point data;
    cell data "density" = the per-element energy densities.  ``v``,
    ``coords``, ``conn`` may be CUDA tensors; with ``dm`` (a DeviceMesh) and
    ``model`` the densities are evaluated on the GPU (fm_energy)."""
    import torch

    def host(x):
        return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)

    if densities is None and dm is not None and model is not None:
        dens = torch.empty(dm.ne, dtype=torch.float64, device="cuda")
        vd = v if isinstance(v, torch.Tensor) and v.is_cuda else torch.as_tensor(
            np.asarray(v, dtype=np.float64)).cuda()
        dm.energy(vd, model, b, densities=dens)
        densities = dens
    coords_h, conn_h, v_h = host(coords), host(conn), host(v).astype(float)
    dim = coords_h.shape[1]
    pdata = dict(point_fields or {})
    if d == dim:
        points = v_h.reshape(-1, d)
    else:
        points = coords_h
        pdata = {"u": v_h, **pdata}
    cdata = {"density": host(densities)} if densities is not None else None
    write_vtk(path, points, conn_h, point_data=pdata or None, cell_data=cdata, title=title)
