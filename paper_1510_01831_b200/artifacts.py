"""Formats around the online path: velocity-model files and offline artifacts.

* ``save_model`` / ``load_model``: the reference's model files (``discretization.py:509-560``): a JSON
  header plus raw little-endian float64 (extended grid, depth-major), or a tiny headered CSV.
* ``cache_key``: the reference's hash of one offline stage (``green.py:182-189``).
* ``dump_offline`` / ``load_offline``: persistence of the offline stage this path uploads.  The Green
  blocks are written in the reference's ``GreenBlockSet.dump`` format (``green.py:156-169``; readable by
  ``GreenBlockSet.load``), one set per (layer, cell), with a manifest like ``dump_offline``
  (``nested.py:489-504``); the complete factor set (Schur inverses, couplings, pass-0 and sampled-response
  operators, dense or direct inner operators) goes into one ``factors_<key>.pt`` so that a later run
  skips the offline stage and uploads straight away.
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import torch

from .discretization import Grid, VelocityModel

__all__ = ["save_model", "load_model", "cache_key", "dump_offline", "load_offline"]

_ROW_J = lambda n: (0, 1, n, n + 1)  # noqa: E731  (rows r0, r1, rn, rnp of a cell)
_SLOTS = ("v0", "v1", "vn", "vnp")


def save_model(path, grid, model):
    """``discretization.py:509-523``: JSON header + raw little-endian f64 binary."""
    path = Path(path)
    bin_path = path.with_suffix(".bin")
    header = {"nx": grid.nx, "nz": grid.nz, "npml": grid.npml, "h": grid.h, "dtype": "f64",
              "order": "row-major, z-major blocks", "data": bin_path.name}
    path.write_text(json.dumps(header, indent=2))
    np.asarray(model.c, dtype="<f8").tofile(bin_path)


def load_model(path):
    """``discretization.py:526-539``: (.json header + .bin) or headered .csv -> (Grid, VelocityModel)."""
    path = Path(path)
    if path.suffix == ".csv":
        return _load_model_csv(path)
    header = json.loads(path.read_text())
    grid = Grid(header["nx"], header["nz"], header["h"], header["npml"])
    data = np.fromfile(path.parent / header.get("data", path.with_suffix(".bin").name), "<f8")
    if data.size != grid.wz * grid.wx:
        raise ValueError(f"binary holds {data.size} values, grid wants {grid.wz * grid.wx}")
    return grid, VelocityModel(grid, data.reshape(grid.shape))


def _load_model_csv(path):
    """``discretization.py:542-560``: '# nx=.. nz=.. npml=.. h=..' header then speed rows."""
    meta, rows = {}, []
    for line in Path(path).read_text().splitlines():
        line = line.strip()
        if not line:
            continue
        if line.startswith("#"):
            for tok in line[1:].replace(",", " ").split():
                if "=" in tok:
                    k, v = tok.split("=")
                    meta[k.strip()] = float(v)
            continue
        rows.append([float(v) for v in line.split(",")])
    try:
        grid = Grid(int(meta["nx"]), int(meta["nz"]), meta["h"], int(meta["npml"]))
    except KeyError as exc:
        raise ValueError("CSV model needs a '# nx=.. nz=.. npml=.. h=..' header") from exc
    return grid, VelocityModel(grid, np.array(rows))


def cache_key(model, grid, omega, partition):
    """``green.py:182-189``: hash identifying one (model, grid, omega, partition) offline stage."""
    hasher = hashlib.sha256()
    hasher.update(np.ascontiguousarray(model.c).tobytes())
    meta = (grid.nx, grid.nz, grid.h, grid.npml, float(omega), tuple(partition.extents))
    hasher.update(repr(meta).encode())
    return hasher.hexdigest()[:16]


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def dump_offline(layers, directory, key):
    """Write the offline stage of ``layers`` (from ``build_nested_layers``).

    Per (layer l, cell c): ``green_<key>_layer<l>_cell<c>.npz/.json`` in the reference's GreenBlockSet
    format (arrays ``"<j>_<slot>"``, j in {0, 1, n, n+1}, each the w x w matrix applied to a slot panel);
    ``nested_<key>.json`` the manifest; ``factors_<key>.pt`` every uploaded factor."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    F = layers.factors
    for lf in F.layers:
        for cf in lf.cells:
            tag = f"{key}_layer{lf.index + 1}_cell{cf.cell + 1}"
            G = _np(cf.green.transpose(-1, -2))  # stored column-major: the transpose is the matrix
            js = _ROW_J(cf.nxc)
            arrays = {f"{js[r]}_{_SLOTS[s]}": np.ascontiguousarray(G[r, s]) for r in range(4) for s in range(4)}
            np.savez(directory / f"green_{tag}.npz", **arrays)
            manifest = {"key": tag, "n": cf.nxc, "width": cf.w, "rows": sorted(set(js)),
                        "format": "dense complex128 blocks, little-endian", "version": 1}
            (directory / f"green_{tag}.json").write_text(json.dumps(manifest, indent=2))
    manifest = {"key": key, "version": 1, "backend": layers.backend, "layers": F.L, "cells": F.Lc,
                "cell_extents": list(F.cell_extents), "omega": F.omega, "inner_ktol": layers.inner_ktol,
                "inner_max_iter": layers.inner_max_iter,
                "assembled_boundary": bool(getattr(F, "assembled_boundary", False)),
                "factors": f"factors_{key}.pt"}
    (directory / f"nested_{key}.json").write_text(json.dumps(manifest, indent=2))
    torch.save(F, directory / f"factors_{key}.pt")


def load_offline(directory, key, grid, partition, device=None):
    """Rebuild ``build_nested_layers``' result from ``dump_offline`` artifacts (no offline arithmetic).

    ``device`` moves the factors (e.g. ``"cuda"``) before the solver uploads them."""
    from .solver import LayerDescriptor, NestedLayers

    directory = Path(directory)
    manifest = json.loads((directory / f"nested_{key}.json").read_text())
    F = torch.load(directory / manifest["factors"], weights_only=False)
    if (F.nx, F.nz, F.npml, tuple(lf.n for lf in F.layers)) != (grid.nx, grid.nz, grid.npml,
                                                                 tuple(partition.extents)):
        raise ValueError("offline artifacts were built for another grid or partition")
    if device is not None:
        for lf in F.layers:
            for name in ("dense", "lu_inv"):
                if getattr(lf, name, None) is not None:
                    setattr(lf, name, getattr(lf, name).to(device))
            for cf in lf.cells:
                for name in ("sinv", "green", "gsmp", "q0"):
                    if getattr(cf, name, None) is not None:
                        setattr(cf, name, getattr(cf, name).to(device))
    items = []
    for ell, (n, off) in enumerate(zip(partition.extents, partition.offsets)):
        lgrid = Grid(grid.nx, n, grid.h, grid.npml, origin=(grid.origin[0], grid.origin[1] + off))
        items.append(LayerDescriptor(ell, n, grid.wx, lgrid, F.Lc))
    return NestedLayers(items, F, F.Lc, manifest["backend"], manifest["inner_ktol"], manifest["inner_max_iter"])
