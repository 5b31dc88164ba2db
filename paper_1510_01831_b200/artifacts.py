"""Formats around the online path: velocity-model files and offline artifacts.

* ``save_model`` / ``load_model``: the reference's velocity-model files (format of
  ``discretization.py:509-560``): a JSON header next to raw little-endian float64 samples of the extended
  grid (depth-major), or a small CSV whose comment line carries ``nx nz npml h``.
* ``cache_key``: the reference's hash of one offline stage (``green.py:182-189``), byte-identical.
* ``dump_offline`` / ``load_offline``: persistence of the offline stage this path uploads.  The Green
  blocks are written in the reference's ``GreenBlockSet.dump`` format (``green.py:156-169``; readable by
  ``GreenBlockSet.load``), one set per (layer, cell), with a manifest like ``dump_offline``
  (``nested.py:489-504``).  The complete factor set (Schur inverses, couplings, pass-0 and
  sampled-response operators, dense or direct inner operators) goes into ``factors_<key>.pt`` as plain
  tensors and scalars (loaded with ``torch.load(weights_only=True)``: no pickled code), so a later run
  skips the offline stage.  The manifest records the stage's ``cache_key``, ``h`` and ``omega``;
  ``load_offline`` rejects artifacts built for another model, frequency, grid or partition.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import re
from pathlib import Path

import numpy as np
import torch

from .discretization import Grid, VelocityModel

__all__ = ["save_model", "load_model", "cache_key", "dump_offline", "load_offline"]

_CELL_ROWS = lambda n: (0, 1, n, n + 1)  # noqa: E731  (sampled rows r0, r1, rn, rnp of a cell)
_SLOT_NAMES = ("v0", "v1", "vn", "vnp")

# ---------------------------------------------------------------------------------------------- model files

_BIN_DTYPE = "<f8"
_ORDER = "row-major, z-major blocks"  # the reference header's "order" string (depth rows are contiguous)
_CSV_KEYS = ("nx", "nz", "npml", "h")


def _grid_from(meta, where):
    missing = [k for k in _CSV_KEYS if k not in meta]
    if missing:
        raise ValueError(f"{where}: model header lacks {', '.join(missing)} (needs nx, nz, npml, h)")
    return Grid(int(meta["nx"]), int(meta["nz"]), float(meta["h"]), int(meta["npml"]))


def _checked(grid, values, where):
    values = np.asarray(values, dtype=float)
    want = grid.wz * grid.wx
    if values.size != want:
        raise ValueError(f"{where}: {values.size} speed samples for a {grid.wz} x {grid.wx} extended grid "
                         f"({want} expected)")
    return grid, VelocityModel(grid, values.reshape(grid.shape))


def save_model(path, grid, model):
    """Header ``<path>`` (JSON) + samples ``<path>.bin`` (little-endian f64, extended grid, depth-major)."""
    path = Path(path)
    data = path.with_suffix(".bin")
    meta = dict(nx=grid.nx, nz=grid.nz, npml=grid.npml, h=grid.h, dtype="f64", order=_ORDER, data=data.name)
    path.write_text(json.dumps(meta, indent=2))
    np.ascontiguousarray(model.c, dtype=_BIN_DTYPE).tofile(data)


def load_model(path):
    """``(Grid, VelocityModel)`` from a JSON header + binary pair or a headered CSV (by suffix)."""
    path = Path(path)
    if path.suffix.lower() == ".csv":
        text = path.read_text()
        meta = {}
        for key, val in re.findall(r"(\w+)\s*=\s*([-+0-9.eE]+)", " ".join(
                ln for ln in text.splitlines() if ln.lstrip().startswith("#"))):
            meta[key] = float(val)
        body = [ln for ln in text.splitlines() if ln.strip() and not ln.lstrip().startswith("#")]
        grid = _grid_from(meta, path.name)
        rows = np.array([[float(v) for v in ln.split(",")] for ln in body]) if body else np.zeros(0)
        return _checked(grid, rows, path.name)
    meta = json.loads(path.read_text())
    grid = _grid_from(meta, path.name)
    binary = path.parent / meta.get("data", path.with_suffix(".bin").name)
    return _checked(grid, np.fromfile(binary, dtype=_BIN_DTYPE), binary.name)


def cache_key(model, grid, omega, partition):
    """``green.py:182-189``: sha256 of the speeds and the (grid, omega, partition) tuple, 16 hex chars.

    Must stay byte-identical to the reference's recipe (artifact names are keyed by it)."""
    h = hashlib.sha256(np.ascontiguousarray(model.c).tobytes())
    h.update(repr((grid.nx, grid.nz, grid.h, grid.npml, float(omega), tuple(partition.extents))).encode())
    return h.hexdigest()[:16]


# ---------------------------------------------------------------------------------------------- factors

def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _to_plain(obj):
    """Dataclasses -> {"__dc__": name, fields...}; numpy arrays -> {"__np__": tensor}: only the types
    ``torch.load(weights_only=True)`` accepts."""
    if dataclasses.is_dataclass(obj):
        out = {"__dc__": type(obj).__name__}
        for f in dataclasses.fields(obj):
            out[f.name] = _to_plain(getattr(obj, f.name))
        return out
    if isinstance(obj, np.ndarray):
        return {"__np__": torch.from_numpy(np.ascontiguousarray(obj))}
    if isinstance(obj, (list, tuple)):
        return type(obj)(_to_plain(v) for v in obj)
    if isinstance(obj, (np.integer, np.floating)):
        return obj.item()
    return obj


def _from_plain(obj):
    from . import offline

    if isinstance(obj, dict) and "__np__" in obj:
        return obj["__np__"].numpy()
    if isinstance(obj, dict) and "__dc__" in obj:
        cls = {"Factors": offline.Factors, "LayerFactors": offline.LayerFactors,
               "CellFactors": offline.CellFactors}[obj["__dc__"]]
        return cls(**{k: _from_plain(v) for k, v in obj.items() if k != "__dc__"})
    if isinstance(obj, (list, tuple)):
        return type(obj)(_from_plain(v) for v in obj)
    return obj


def dump_offline(layers, directory, key, model=None, grid=None, omega=None, partition=None):
    """Write the offline stage of ``layers`` (from ``build_nested_layers``).

    Per (layer l, cell c): ``green_<key>_layer<l>_cell<c>.npz/.json`` in the reference's GreenBlockSet
    format (arrays ``"<j>_<slot>"``, j in {0, 1, n, n+1}, each the w x w matrix applied to a slot panel);
    ``nested_<key>.json`` the manifest; ``factors_<key>.pt`` every uploaded factor.  With ``model``,
    ``grid``, ``omega`` and ``partition`` the manifest also records their ``cache_key``."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    F = layers.factors
    for lf in F.layers:
        for cf in lf.cells:
            tag = f"{key}_layer{lf.index + 1}_cell{cf.cell + 1}"
            blocks = _np(cf.green.transpose(-1, -2))  # stored column-major: the transpose is the matrix
            rows = _CELL_ROWS(cf.nxc)
            np.savez(directory / f"green_{tag}.npz",
                     **{f"{rows[r]}_{_SLOT_NAMES[s]}": np.ascontiguousarray(blocks[r, s])
                        for r in range(4) for s in range(4)})
            (directory / f"green_{tag}.json").write_text(json.dumps(
                {"key": tag, "n": cf.nxc, "width": cf.w, "rows": sorted(set(rows)),
                 "format": "dense complex128 blocks, little-endian", "version": 1}, indent=2))
    stage_key = None
    if model is not None and grid is not None and partition is not None:
        stage_key = cache_key(model, grid, F.omega if omega is None else omega, partition)
    manifest = {"key": key, "version": 2, "backend": layers.backend, "layers": F.L, "cells": F.Lc,
                "cell_extents": list(F.cell_extents), "omega": F.omega, "h": F.h,
                "nx": F.nx, "nz": F.nz, "npml": F.npml, "layer_extents": [lf.n for lf in F.layers],
                "cache_key": stage_key, "inner_ktol": layers.inner_ktol,
                "inner_max_iter": layers.inner_max_iter,
                "assembled_boundary": bool(getattr(F, "assembled_boundary", False)),
                "factors": f"factors_{key}.pt"}
    (directory / f"nested_{key}.json").write_text(json.dumps(manifest, indent=2))
    torch.save(_to_plain(F), directory / f"factors_{key}.pt")


def load_offline(directory, key, grid, partition, model=None, omega=None, device=None):
    """Rebuild ``build_nested_layers``' result from ``dump_offline`` artifacts (no offline arithmetic).

    Raises ``ValueError`` when the artifacts were built for another grid, partition, frequency ``omega``
    or velocity ``model`` (checked against the manifest's ``cache_key`` when both sides have one).
    ``device`` moves the factors (e.g. ``"cuda"``) before the solver uploads them."""
    from .solver import LayerDescriptor, NestedLayers

    directory = Path(directory)
    manifest = json.loads((directory / f"nested_{key}.json").read_text())
    want = (grid.nx, grid.nz, grid.npml, tuple(partition.extents))
    have = (manifest.get("nx"), manifest.get("nz"), manifest.get("npml"), tuple(manifest.get("layer_extents", ())))
    if have != want:
        raise ValueError(f"offline artifacts were built for grid/partition {have}, not {want}")
    if abs(float(manifest.get("h", grid.h)) - grid.h) > 1e-15 * grid.h:
        raise ValueError(f"offline artifacts were built for h = {manifest.get('h')}, not {grid.h}")
    if omega is not None and float(manifest["omega"]) != float(omega):
        raise ValueError(f"offline artifacts were built for omega = {manifest['omega']}, not {omega}")
    if model is not None:
        if manifest.get("cache_key") is None:
            raise ValueError("offline artifacts carry no cache_key to check the velocity model against")
        got = cache_key(model, grid, manifest["omega"] if omega is None else omega, partition)
        if got != manifest["cache_key"]:
            raise ValueError(f"offline artifacts were built for another model (cache_key "
                             f"{manifest['cache_key']} != {got})")
    F = _from_plain(torch.load(directory / manifest["factors"], weights_only=True))
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
    out = NestedLayers(items, F, F.Lc, manifest["backend"], manifest["inner_ktol"], manifest["inner_max_iter"])
    return out
