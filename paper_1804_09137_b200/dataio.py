"""CSV ingestion on either side of the likelihood path.

Same file formats, policies and errors as the reference's dataio.py
(/root/reference/pkg/src/tlrgeo/dataio.py:1-14,141-221):

  locations   x,y  | lon,lat                  load_locations / save_locations
  values      value                           load_values / save_values
  dataset     x,y,value | lon,lat,value       load_dataset / save_dataset
  trace       iter,theta1,theta2,theta3,loglik,seconds   save_trace
  prediction  x,y,predicted[,truth]           save_predictions / load_predictions

UTF-8, LF line endings, a header row, floats written with 17 significant
digits so save -> load is bitwise.  Dataset rows whose value is empty or
"NA" are dropped ("drop", the default) or raise ("strict").  Coordinates
are handed to the device path untouched (api.LocationSet); this module is
host-only file handling.
"""
from __future__ import annotations

import csv
import logging
from dataclasses import dataclass

import numpy as np

from .api import Euclidean, LocationSet, sphere_radius

log = logging.getLogger(__name__)

MISSING = frozenset(("", "NA"))


class DataError(Exception):
    """Malformed or inconsistent input data (dataio.py:30-31)."""


@dataclass(frozen=True)
class Dataset:
    """Locations + one measurement per location (dataio.py:34-48)."""

    locations: LocationSet
    values: np.ndarray
    provenance: str = ""

    def __post_init__(self):
        if self.values.shape != (len(self.locations),):
            raise DataError(f"values shape {self.values.shape} does not match "
                            f"{len(self.locations)} locations")
        if not np.isfinite(self.values).all():
            raise DataError("dataset values must be finite")


def _num(v) -> str:
    return format(float(v), ".17g")


def _coord_names(metric) -> list[str]:
    return ["lon", "lat"] if sphere_radius(metric) > 0 else ["x", "y"]


def _rows(path, header: list[str]):
    """Yield (line_no, fields) of the non-blank data rows after checking the
    header (case / whitespace-insensitive)."""
    with open(path, newline="", encoding="utf-8") as fh:
        it = csv.reader(fh)
        got = next(it, None)
        if got is None:
            raise DataError(f"{path}: empty file")
        if [h.strip().lower() for h in got] != header:
            raise DataError(f"{path}: expected header {','.join(header)!r}, got {','.join(got)!r}")
        for line_no, fields in enumerate(it, start=2):
            if fields:
                yield line_no, fields


def _float(text: str, line_no: int, path) -> float:
    try:
        return float(text)
    except ValueError:
        raise DataError(f"{path}:{line_no}: malformed number {text!r}") from None


def _locations(coords: list, lines: list[int], metric, path) -> LocationSet:
    xy = np.array(coords, dtype=float)
    where: dict = {}
    for k, key in enumerate(map(tuple, xy)):
        where.setdefault(key, []).append(lines[k])
    dups = sorted(key for key, at in where.items() if len(at) > 1)
    if dups:   # the lexicographically smallest repeated point, like np.unique order
        at = where[dups[0]]
        raise DataError(f"{path}: duplicate location {dups[0]} at lines {at[0]} and {at[1]}")
    try:
        return LocationSet(xy, metric)
    except ValueError as exc:
        raise DataError(f"{path}: {exc}") from None


def load_locations(path, metric=None) -> LocationSet:
    metric = Euclidean() if metric is None else metric
    coords, lines = [], []
    for line_no, f in _rows(path, _coord_names(metric)):
        if len(f) != 2:
            raise DataError(f"{path}:{line_no}: expected 2 fields, got {len(f)}")
        coords.append((_float(f[0], line_no, path), _float(f[1], line_no, path)))
        lines.append(line_no)
    if not coords:
        raise DataError(f"{path}: no locations")
    return _locations(coords, lines, metric, path)


def save_locations(path, locs) -> None:
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write(",".join(_coord_names(locs.metric)) + "\n")
        fh.writelines(f"{_num(x)},{_num(y)}\n" for x, y in locs.coords)


def load_values(path) -> np.ndarray:
    vals = [_float(f[0], line_no, path) for line_no, f in _rows(path, ["value"])]
    if not vals:
        raise DataError(f"{path}: no values")
    return np.array(vals)


def save_values(path, values) -> None:
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write("value\n")
        fh.writelines(_num(v) + "\n" for v in np.asarray(values, dtype=float))


def load_dataset(path, metric=None, missing_policy: str = "drop") -> Dataset:
    """Read a coordinates + value dataset (dataio.py:141-184)."""
    if missing_policy not in ("drop", "strict"):
        raise ValueError(f"unknown missing policy {missing_policy!r}")
    metric = Euclidean() if metric is None else metric
    coords, vals, lines, dropped = [], [], [], 0
    for line_no, f in _rows(path, _coord_names(metric) + ["value"]):
        if len(f) != 3:
            raise DataError(f"{path}:{line_no}: expected 3 fields, got {len(f)}")
        if f[2].strip() in MISSING:
            if missing_policy == "strict":
                raise DataError(f"{path}:{line_no}: missing value")
            dropped += 1
            continue
        coords.append((_float(f[0], line_no, path), _float(f[1], line_no, path)))
        vals.append(_float(f[2], line_no, path))
        lines.append(line_no)
    if not coords:
        raise DataError(f"{path}: no usable rows")
    if dropped:
        log.info("%s: dropped %d rows with missing values", path, dropped)
    return Dataset(_locations(coords, lines, metric, path), np.array(vals), provenance=str(path))


def save_dataset(path, ds: Dataset) -> None:
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write(",".join(_coord_names(ds.locations.metric) + ["value"]) + "\n")
        fh.writelines(f"{_num(x)},{_num(y)},{_num(v)}\n"
                      for (x, y), v in zip(ds.locations.coords, ds.values))


def partition_regions(ds: Dataset, rows: int, cols: int) -> list[Dataset]:
    """Equal-cell rows x cols split of the bounding box; non-empty cells in
    row-major order from (ymin, xmin) become R0, R1, ... (dataio.py:187-221)."""
    if rows < 1 or cols < 1:
        raise ValueError(f"need rows, cols >= 1, got {rows}x{cols}")
    c = ds.locations.coords
    lo, hi = c.min(axis=0), c.max(axis=0)
    span = np.where(hi - lo == 0, 1.0, hi - lo)
    ci = np.minimum((cols * (c[:, 0] - lo[0]) / span[0]).astype(int), cols - 1)
    ri = np.minimum((rows * (c[:, 1] - lo[1]) / span[1]).astype(int), rows - 1)
    cell = ri * cols + ci
    out: list[Dataset] = []
    for k in range(rows * cols):
        sel = cell == k
        if not sel.any():
            log.info("region cell %d of %dx%d grid is empty; skipped", k, rows, cols)
            continue
        name = f"R{len(out)}"
        out.append(Dataset(LocationSet(c[sel], ds.locations.metric), ds.values[sel],
                           provenance=f"{ds.provenance}/{name}" if ds.provenance else name))
    return out


def save_trace(path, trace) -> None:
    """MLE trace (mle.TraceEntry rows)."""
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write("iter,theta1,theta2,theta3,loglik,seconds\n")
        for t in trace:
            fh.write(",".join([str(t.index), *map(_num, t.theta), _num(t.loglik), _num(t.seconds)]) + "\n")


def save_predictions(path, unknown, pred, truth=None) -> None:
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write("x,y,predicted" + (",truth" if truth is not None else "") + "\n")
        for i, (x, y) in enumerate(unknown.coords):
            tail = f",{_num(truth[i])}" if truth is not None else ""
            fh.write(f"{_num(x)},{_num(y)},{_num(pred[i])}{tail}\n")


def load_predictions(path):
    """(coords, predicted, truth or None) of a prediction CSV."""
    with open(path, newline="", encoding="utf-8") as fh:
        head = next(csv.reader(fh), None)
    if head is None:
        raise DataError(f"{path}: empty file")
    names = [h.strip().lower() for h in head]
    if names not in (["x", "y", "predicted"], ["x", "y", "predicted", "truth"]):
        raise DataError(f"{path}: unexpected prediction header {head!r}")
    recs = [[_float(t, line_no, path) for t in f[:len(names)]] for line_no, f in _rows(path, names)]
    a = np.array(recs, dtype=float).reshape(-1, len(names))
    return a[:, :2].copy(), a[:, 2].copy(), (a[:, 3].copy() if len(names) == 4 else None)
