"""On-disk dataset and arch formats (the reference's space.py:203-392 and
counters.py:183-255), so B200 sweeps and the reference's datasets are
interchangeable.

    space.csv         `param:<name>` header, `binary:<0|1>` row, one row of
                      parameter values per configuration (row = index)
    measurements.csv  `config_index,runtime_us,global_threads,<counter>...`;
                      counter columns are canonical abbreviations or raw
                      per-generation names (canonicalised on load)
    arch.txt          `key = value`: name, generation, cores, map.<raw>,
                      ratio.<raw>

Floats are written with repr: a load/save cycle is byte-stable and byte-
identical to the reference's writers (tests/test_formats.py pins both
against files the reference wrote).  Loading builds the array-backed
Dataset directly (no per-record objects).
"""

import csv
import os
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import counters as cc
from .counters import ArchProfile
from .errors import DatasetFormatError, UnknownCounterError
from .space import Dataset, TuningParameter, TuningSpace

SPACE_FILENAME = "space.csv"
MEASUREMENTS_FILENAME = "measurements.csv"
ARCH_FILENAME = "arch.txt"

# counters.py:116-124: admissible ranges of the stress counters (0-10
# utilisation levels / percent); OPS counters are only bounded below by 0
VALUE_RANGES: Dict[str, Tuple[float, Optional[float]]] = {
    "DRAM_U": (0.0, 10.0), "L2_U": (0.0, 100.0),
    "TEX_U": (0.0, 10.0), "SHR_U": (0.0, 10.0), "SM_E": (0.0, 100.0), "WARP_E": (0.0, 100.0),
    "WARP_NP_E": (0.0, 100.0),
}


def _fmt(value: float) -> str:
    return repr(float(value))


# ------------------------------------------------------------------- space
def load_space(path) -> TuningSpace:
    """space.py:207-272 (same validation, same messages)."""
    with open(path, "r", encoding="utf-8", newline="") as fh:
        reader = csv.reader(fh)
        try:
            header = next(reader)
        except StopIteration:
            raise DatasetFormatError(path, 1, "empty space file")
        names = []
        for col, cell in enumerate(header):
            if not cell.startswith("param:") or not cell[len("param:"):]:
                raise DatasetFormatError(path, 1, f"column {col + 1}: expected 'param:<name>', "
                                                  f"got {cell!r}")
            names.append(cell[len("param:"):])
        if len(set(names)) != len(names):
            raise DatasetFormatError(path, 1, "duplicate parameter name in header")
        try:
            flag_row = next(reader)
        except StopIteration:
            raise DatasetFormatError(path, 2, "missing binary flag row")
        if len(flag_row) != len(names):
            raise DatasetFormatError(path, 2, "flag row width differs from header")
        flags = []
        for col, cell in enumerate(flag_row):
            if cell not in ("binary:0", "binary:1"):
                raise DatasetFormatError(path, 2, f"column {col + 1}: expected 'binary:0' or "
                                                  f"'binary:1', got {cell!r}")
            flags.append(cell == "binary:1")
        rows: List[Tuple[float, ...]] = []
        seen = {}
        for lineno, row in enumerate(reader, start=3):
            if not row:
                continue
            if len(row) != len(names):
                raise DatasetFormatError(path, lineno, f"expected {len(names)} values, "
                                                       f"got {len(row)}")
            try:
                values = tuple(float(c) for c in row)
            except ValueError:
                raise DatasetFormatError(path, lineno, f"non-numeric parameter value in {row!r}")
            if values in seen:
                raise DatasetFormatError(path, lineno, "duplicate configuration (first at line "
                                                       f"{seen[values]})")
            seen[values] = lineno
            for i, v in enumerate(values):
                if flags[i] and v not in (0.0, 1.0):
                    raise DatasetFormatError(path, lineno, f"parameter {names[i]!r} is binary "
                                                           f"but has value {row[i]!r}")
            rows.append(values)
        if not rows:
            raise DatasetFormatError(path, 3, "space file has no configurations")
    grid = np.array(rows, dtype=np.float64)
    params = []
    for i, name in enumerate(names):
        if flags[i]:
            values = (0.0, 1.0)
        else:
            values = tuple(sorted(set(grid[:, i].tolist())))
            if set(values) == {0.0, 1.0}:
                raise DatasetFormatError(path, 2, f"parameter {name!r} takes exactly the values "
                                                  f"0 and 1 and must be flagged binary:1")
        params.append(TuningParameter(name=name, values=values, is_binary=flags[i]))
    return TuningSpace.from_assignments(params, grid)


def save_space(space: TuningSpace, path) -> None:
    lines = [",".join(f"param:{p.name}" for p in space.parameters),
             ",".join(f"binary:{1 if p.is_binary else 0}" for p in space.parameters)]
    for row in space.assignments.tolist():
        lines.append(",".join(_fmt(v) for v in row))
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


# ------------------------------------------------------------ measurements
def _check_range(idx, abbr, value):
    lo, hi = VALUE_RANGES.get(abbr, (0.0, None))
    if not value >= lo or (hi is not None and value > hi):
        bound = f"<{lo}, {hi}>" if hi is not None else f">= {lo}"
        raise ValueError(f"config {idx}: counter {abbr} value {value!r} outside {bound}")


def load_measurements(path, space: TuningSpace, arch: ArchProfile):
    """space.py:286-350 -> (runtime[n], threads[n], names, matrix[n x k], has_record[n],
    config indices in file order)."""
    n = len(space)
    with open(path, "r", encoding="utf-8", newline="") as fh:
        reader = csv.reader(fh)
        try:
            header = next(reader)
        except StopIteration:
            raise DatasetFormatError(path, 1, "empty measurements file")
        if header[:3] != ["config_index", "runtime_us", "global_threads"]:
            raise DatasetFormatError(path, 1, "header must start with "
                                              "'config_index,runtime_us,global_threads'")
        columns = []
        for cell in header[3:]:
            if cell == cc.GLOBAL_THREADS:
                raise DatasetFormatError(path, 1, "GLOBAL_THREADS is carried by the "
                                                  "global_threads column, not a counter column")
            try:
                abbr, _ = cc.canonicalize(cell, 0.0, arch)
            except KeyError:
                raise UnknownCounterError(path, 1, f"unknown counter column {cell!r} for "
                                                   f"arch {arch.name!r} ({arch.generation})")
            columns.append((cell, abbr))
        abbrs = [a for _, a in columns]
        if len(set(abbrs)) != len(abbrs):
            raise DatasetFormatError(path, 1, "two counter columns canonicalize to the same "
                                              "abbreviation")
        names = tuple(a for a in cc.ABBREVIATIONS if a in set(abbrs))
        pos = [names.index(a) for a in abbrs]
        rt = np.zeros(n)
        th = np.zeros(n, dtype=np.int64)
        cm = np.zeros((n, len(names)))
        hr = np.zeros(n, dtype=bool)
        seen = {}
        order = []
        for lineno, row in enumerate(reader, start=2):
            if not row:
                continue
            if len(row) != 3 + len(columns):
                raise DatasetFormatError(path, lineno, f"expected {3 + len(columns)} cells, "
                                                       f"got {len(row)}")
            try:
                idx = int(row[0])
            except ValueError:
                raise DatasetFormatError(path, lineno, f"config_index must be an integer, "
                                                       f"got {row[0]!r}")
            if not 0 <= idx < n:
                raise DatasetFormatError(path, lineno, f"config_index {idx} outside the space "
                                                       f"(0..{n - 1})")
            if idx in seen:
                raise DatasetFormatError(path, lineno, f"duplicate config_index {idx} "
                                                       f"(first at line {seen[idx]})")
            seen[idx] = lineno
            try:
                runtime = float(row[1])
                threads = int(row[2])
                raw_values = [float(c) for c in row[3:]]
            except ValueError:
                raise DatasetFormatError(path, lineno, f"non-numeric cell in {row!r}")
            try:
                if not runtime > 0:
                    raise ValueError(f"config {idx}: runtime_us must be > 0, got {runtime!r}")
                if threads < 1:
                    raise ValueError(f"config {idx}: global_threads must be >= 1")
                for (raw_name, abbr), value, j in zip(columns, raw_values, pos):
                    _, canon = cc.canonicalize(raw_name, value, arch)
                    _check_range(idx, abbr, canon)
                    cm[idx, j] = canon
            except ValueError as exc:
                raise DatasetFormatError(path, lineno, str(exc))
            rt[idx], th[idx], hr[idx] = runtime, threads, True
            order.append(idx)
        if not hr.any():
            raise DatasetFormatError(path, 2, "no records")
    return rt, th, names, cm, hr, np.array(order, dtype=np.int64)


def save_measurements(dataset: Dataset, path) -> None:
    """Canonical form: ascending index, catalog column order (space.py:353-362)."""
    names = dataset.counter_names
    header = "config_index,runtime_us,global_threads," + ",".join(names)
    lines = [header.rstrip(",")]
    rt, th, cm = dataset.runtime_us, dataset.global_threads, dataset.counter_matrix
    for i in np.flatnonzero(dataset.has_record).tolist():
        cells = [str(i), _fmt(rt[i]), str(int(th[i]))]
        cells.extend(_fmt(v) for v in cm[i].tolist())
        lines.append(",".join(cells))
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


# -------------------------------------------------------------------- arch
def load_arch(path) -> ArchProfile:
    """counters.py:183-239."""
    name = generation = cores = None
    maps: Dict[str, str] = {}
    ratios: Dict[str, float] = {}
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            stripped = line.strip()
            if not stripped or stripped.startswith("#"):
                continue
            if "=" not in stripped:
                raise DatasetFormatError(path, lineno, f"expected 'key = value', got {stripped!r}")
            key, _, val = stripped.partition("=")
            key, val = key.strip(), val.strip()
            if key == "name":
                name = val
            elif key == "generation":
                if val not in cc.GENERATIONS:
                    raise DatasetFormatError(
                        path, lineno, f"generation must be one of {cc.GENERATIONS}, got {val!r}")
                generation = val
            elif key == "cores":
                try:
                    cores = int(val)
                except ValueError:
                    raise DatasetFormatError(path, lineno, f"cores must be an integer, got {val!r}")
                if cores < 1:
                    raise DatasetFormatError(path, lineno, f"cores must be >= 1, got {cores}")
            elif key.startswith("map."):
                if val not in cc.ABBREVIATIONS:
                    raise DatasetFormatError(path, lineno,
                                             f"map target {val!r} is not a canonical counter")
                maps[key[len("map."):]] = val
            elif key.startswith("ratio."):
                try:
                    ratios[key[len("ratio."):]] = float(val)
                except ValueError:
                    raise DatasetFormatError(path, lineno, f"ratio must be a number, got {val!r}")
            else:
                raise DatasetFormatError(path, lineno, f"unknown key {key!r}")
    if name is None or generation is None or cores is None:
        raise DatasetFormatError(path, 0, "arch file must define name, generation, and cores")
    for raw in ratios:
        if raw not in maps:
            raise DatasetFormatError(path, 0, f"ratio.{raw} given without a matching map.{raw}")
    overrides = {raw: (abbr, ratios.get(raw, 1.0)) for raw, abbr in maps.items()}
    return ArchProfile(name=name, generation=generation, cores=cores, overrides=overrides)


def save_arch(arch: ArchProfile, path) -> None:
    lines = [f"name = {arch.name}", f"generation = {arch.generation}", f"cores = {arch.cores}"]
    overrides = getattr(arch, "overrides", {}) or {}
    for raw in sorted(overrides):
        abbr, ratio = overrides[raw]
        lines.append(f"map.{raw} = {abbr}")
        if ratio != 1.0:
            lines.append(f"ratio.{raw} = {ratio!r}")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


# ----------------------------------------------------------------- dataset
def load_dataset(space_path, measurements_path, arch_path,
                 input_label: Optional[str] = None) -> Dataset:
    space = load_space(space_path)
    arch = load_arch(arch_path)
    rt, th, names, cm, hr, order = load_measurements(measurements_path, space, arch)
    if input_label is None:
        input_label = os.path.basename(os.path.dirname(os.path.abspath(measurements_path)))
    return Dataset(space, arch, input_label, runtime_us=rt, global_threads=th,
                   counter_names=names, counter_matrix=cm, has_record=hr, record_order=order)


def load_dataset_dir(directory, input_label: Optional[str] = None) -> Dataset:
    if input_label is None:
        input_label = os.path.basename(os.path.normpath(directory))
    return load_dataset(os.path.join(directory, SPACE_FILENAME),
                        os.path.join(directory, MEASUREMENTS_FILENAME),
                        os.path.join(directory, ARCH_FILENAME), input_label=input_label)


def save_dataset(dataset: Dataset, directory) -> None:
    os.makedirs(directory, exist_ok=True)
    save_space(dataset.space, os.path.join(directory, SPACE_FILENAME))
    save_measurements(dataset, os.path.join(directory, MEASUREMENTS_FILENAME))
    save_arch(dataset.arch, os.path.join(directory, ARCH_FILENAME))
