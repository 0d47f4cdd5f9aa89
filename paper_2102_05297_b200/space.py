"""Tuning spaces and replay datasets -- the data types on both sides of the
searcher hot path (the reference's space.py:37-186), array-backed.

The reference stores a space as a tuple of TuningConfiguration objects and a
dataset as a tuple of MeasurementRecord objects with counter dicts.  The
device path wants the same data as dense float64 arrays (one row per
configuration), so both types here keep arrays as the primary storage and
materialise the reference's object views lazily.  Objects built from the
reference's own classes are accepted anywhere a Dataset / TuningSpace is
expected (duck typing on .space / .records / .configurations).
"""

from dataclasses import dataclass
from typing import Dict, FrozenSet, Optional, Sequence, Tuple

import numpy as np

from . import counters as cc
from .counters import ArchProfile


@dataclass(frozen=True)
class TuningParameter:
    """One tuning parameter and its admissible values (space.py:37-64)."""

    name: str
    values: Tuple[float, ...]
    is_binary: bool = False

    def __post_init__(self):
        if not self.values:
            raise ValueError(f"parameter {self.name!r} has no values")
        if list(self.values) != sorted(set(self.values)):
            raise ValueError(f"parameter {self.name!r} values must be ascending and unique")
        if self.is_binary and tuple(self.values) != (0.0, 1.0):
            raise ValueError(f"binary parameter {self.name!r} must have values (0, 1)")

    @classmethod
    def make(cls, name: str, values) -> "TuningParameter":
        vals = tuple(sorted(set(float(v) for v in values)))
        return cls(name=name, values=vals, is_binary=vals == (0.0, 1.0))


@dataclass(frozen=True)
class TuningConfiguration:
    """A point of the space; index is its row in the space (space.py:67-72)."""

    assignment: Tuple[float, ...]
    index: int


class TuningSpace:
    """Post-constraint enumeration of assignments (space.py:75-104)."""

    def __init__(self, parameters: Sequence[TuningParameter], configurations=None,
                 assignments: Optional[np.ndarray] = None):
        self.parameters = tuple(parameters)
        if assignments is None:
            if configurations is None:
                raise ValueError("a space needs configurations or an assignment array")
            configurations = tuple(configurations)
            for i, conf in enumerate(configurations):
                if conf.index != i:
                    raise ValueError(f"configuration at row {i} carries index {conf.index}")
            assignments = np.array([c.assignment for c in configurations], dtype=np.float64)
            if assignments.size == 0:
                assignments = assignments.reshape(0, len(self.parameters))
            self._configurations = configurations
        else:
            self._configurations = None
        a = np.ascontiguousarray(assignments, dtype=np.float64)
        if a.ndim != 2 or a.shape[1] != len(self.parameters):
            raise ValueError("assignment array must be n x len(parameters)")
        self._assignments = a

    @classmethod
    def from_assignments(cls, parameters, assignments: np.ndarray) -> "TuningSpace":
        return cls(parameters, assignments=assignments)

    @property
    def configurations(self) -> Tuple[TuningConfiguration, ...]:
        if self._configurations is None:
            self._configurations = tuple(
                TuningConfiguration(assignment=tuple(float(v) for v in row), index=i)
                for i, row in enumerate(self._assignments))
        return self._configurations

    @property
    def assignments(self) -> np.ndarray:
        return self._assignments

    def __len__(self):
        return self._assignments.shape[0]

    @property
    def parameter_names(self) -> Tuple[str, ...]:
        return tuple(p.name for p in self.parameters)


@dataclass(frozen=True)
class MeasurementRecord:
    """One benchmarked configuration (space.py:107-127)."""

    config_index: int
    runtime_us: float
    global_threads: int
    counters: Dict[str, float]

    def __post_init__(self):
        if not self.runtime_us > 0:
            raise ValueError(f"config {self.config_index}: runtime_us must be > 0, "
                             f"got {self.runtime_us!r}")
        if self.global_threads < 1:
            raise ValueError(f"config {self.config_index}: global_threads must be >= 1")


class Dataset:
    """A space exhaustively measured on one GPU for one input (space.py:130-174).

    Primary storage: runtime_us[n], global_threads[n], a counter matrix
    n x len(counter_names) in catalog order and has_record[n].
    """

    def __init__(self, space, arch: ArchProfile, input_label: str, records=None, *,
                 runtime_us=None, global_threads=None, counter_names=None,
                 counter_matrix=None, has_record=None, record_order=None):
        self.space = space
        self.arch = arch
        self.input_label = input_label
        n = len(space)
        if records is not None:
            records = tuple(records)
            if not records:
                raise ValueError("dataset has no records")
            names = tuple(a for a in cc.ABBREVIATIONS if a in set(records[0].counters))
            rt = np.zeros(n)
            th = np.zeros(n, dtype=np.int64)
            cm = np.zeros((n, len(names)))
            hr = np.zeros(n, dtype=bool)
            keys = set(records[0].counters)
            for rec in records:
                i = rec.config_index
                if not 0 <= i < n:
                    raise ValueError(f"record references configuration {i}, space has {n}")
                if hr[i]:
                    raise ValueError(f"duplicate measurement for configuration {i}")
                if set(rec.counters) != keys:
                    raise ValueError(f"record {i} has a different counter set than the first record")
                hr[i] = True
                rt[i] = rec.runtime_us
                th[i] = rec.global_threads
                cm[i] = [rec.counters[a] for a in names]
            self._records = records
            order = np.array([rec.config_index for rec in records], dtype=np.int64)
        else:
            names = tuple(counter_names)
            rt = np.ascontiguousarray(runtime_us, dtype=np.float64)
            th = np.ascontiguousarray(global_threads, dtype=np.int64)
            cm = np.ascontiguousarray(counter_matrix, dtype=np.float64)
            hr = (np.ones(n, dtype=bool) if has_record is None
                  else np.ascontiguousarray(has_record, dtype=bool))
            if rt.shape != (n,) or th.shape != (n,) or cm.shape != (n, len(names)):
                raise ValueError("dataset arrays do not match the space size")
            if not hr.any():
                raise ValueError("dataset has no records")
            if np.any(rt[hr] <= 0) or np.any(th[hr] < 1):
                raise ValueError("runtime_us must be > 0 and global_threads >= 1")
            self._records = None
            order = (np.flatnonzero(hr) if record_order is None
                     else np.ascontiguousarray(record_order, dtype=np.int64))
            if record_order is not None and not np.array_equal(np.sort(order), np.flatnonzero(hr)):
                raise ValueError("record_order must list every recorded configuration once")
        self.runtime_us = rt
        self.global_threads = th
        self.counter_names = names
        self.counter_matrix = cm
        self.has_record = hr
        # configuration indices of the records in file order (the reference
        # keeps Dataset.records in measurements.csv order, space.py:286-350;
        # model training and counter errors iterate records in that order)
        self.record_order = order

    @property
    def records(self) -> Tuple[MeasurementRecord, ...]:
        if self._records is None:
            names = self.counter_names
            self._records = tuple(
                MeasurementRecord(config_index=int(i), runtime_us=float(self.runtime_us[i]),
                                  global_threads=int(self.global_threads[i]),
                                  counters=dict(zip(names, map(float, self.counter_matrix[i]))))
                for i in self.record_order)
        return self._records

    @property
    def best_runtime(self) -> float:
        return float(self.runtime_us[self.has_record].min())

    def record_for(self, config_index: int) -> MeasurementRecord:
        if not (0 <= config_index < len(self.space)) or not self.has_record[config_index]:
            raise KeyError(config_index)
        i = config_index
        return MeasurementRecord(config_index=int(i), runtime_us=float(self.runtime_us[i]),
                                 global_threads=int(self.global_threads[i]),
                                 counters=dict(zip(self.counter_names,
                                                   map(float, self.counter_matrix[i]))))


def well_performing_set(dataset, slack: float = 1.1) -> FrozenSet[int]:
    """Configurations within slack x the best runtime (space.py:177-186)."""
    if slack < 1.0:
        raise ValueError(f"slack must be >= 1.0, got {slack}")
    rt, _, _, hr = replay_arrays(dataset)
    limit = slack * float(rt[hr].min())
    return frozenset(int(i) for i in np.flatnonzero(hr & (rt <= limit)))


def well_performing_mask(dataset, slack: float = 1.1) -> np.ndarray:
    rt, _, _, hr = replay_arrays(dataset)
    if slack < 1.0:
        raise ValueError(f"slack must be >= 1.0, got {slack}")
    limit = slack * float(rt[hr].min())
    return hr & (rt <= limit)


def _names_of(dataset):
    return cc.dataset_counter_names(dataset)


def replay_arrays(dataset):
    """(runtime_us[n], global_threads[n], required counters[n, 23], has_record[n]).

    Works for this module's Dataset and for any object with the reference's
    Dataset attributes.  A dataset that lacks one of the 23 counters analyze()
    needs yields a NaN column; the caller raises AnalysisError for it.
    """
    cached = getattr(dataset, "_ct_replay_cache", None)
    if cached is not None:
        return cached
    n = len(dataset.space)
    if isinstance(dataset, Dataset):
        rt, th, hr = dataset.runtime_us, dataset.global_threads, dataset.has_record
        pos = {a: j for j, a in enumerate(dataset.counter_names)}
        req = np.full((n, len(cc.REQUIRED_COUNTERS)), np.nan)
        for k, a in enumerate(cc.REQUIRED_COUNTERS):
            if a in pos:
                req[:, k] = dataset.counter_matrix[:, pos[a]]
    else:
        rt = np.zeros(n)
        th = np.ones(n, dtype=np.int64)
        hr = np.zeros(n, dtype=bool)
        req = np.full((n, len(cc.REQUIRED_COUNTERS)), np.nan)
        for rec in dataset.records:
            i = rec.config_index
            hr[i] = True
            rt[i] = rec.runtime_us
            th[i] = rec.global_threads
            req[i] = [rec.counters.get(a, np.nan) for a in cc.REQUIRED_COUNTERS]
    out = (np.ascontiguousarray(rt, dtype=np.float64), np.ascontiguousarray(th, dtype=np.int64),
           np.ascontiguousarray(req), np.ascontiguousarray(hr, dtype=bool))
    try:
        dataset._ct_replay_cache = out
    except AttributeError:
        pass
    return out


def missing_required(dataset) -> Tuple[str, ...]:
    present = set(_names_of(dataset))
    return tuple(a for a in cc.REQUIRED_COUNTERS if a not in present)


def assignments_of(space) -> np.ndarray:
    a = getattr(space, "assignments", None)
    if isinstance(a, np.ndarray):
        return a
    return np.array([c.assignment for c in space.configurations], dtype=np.float64)
