"""Replay experiments on the GPU (the reference's harness.py:49-398).

simulate() runs all R repetitions of one ExperimentSpec as ONE batched device
launch (one CTA per repetition, the numpy Generator streams regenerated on
the device from the master seed), or split over several GPUs by contiguous
repetition ranges.  Aggregation follows harness.py:187-244 operation for
operation, so reports are byte-identical to the reference's for the same
trajectories.
"""

import math
import os
import threading
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native
from . import counters as cc
from .counters import GLOBAL_THREADS
from .errors import AnalysisError, CounterTuneError
from .search import (DEFAULT_INST_REACTION, PredictionTable, _as_table, rep_error,
                     search_params)
from .space import assignments_of, missing_required, replay_arrays, well_performing_mask

WORKERS_ENV = "COUNTERTUNE_WORKERS"
SEARCHER_PROFILE = "profile"
SEARCHER_RANDOM = "random"
DEFAULT_REPETITIONS = 1000
DEFAULT_TIME_REPETITIONS = 100
DEFAULT_PROFILING_OVERHEAD = 3.0
TIME_GRID_POINTS = 100


@dataclass
class ExperimentSpec:
    """Everything one batch of simulated repetitions depends on (harness.py:49-96)."""

    dataset: object
    searcher: str = SEARCHER_RANDOM
    model: object = None
    name: str = "experiment"
    repetitions: int = DEFAULT_REPETITIONS
    inner_steps: int = 5
    outer_iterations: Optional[int] = None
    seed: int = 0
    slack: float = 1.1
    profiling_overhead: float = DEFAULT_PROFILING_OVERHEAD
    inst_reaction: float = DEFAULT_INST_REACTION
    literal_sign: bool = False
    score_top_k: Optional[int] = None
    time_repetitions: Optional[int] = None
    # extension: False replays every repetition for its full budget
    # (stop_indices=frozenset(), the throughput mode of BASELINE.md)
    stop_at_well_performing: bool = True

    def __post_init__(self):
        if self.searcher not in (SEARCHER_PROFILE, SEARCHER_RANDOM):
            raise ValueError(f"unknown searcher {self.searcher!r}")
        if self.repetitions < 1:
            raise ValueError("repetitions must be >= 1")
        if self.time_repetitions is not None and self.time_repetitions < 1:
            raise ValueError("time_repetitions must be >= 1")
        if self.slack < 1.0:
            raise ValueError("slack must be >= 1.0")
        if self.profiling_overhead < 1.0:
            raise ValueError("profiling_overhead must be >= 1.0")
        if self.inner_steps < 0:
            raise ValueError("inner_steps must be >= 0")
        if self.searcher == SEARCHER_PROFILE and self.model is None:
            raise ValueError("the profile searcher needs a model")

    def resolved_outer_iterations(self) -> int:
        if self.outer_iterations is not None:
            if self.outer_iterations < 1:
                raise ValueError("outer_iterations must be >= 1")
            return self.outer_iterations
        n = len(self.dataset.space)
        if self.inner_steps == 0:
            return n
        return max(1, math.ceil((n - 1) / self.inner_steps))


@dataclass
class ConvergenceReport:
    """Aggregated outcome of one experiment's repetitions (harness.py:98-132)."""

    name: str
    searcher: str
    dataset_label: str
    repetitions: int
    inner_steps: int
    outer_iterations: int
    seed: int
    slack: float
    profiling_overhead: float
    steps: np.ndarray
    censored: int
    mean_time_seconds: float
    step_curve_mean: np.ndarray
    step_curve_std: np.ndarray
    time_grid_seconds: np.ndarray
    time_curve_mean: np.ndarray
    time_curve_std: np.ndarray
    baseline_name: Optional[str] = None
    improvement: Optional[float] = None
    # device-side accounting of the run (not part of the reference's report)
    configs_scored: int = 0
    uncertified_draws: int = 0

    @property
    def mean_steps(self) -> float:
        return float(np.mean(self.steps))

    @property
    def median_steps(self) -> float:
        return float(np.median(self.steps))

    @property
    def stddev_steps(self) -> float:
        return float(np.std(self.steps))


def _worker_count() -> int:
    """COUNTERTUNE_WORKERS is validated as in the reference (harness.py:166-172);
    the device batch makes process fan-out unnecessary."""
    raw = os.environ.get(WORKERS_ENV, "1")
    try:
        workers = int(raw)
    except ValueError:
        raise CounterTuneError(f"{WORKERS_ENV} must be an integer, got {raw!r}")
    return max(1, workers)


@dataclass
class BatchResult:
    """Raw trajectories of R repetitions (rows), as the device returns them."""

    step_index: np.ndarray      # R x max_steps int32
    step_profiled: np.ndarray   # R x max_steps uint8
    n_steps: np.ndarray         # R int32
    status: np.ndarray          # R int32
    configs_scored: int
    uncertified: int
    draws: int
    algorithmic_bytes: int = 0


def prepare_device(ctx: "_native.Context", spec: ExperimentSpec, table=None):
    """Upload replay data, stop mask and (profile searcher) the prediction table."""
    ds = spec.dataset
    rt, th, req, hr = replay_arrays(ds)
    stop = well_performing_mask(ds, spec.slack)
    if not spec.stop_at_well_performing:
        stop[:] = False
    if spec.searcher == SEARCHER_RANDOM:
        # random search never reads counters; a dataset without some of them
        # has NaN columns there, which must not reach the device
        req = np.nan_to_num(req, nan=0.0, posinf=np.inf, neginf=-np.inf)
    # the profile searcher sees the counters as recorded (+-inf included, as
    # the reference's analyze() does; a missing counter raises below)
    ctx.upload_replay(rt, th, req, hr, stop.astype(np.uint8))
    params = None
    if spec.searcher == SEARCHER_PROFILE:
        missing = missing_required(ds)
        if missing:
            raise AnalysisError(f"counter map is missing {', '.join(missing)}")
        if table is None:
            table = _as_table(spec.model, ds.space)
        ctx.upload_table(table.matrix, key=table.matrix)
        if spec.score_top_k is not None:
            if spec.score_top_k < 0:
                raise ValueError("score_top_k must be >= 0")
            # top-K neighbourhoods (search.py:133-140, harness.py:155-158)
            ctx.upload_space(assignments_of(ds.space), key=ds.space)
        params = search_params(table, ds.arch, i=spec.resolved_outer_iterations(),
                               n=spec.inner_steps, inst_reaction=spec.inst_reaction,
                               literal_sign=spec.literal_sign, score_top_k=spec.score_top_k,
                               use_stop=True)
        if not 0.0 < spec.inst_reaction < 1.0:
            raise ValueError(f"inst_reaction must lie in (0, 1), got {spec.inst_reaction}")
    return params, rt


def launch(ctx, spec: ExperimentSpec, params, rep_offset: int, n_reps: int):
    seeds = _native.SeedWords(spec.seed, child_per_rep=True, rep_offset=rep_offset)
    if spec.searcher == SEARCHER_RANDOM:
        ctx.launch_random(seeds, n_reps, None, use_stop=True)
    else:
        ctx.launch_profile(params, seeds, n_reps)


def _launch_all(spec: ExperimentSpec, devices: Sequence[int], table=None):
    """Upload and launch every device's contiguous repetition range.

    Returns [(context, first_rep, n_reps)] in repetition order and the
    runtime vector; the launches are asynchronous."""
    R = spec.repetitions
    parts = np.array_split(np.arange(R), len(devices))
    if table is None and spec.searcher == SEARCHER_PROFILE:
        table = _as_table(spec.model, spec.dataset.space)
    launched = [None] * len(devices)
    errors = [None] * len(devices)
    runtime = [None]

    def work(k):
        try:
            # one context per entry, so a device listed twice gets two
            slot = devices[:k].count(devices[k])
            ctx = _native.context(devices[k], slot)
            params, rt = prepare_device(ctx, spec, table)
            runtime[0] = rt
            idxs = parts[k]
            if idxs.size == 0:
                return
            launch(ctx, spec, params, int(idxs[0]), int(idxs.size))
            launched[k] = (ctx, int(idxs[0]), int(idxs.size))
        except BaseException as exc:   # re-raised on the caller's thread
            errors[k] = exc

    if len(devices) == 1:
        work(0)
    else:
        threads = [threading.Thread(target=work, args=(k,)) for k in range(len(devices))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    for exc in errors:
        if exc is not None:
            raise exc
    return [x for x in launched if x is not None], runtime[0]


def run_batch(spec: ExperimentSpec, devices: Optional[Sequence[int]] = None,
              table=None) -> Tuple[BatchResult, np.ndarray]:
    """All repetitions of spec on the given GPUs (contiguous rep ranges),
    trajectories fetched to the host."""
    devices = list(devices) if devices else [0]
    launched, runtime = _launch_all(spec, devices, table)
    parts_ok = [ctx.fetch(n) for ctx, _, n in launched]
    width = max(r[0].shape[1] for r in parts_ok)

    def cat(j, dtype):
        rows = []
        for r in parts_ok:
            a = r[j]
            if a.ndim == 2 and a.shape[1] < width:
                a = np.pad(a, ((0, 0), (0, width - a.shape[1])))
            rows.append(a)
        return np.concatenate(rows).astype(dtype, copy=False)

    res = BatchResult(step_index=cat(0, np.int32), step_profiled=cat(1, np.uint8),
                      n_steps=cat(2, np.int32), status=cat(3, np.int32),
                      configs_scored=sum(r[5].configs_scored for r in parts_ok),
                      uncertified=sum(r[5].uncertified for r in parts_ok),
                      draws=sum(r[5].draws for r in parts_ok),
                      algorithmic_bytes=sum(r[5].algorithmic_bytes for r in parts_ok))
    err = cat(4, np.int32)
    bad = np.flatnonzero(res.status == _native.CT_STATUS_ERROR)
    if bad.size:
        r = int(bad[0])
        ns = int(res.n_steps[r])
        failing = int(res.step_index[r, ns]) if ns < res.step_index.shape[1] else -1
        raise rep_error(int(err[r]), failing)
    return res, runtime


def aggregate(spec: ExperimentSpec, res: BatchResult, runtime: np.ndarray) -> ConvergenceReport:
    """harness.py:187-244 on the device trajectories (same float operations)."""
    reps = spec.repetitions
    nst = res.n_steps.astype(np.int64)
    hit = res.status == _native.CT_STATUS_STOPPED
    idx = res.step_index
    valid = np.arange(idx.shape[1])[None, :] < nst[:, None]
    rts = np.where(valid, runtime[np.where(valid, idx, 0)], np.inf)
    overhead = spec.profiling_overhead
    costs = np.where(valid, rts * np.where(res.step_profiled.astype(bool), overhead, 1.0), 0.0)
    bsf_all = np.minimum.accumulate(rts, axis=1)
    times_all = np.cumsum(costs, axis=1)

    steps = nst.astype(float)
    censored = int(np.count_nonzero(~hit))
    total_times = times_all[np.arange(reps), nst - 1]

    max_len = int(nst.max())
    col_sum = np.zeros(max_len)
    col_sq = np.zeros(max_len)
    for r in range(reps):
        bsf = bsf_all[r, :nst[r]]
        padded = np.concatenate([bsf, np.full(max_len - nst[r], bsf[-1])])
        col_sum += padded
        col_sq += padded * padded
    mean = col_sum / reps
    var = np.maximum(0.0, col_sq / reps - mean * mean)
    step_std = np.sqrt(var)

    tr = reps if spec.time_repetitions is None else min(reps, spec.time_repetitions)
    t_start = max(float(times_all[r, 0]) for r in range(tr))
    t_end = max(float(times_all[r, nst[r] - 1]) for r in range(tr))
    if t_end > t_start:
        grid = np.linspace(t_start, t_end, TIME_GRID_POINTS)
    else:
        grid = np.array([t_start])
    tc_sum = np.zeros(grid.size)
    tc_sq = np.zeros(grid.size)
    for r in range(tr):
        times = times_all[r, :nst[r]]
        bsf = bsf_all[r, :nst[r]]
        pos = np.searchsorted(times, grid, side="right") - 1
        sampled = bsf[np.clip(pos, 0, len(bsf) - 1)]
        tc_sum += sampled
        tc_sq += sampled * sampled
    tmean = tc_sum / tr
    tvar = np.maximum(0.0, tc_sq / tr - tmean * tmean)
    ds = spec.dataset
    return ConvergenceReport(
        name=spec.name, searcher=spec.searcher,
        dataset_label=f"{ds.arch.name}/{ds.input_label}", repetitions=reps,
        inner_steps=spec.inner_steps, outer_iterations=spec.resolved_outer_iterations(),
        seed=spec.seed, slack=spec.slack, profiling_overhead=spec.profiling_overhead,
        steps=steps, censored=censored, mean_time_seconds=float(np.mean(total_times)) / 1e6,
        step_curve_mean=mean, step_curve_std=step_std, time_grid_seconds=grid / 1e6,
        time_curve_mean=tmean, time_curve_std=np.sqrt(tvar),
        configs_scored=int(res.configs_scored), uncertified_draws=int(res.uncertified))


def simulate(spec: ExperimentSpec, devices: Optional[Sequence[int]] = None) -> ConvergenceReport:
    """Run the repetitions on the GPU(s) and aggregate (harness.py:175-244).

    The trajectories never leave the GPU: the report's sums are taken on the
    device in the reference's order (ct_aggregate_steps / ct_aggregate_time,
    chained across devices in repetition order), so only O(R + steps)
    numbers come back and the report is byte-identical to aggregate() on the
    fetched trajectories."""
    _worker_count()
    devices = list(devices) if devices else [0]
    launched, _ = _launch_all(spec, devices)
    reps = spec.repetitions
    if len(launched) == 1:
        return _report_one_device(spec, launched[0][0])
    nst_l, status_l, scored, uncert = [], [], 0, 0
    for ctx, first, n in launched:
        nst, status, err, stats = ctx.fetch_status(n)
        bad = np.flatnonzero(status == _native.CT_STATUS_ERROR)
        if bad.size:
            r = int(bad[0])
            raise rep_error(int(err[r]), ctx.failing_index(r, n))
        nst_l.append(nst)
        status_l.append(status)
        scored += stats.configs_scored
        uncert += stats.uncertified
    nst = np.concatenate(nst_l).astype(np.int64)
    status = np.concatenate(status_l)
    max_len = int(nst.max())

    col_sum = col_sq = None
    totals, firsts = [], []
    for ctx, first, n in launched:
        col_sum, col_sq, tot, fst = ctx.aggregate_steps(spec.profiling_overhead, n, max_len,
                                                        col_sum, col_sq)
        totals.append(tot)
        firsts.append(fst)
    total_times = np.concatenate(totals)
    first_times = np.concatenate(firsts)
    mean = col_sum / reps
    var = np.maximum(0.0, col_sq / reps - mean * mean)
    step_std = np.sqrt(var)

    tr = reps if spec.time_repetitions is None else min(reps, spec.time_repetitions)
    # max of floats is exact in any order (harness.py:207-210 takes Python's max)
    t_start = float(np.max(first_times[:tr]))
    t_end = float(np.max(total_times[:tr]))
    if t_end > t_start:
        grid = np.linspace(t_start, t_end, TIME_GRID_POINTS)
    else:
        grid = np.array([t_start])
    tc_sum = tc_sq = None
    for ctx, first, n in launched:
        count = min(n, max(0, tr - first))
        if count == 0:
            continue
        tc_sum, tc_sq = ctx.aggregate_time(count, grid, tc_sum, tc_sq)
    tmean = tc_sum / tr
    tvar = np.maximum(0.0, tc_sq / tr - tmean * tmean)
    ds = spec.dataset
    return ConvergenceReport(
        name=spec.name, searcher=spec.searcher,
        dataset_label=f"{ds.arch.name}/{ds.input_label}", repetitions=reps,
        inner_steps=spec.inner_steps, outer_iterations=spec.resolved_outer_iterations(),
        seed=spec.seed, slack=spec.slack, profiling_overhead=spec.profiling_overhead,
        steps=nst.astype(float), censored=int(np.count_nonzero(status != _native.CT_STATUS_STOPPED)),
        mean_time_seconds=float(np.mean(total_times)) / 1e6,
        step_curve_mean=mean, step_curve_std=step_std, time_grid_seconds=grid / 1e6,
        time_curve_mean=tmean, time_curve_std=np.sqrt(tvar),
        configs_scored=int(scored), uncertified_draws=int(uncert))


def _report_one_device(spec: ExperimentSpec, ctx) -> ConvergenceReport:
    """simulate() of a launch on one device: the report's sums, maxima and
    time grid come back from one ct_report call (one synchronisation); the
    final divisions are the reference's numpy operations (harness.py:202-224)."""
    reps = spec.repetitions
    tr = reps if spec.time_repetitions is None else min(reps, spec.time_repetitions)
    out = ctx.report(spec.profiling_overhead, reps, tr)
    status = out["status"]
    bad = np.flatnonzero(status == _native.CT_STATUS_ERROR)
    if bad.size:
        r = int(bad[0])
        raise rep_error(int(out["rep_error"][r]), ctx.failing_index(r, reps))
    nst = out["n_steps"].astype(np.int64)
    mean = out["col_sum"] / reps
    var = np.maximum(0.0, out["col_sq"] / reps - mean * mean)
    tmean = out["tc_sum"] / tr
    tvar = np.maximum(0.0, out["tc_sq"] / tr - tmean * tmean)
    ds = spec.dataset
    stats = out["stats"]
    return ConvergenceReport(
        name=spec.name, searcher=spec.searcher,
        dataset_label=f"{ds.arch.name}/{ds.input_label}", repetitions=reps,
        inner_steps=spec.inner_steps, outer_iterations=spec.resolved_outer_iterations(),
        seed=spec.seed, slack=spec.slack, profiling_overhead=spec.profiling_overhead,
        steps=nst.astype(float), censored=int(np.count_nonzero(status != _native.CT_STATUS_STOPPED)),
        mean_time_seconds=float(np.mean(out["total"])) / 1e6,
        step_curve_mean=mean, step_curve_std=np.sqrt(var), time_grid_seconds=out["grid"] / 1e6,
        time_curve_mean=tmean, time_curve_std=np.sqrt(tvar),
        configs_scored=int(stats.configs_scored), uncertified_draws=int(stats.uncertified))


def simulate_host_aggregate(spec: ExperimentSpec,
                            devices: Optional[Sequence[int]] = None) -> ConvergenceReport:
    """simulate() with the trajectories fetched and aggregated on the host
    (aggregate()); the device-aggregation path is checked against it."""
    _worker_count()
    res, runtime = run_batch(spec, devices)
    return aggregate(spec, res, runtime)


def pair_with_baseline(candidate: ConvergenceReport,
                       baseline: ConvergenceReport) -> ConvergenceReport:
    if candidate.repetitions != baseline.repetitions:
        raise ValueError("improvement factors require identical repetition counts")
    candidate.baseline_name = baseline.name
    candidate.improvement = baseline.mean_steps / candidate.mean_steps
    return candidate


def _fmt(value) -> str:
    if value is None:
        return ""
    if isinstance(value, float):
        return repr(value)
    return str(value)


def _safe_name(name: str) -> str:
    return "".join(ch if ch.isalnum() or ch in "-_" else "-" for ch in name)


SUMMARY_COLUMNS = ("name", "searcher", "dataset", "repetitions", "n", "i", "seed",
                   "slack", "profiling_overhead", "mean_steps", "median_steps",
                   "stddev_steps", "censored", "mean_time_seconds",
                   "improvement_vs_baseline", "baseline")


def report(reports: List[ConvergenceReport], out_dir) -> List[str]:
    """summary.csv + per-experiment curves, byte-stable (harness.py:344-388)."""
    os.makedirs(out_dir, exist_ok=True)
    written = []
    lines = [",".join(SUMMARY_COLUMNS)]
    for rep in reports:
        lines.append(",".join([
            rep.name, rep.searcher, rep.dataset_label, str(rep.repetitions),
            str(rep.inner_steps), str(rep.outer_iterations), str(rep.seed),
            _fmt(rep.slack), _fmt(rep.profiling_overhead), _fmt(rep.mean_steps),
            _fmt(rep.median_steps), _fmt(rep.stddev_steps), str(rep.censored),
            _fmt(rep.mean_time_seconds), _fmt(rep.improvement), rep.baseline_name or "",
        ]))
    path = os.path.join(out_dir, "summary.csv")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")
    written.append(path)
    for rep in reports:
        base = _safe_name(rep.name)
        rows = ["step,mean,stddev"]
        for i in range(rep.step_curve_mean.size):
            rows.append(f"{i + 1},{_fmt(float(rep.step_curve_mean[i]))},"
                        f"{_fmt(float(rep.step_curve_std[i]))}")
        path = os.path.join(out_dir, f"curve_{base}.csv")
        with open(path, "w", encoding="utf-8", newline="\n") as fh:
            fh.write("\n".join(rows) + "\n")
        written.append(path)
        rows = ["seconds,mean,stddev"]
        for i in range(rep.time_grid_seconds.size):
            rows.append(f"{_fmt(float(rep.time_grid_seconds[i]))},"
                        f"{_fmt(float(rep.time_curve_mean[i]))},"
                        f"{_fmt(float(rep.time_curve_std[i]))}")
        path = os.path.join(out_dir, f"curve_{base}_time.csv")
        with open(path, "w", encoding="utf-8", newline="\n") as fh:
            fh.write("\n".join(rows) + "\n")
        written.append(path)
    return written


@dataclass
class CrossEvalReport:
    """Model portability check against a dataset it was not trained on
    (harness.py:257-265)."""

    model_label: str
    dataset_label: str
    counter_errors: Dict[str, Tuple[float, float]]
    profile_report: ConvergenceReport
    random_report: ConvergenceReport


def counter_prediction_errors(models, dataset) -> Dict[str, Tuple[float, float]]:
    """Per-counter (MAE, RMSE) over all records (harness.py:268-289)."""
    table = PredictionTable.from_model_set(models, dataset.space)
    rt, th, _, hr = replay_arrays(dataset)
    names = getattr(dataset, "counter_names", None)
    errors: Dict[str, Tuple[float, float]] = {}
    for abbr in table.counter_names:
        col = table.column[abbr]
        measured, predicted = [], []
        for rec in dataset.records:
            if abbr == GLOBAL_THREADS:
                measured.append(float(rec.global_threads))
            elif abbr in rec.counters:
                measured.append(rec.counters[abbr])
            else:
                continue
            predicted.append(table.matrix[rec.config_index, col])
        if not measured:
            continue
        err = np.array(predicted) - np.array(measured)
        errors[abbr] = (float(np.mean(np.abs(err))), float(math.sqrt(np.mean(err * err))))
    del rt, th, hr, names
    return errors


def cross_evaluate(models, dataset, repetitions: int = DEFAULT_REPETITIONS,
                   inner_steps: int = 5, outer_iterations: Optional[int] = None,
                   seed: int = 0, slack: float = 1.1,
                   profiling_overhead: float = DEFAULT_PROFILING_OVERHEAD,
                   inst_reaction: float = DEFAULT_INST_REACTION,
                   devices: Optional[Sequence[int]] = None) -> CrossEvalReport:
    """Judge a foreign model on this dataset (harness.py:292-323): its
    per-counter prediction errors over every record, and the profile searcher
    it drives against the uniform-random baseline with the same seeds.

    The model's prediction table is evaluated on the GPU (ct_model_predict)
    and both searchers run as batched device launches (simulate); the
    report is the reference's, field for field."""
    errors = counter_prediction_errors(models, dataset)
    profile_spec = ExperimentSpec(dataset=dataset, searcher=SEARCHER_PROFILE, model=models,
                                  name="profile-foreign-model", repetitions=repetitions,
                                  inner_steps=inner_steps, outer_iterations=outer_iterations,
                                  seed=seed, slack=slack,
                                  profiling_overhead=profiling_overhead,
                                  inst_reaction=inst_reaction)
    random_spec = ExperimentSpec(dataset=dataset, searcher=SEARCHER_RANDOM,
                                 name="random-baseline", repetitions=repetitions,
                                 seed=seed, slack=slack,
                                 profiling_overhead=profiling_overhead)
    profile_report = simulate(profile_spec, devices)
    random_report = simulate(random_spec, devices)
    pair_with_baseline(profile_report, random_report)
    model_label = getattr(models, "source_arch", "?")
    model_input = getattr(models, "source_input", "?")
    return CrossEvalReport(model_label=f"{model_label}/{model_input}",
                           dataset_label=f"{dataset.arch.name}/{dataset.input_label}",
                           counter_errors=errors,
                           profile_report=profile_report,
                           random_report=random_report)


def write_counter_errors(errors: Dict[str, Tuple[float, float]], path) -> None:
    """counter_errors.csv, catalog order, repr floats (harness.py:391-398)."""
    lines = ["counter,mae,rmse"]
    for abbr in cc.ABBREVIATIONS:
        if abbr in errors:
            mae, rmse = errors[abbr]
            lines.append(f"{abbr},{repr(mae)},{repr(rmse)}")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")
