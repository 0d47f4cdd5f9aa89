"""The searcher's hot path behind the reference's Python API (search.py:38-399).

Same names, signatures, argument meaning and exceptions as the reference's
`countertune.search`; every numeric step runs in libct_b200.so on the GPU:

    score_configurations  -> ct_score       (Eq. 16, bit-exact FP64)
    normalize_scores      -> ct_normalize   (Eq. 17, x**8 within 1 ulp, as numpy's pow)
    weighted_select       -> ct_select      (exact prefix, certified draw)
    run_profile_search    -> ct_profile_search_launch (whole search on device)
                             for replayed datasets; otherwise the host drives
                             the measurement source and calls the device per
                             step (ct_analyze_react / ct_score / ...).
    run_random_search     -> ct_random_search_launch for replayed datasets.
"""

import copy
import shlex
import subprocess
from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Sequence, Set

import numpy as np

from . import _native
from . import counters as cc
from .counters import ArchProfile
from .errors import AnalysisError, CounterTuneError, SpaceExhaustedError
from .space import assignments_of, missing_required, replay_arrays

SCORE_EXPONENT = 8
SCORE_FLOOR = 0.0001
SCORE_CEILING = 256.0
DEFAULT_GAMMA = -0.25
DEFAULT_INNER_STEPS = 5
DEFAULT_INST_REACTION = 0.7
INSTRUCTION_BOUND_REACTION = 0.5
ISSUE_DELTA_SIGN = -1.0

STATUS_BUDGET = "budget"
STATUS_STOPPED = "stopped"
STATUS_EXHAUSTED = "exhausted"
_STATUS = {_native.CT_STATUS_BUDGET: STATUS_BUDGET, _native.CT_STATUS_STOPPED: STATUS_STOPPED,
           _native.CT_STATUS_EXHAUSTED: STATUS_EXHAUSTED}

MAX_SCORE_KEYS = 32


# --------------------------------------------------------------------- tables
class PredictionTable:
    """Model predictions for every configuration (search.py:38-63).

    matrix is n x counters float64 (row-major, as the reference keeps it); the
    device copy is column-major.  Counters a model omits are 0.
    """

    def __init__(self, space, counter_names: Sequence[str], matrix: np.ndarray):
        self.space = space
        self.counter_names = tuple(counter_names)
        self.column = {name: i for i, name in enumerate(self.counter_names)}
        self.matrix = matrix

    @classmethod
    def from_model_set(cls, models, space) -> "PredictionTable":
        models.check_space(space)
        names = tuple(models.counters)
        fast = getattr(models, "prediction_matrix", None)
        if fast is not None:
            return cls(space, names, fast(space))
        matrix = np.zeros((len(space), len(names)))
        for conf in space.configurations:
            predicted = models.predict(conf)
            for j, name in enumerate(names):
                matrix[conf.index, j] = predicted.get(name, 0.0)
        return cls(space, names, matrix)

    def delta_columns(self, keys: Sequence[str] = cc.DELTA_KEYS) -> List[int]:
        return [self.column.get(k, -1) for k in keys]


def _as_table(models, space) -> PredictionTable:
    if isinstance(models, PredictionTable) or (
            hasattr(models, "matrix") and hasattr(models, "column")):
        if models.space is not space and len(models.space) != len(space):
            raise CounterTuneError("prediction table was built for a different space")
        return models
    return PredictionTable.from_model_set(models, space)


class ExactModelSet:
    """Replays measured counters as predictions (models.py:372-410)."""

    family = "exact"

    def __init__(self, dataset):
        self.param_names = dataset.space.parameter_names
        self.param_binary = tuple(p.is_binary for p in dataset.space.parameters)
        self.source_arch = dataset.arch.name
        self.source_input = dataset.input_label
        self.counters = cc.modeled_counters(dataset)
        self._dataset = dataset

    def check_space(self, space) -> None:
        from .errors import ParameterMismatchError
        if (tuple(space.parameter_names) != tuple(self.param_names)
                or tuple(p.is_binary for p in space.parameters) != self.param_binary):
            raise ParameterMismatchError("replay table was built for a different parameter list")

    def prediction_matrix(self, space) -> np.ndarray:
        ds = self._dataset
        rt, th, _, hr = replay_arrays(ds)
        if not hr.all():
            missing = int(np.flatnonzero(~hr)[0])
            raise CounterTuneError(f"no measurement recorded for configuration {missing}")
        names = cc.dataset_counter_names(ds)
        n = len(ds.space)
        out = np.zeros((n, len(self.counters)))
        if hasattr(ds, "counter_matrix"):
            pos = {a: j for j, a in enumerate(ds.counter_names)}
            for j, a in enumerate(self.counters):
                out[:, j] = th.astype(np.float64) if a == cc.GLOBAL_THREADS else ds.counter_matrix[:, pos[a]]
        else:
            for rec in ds.records:
                out[rec.config_index] = [float(rec.global_threads) if a == cc.GLOBAL_THREADS
                                         else rec.counters[a] for a in self.counters]
        del names
        return out

    def predict(self, config) -> Dict[str, float]:
        row = self.prediction_matrix(self._dataset.space)[config.index]
        return dict(zip(self.counters, map(float, row)))


# ----------------------------------------------------------------- hot path
@dataclass
class ScoreVector:
    """Raw and normalized scores aligned with configuration indices."""

    raw: np.ndarray
    explored: np.ndarray
    norm: Optional[np.ndarray] = None
    scoreable: Optional[np.ndarray] = None

    def pool(self) -> np.ndarray:
        if self.scoreable is not None:
            return self.scoreable & ~self.explored
        return ~self.explored


def _ctx():
    return _native.context(0)


def _explored_mask(explored, n) -> np.ndarray:
    if isinstance(explored, np.ndarray) and explored.dtype == bool:
        return explored.copy()
    mask = np.zeros(n, dtype=bool)
    for idx in explored:
        mask[idx] = True
    return mask


def score_configurations(models, c_profile, delta: Dict[str, float], space,
                         explored: Iterable[int], literal_sign: bool = False,
                         score_top_k: Optional[int] = None) -> ScoreVector:
    """Eq. 16 for every unexplored configuration, on the GPU (search.py:89-141)."""
    table = _as_table(models, space)
    n = len(space)
    explored_mask = _explored_mask(explored, n)
    if score_top_k is not None and score_top_k < 0:
        raise ValueError("score_top_k must be >= 0")
    cols, vals = [], []
    for name, d in delta.items():
        j = table.column.get(name)
        if d == 0.0 or j is None:
            continue
        cols.append(j)
        vals.append(float(d))
    if len(cols) > MAX_SCORE_KEYS:
        raise ValueError(f"at most {MAX_SCORE_KEYS} scored counters are supported")
    ctx = _ctx()
    # keyed by the array objects: the host-driven, live and ask/tell loops
    # call this every outer iteration with the same table and space
    ctx.upload_table(table.matrix, key=table.matrix)
    if score_top_k is not None and score_top_k < int((~explored_mask).sum()):
        ctx.upload_space(assignments_of(space), key=space)
    raw, scoreable = ctx.score(c_profile.index, cols, vals, explored_mask, literal_sign,
                               score_top_k, n)
    return ScoreVector(raw=raw, explored=explored_mask, scoreable=scoreable)


def normalize_scores(scores: ScoreVector, gamma: float = DEFAULT_GAMMA) -> ScoreVector:
    """Eq. 17 weights in <0.0001, 256>, on the GPU (search.py:144-172)."""
    pool = scores.pool()
    if not pool.any():
        raise SpaceExhaustedError("no unexplored configurations to normalize")
    norm = _ctx().normalize(scores.raw, pool, gamma)
    return ScoreVector(raw=scores.raw, explored=scores.explored, norm=norm,
                       scoreable=scores.scoreable)


def weighted_select(scores: ScoreVector, rng: np.random.Generator) -> int:
    """Inverse-CDF draw on the GPU (search.py:175-185); consumes one rng.random()."""
    if scores.norm is None:
        raise ValueError("scores must be normalized before selection")
    weights = scores.norm
    if weights.size == 0:
        raise SpaceExhaustedError("every configuration is explored")
    state = rng.bit_generator.state
    u = rng.random()
    try:
        chosen, _ = _ctx().select(weights, u)
    except SpaceExhaustedError:
        rng.bit_generator.state = state   # the reference raises before drawing
        raise
    return chosen


# ------------------------------------------------------------ measurements
@dataclass
class Measurement:
    runtime_us: float
    global_threads: Optional[int] = None
    counters: Optional[Dict[str, float]] = None


class DatasetReplaySource:
    """Serves measurements from an exhaustive dataset (search.py:197-217)."""

    def __init__(self, dataset):
        self.dataset = dataset
        self.space = dataset.space
        self.arch = dataset.arch

    def measure(self, config_index: int, profiled: bool) -> Measurement:
        try:
            rec = self.dataset.record_for(config_index)
        except KeyError:
            raise CounterTuneError(f"dataset holds no measurement for configuration "
                                   f"{config_index}")
        if not profiled:
            return Measurement(runtime_us=rec.runtime_us)
        return Measurement(runtime_us=rec.runtime_us, global_threads=rec.global_threads,
                           counters=dict(rec.counters))

    def close(self) -> None:
        pass


class SubprocessMeasurementSource:
    """Live runner over the reference's line protocol (search.py:220-275)."""

    def __init__(self, command, space, arch: ArchProfile):
        self.space = space
        self.arch = arch
        if isinstance(command, str):
            command = shlex.split(command)
        self._proc = subprocess.Popen(command, stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                                      text=True, bufsize=1)

    def measure(self, config_index: int, profiled: bool) -> Measurement:
        conf = self.space.configurations[config_index]
        request = ",".join(repr(v) for v in conf.assignment) + f",{1 if profiled else 0}\n"
        self._proc.stdin.write(request)
        self._proc.stdin.flush()
        line = self._proc.stdout.readline()
        if not line:
            raise CounterTuneError("measurement runner closed its pipe")
        cells = line.strip().split(",")
        try:
            runtime = float(cells[0])
        except ValueError:
            raise CounterTuneError(f"runner sent a malformed runtime: {line.strip()!r}")
        if not profiled:
            return Measurement(runtime_us=runtime)
        if len(cells) < 2:
            raise CounterTuneError("profiled response is missing global_threads")
        threads = int(cells[1])
        counter_map: Dict[str, float] = {}
        for cell in cells[2:]:
            name, _, value = cell.partition("=")
            abbr, canonical = cc.canonicalize(name, float(value), self.arch)
            counter_map[abbr] = canonical
        return Measurement(runtime_us=runtime, global_threads=threads, counters=counter_map)

    def close(self) -> None:
        if self._proc.stdin:
            self._proc.stdin.close()
        self._proc.wait(timeout=10)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ------------------------------------------------------------------ traces
@dataclass
class TraceStep:
    step: int
    config_index: int
    runtime_us: float
    profiled: bool


@dataclass
class SearchTrace:
    """Every empirical test of one search, in execution order."""

    steps: List[TraceStep]
    seed: object
    status: str

    def runtimes(self) -> np.ndarray:
        return np.array([s.runtime_us for s in self.steps])

    def best_so_far(self) -> np.ndarray:
        return np.minimum.accumulate(self.runtimes())

    def completion_times_us(self, profiling_overhead: float = 1.0) -> np.ndarray:
        costs = np.array([s.runtime_us * (profiling_overhead if s.profiled else 1.0)
                          for s in self.steps])
        return np.cumsum(costs)

    def selected_indices(self) -> List[int]:
        seen: Set[int] = set()
        out = []
        for s in self.steps:
            if s.config_index not in seen:
                seen.add(s.config_index)
                out.append(s.config_index)
        return out


def _is_replay(source) -> bool:
    return isinstance(source, DatasetReplaySource) or (
        hasattr(source, "dataset") and type(source).__name__ == "DatasetReplaySource")


def _regenerable(seed) -> bool:
    return not isinstance(seed, (np.random.Generator, np.random.BitGenerator))


def stop_mask_of(stop_indices, n) -> Optional[np.ndarray]:
    if stop_indices is None:
        return None
    mask = np.zeros(n, dtype=np.uint8)
    for idx in stop_indices:
        if 0 <= idx < n:
            mask[idx] = 1
    return mask


def rep_error(code: int, failing_index: int) -> Exception:
    if code == _native.CT_ERR_NO_RECORD:
        return CounterTuneError(f"dataset holds no measurement for configuration {failing_index}")
    if code == _native.CT_ERR_EXHAUSTED:
        return SpaceExhaustedError("no unexplored configurations to normalize")
    if code == _native.CT_ERR_NONFINITE:
        return CounterTuneError("selection weights are not finite (negative or NaN predictions)")
    return CounterTuneError(f"device search failed with status {code}")


def trace_from_row(idx_row, prof_row, n_steps, status, runtime, seed) -> SearchTrace:
    steps = [TraceStep(step=k + 1, config_index=int(idx_row[k]),
                       runtime_us=float(runtime[idx_row[k]]), profiled=bool(prof_row[k]))
             for k in range(int(n_steps))]
    return SearchTrace(steps=steps, seed=seed, status=_STATUS[int(status)])


def run_random_search(source, seed=0, stop_indices: Optional[Set[int]] = None,
                      max_steps: Optional[int] = None) -> SearchTrace:
    """Uniform random search without replacement (search.py:317-335)."""
    n = len(source.space)
    if _is_replay(source) and _regenerable(seed):
        rt, th, req, hr = replay_arrays(source.dataset)
        ctx = _ctx()
        stop = stop_mask_of(stop_indices, n)
        ctx.upload_replay(rt, th, np.nan_to_num(req), hr, stop)
        ctx.launch_random(_native.SeedWords(seed, child_per_rep=False), 1, max_steps,
                          use_stop=stop is not None)
        idx, prof, nst, status, err, _ = ctx.fetch(1)
        if status[0] == _native.CT_STATUS_ERROR:
            raise rep_error(int(err[0]), int(idx[0, nst[0]]) if nst[0] < idx.shape[1] else -1)
        return trace_from_row(idx[0], prof[0], nst[0], status[0], rt, seed)
    # live sources: the permutation is the baseline's only computation
    rng = np.random.default_rng(seed)
    order = rng.permutation(n)
    if max_steps is not None:
        order = order[:max_steps]
    steps: List[TraceStep] = []
    status = STATUS_EXHAUSTED if max_steps is None or max_steps >= n else STATUS_BUDGET
    for pos, idx in enumerate(order, start=1):
        idx = int(idx)
        m = source.measure(idx, profiled=False)
        steps.append(TraceStep(step=pos, config_index=idx, runtime_us=m.runtime_us,
                               profiled=False))
        if stop_indices is not None and idx in stop_indices:
            status = STATUS_STOPPED
            break
    return SearchTrace(steps=steps, seed=seed, status=status)


def search_params(table: PredictionTable, arch, *, i, n, inst_reaction, literal_sign,
                  score_top_k, use_stop, gamma=DEFAULT_GAMMA,
                  issue_sign=ISSUE_DELTA_SIGN) -> "_native.SearchParams":
    p = _native.SearchParams()
    p.outer_iterations = int(i)
    p.inner_steps = int(n)
    p.inst_reaction = float(inst_reaction)
    p.issue_delta_sign = float(issue_sign)
    p.gamma = float(gamma)
    p.literal_sign = int(bool(literal_sign))
    p.score_top_k = -1 if score_top_k is None else int(score_top_k)
    p.use_stop = int(bool(use_stop))
    p.generation = cc.generation_code(arch)
    p.cores = int(arch.cores)
    for k, col in enumerate(table.delta_columns()):
        p.delta_columns[k] = col
    return p


def _check_inst_reaction(inst_reaction):
    if not 0.0 < inst_reaction < 1.0:
        raise ValueError(f"inst_reaction must lie in (0, 1), got {inst_reaction}")


def run_profile_search(source, models, *, i: int, n: int = DEFAULT_INNER_STEPS, seed=0,
                       inst_reaction: float = DEFAULT_INST_REACTION, literal_sign: bool = False,
                       stop_indices: Optional[Set[int]] = None,
                       score_top_k: Optional[int] = None) -> SearchTrace:
    """Alg. 1: i outer iterations of n biased draws (search.py:338-399)."""
    if i < 1:
        raise ValueError(f"need at least one outer iteration, got i={i}")
    if n < 0:
        raise ValueError(f"inner step count must be >= 0, got n={n}")
    space = source.space
    table = _as_table(models, space)
    total = len(space)
    if score_top_k is not None and score_top_k < 0:
        raise ValueError("score_top_k must be >= 0")
    if _is_replay(source) and _regenerable(seed):
        return _profile_search_device(source, table, i=i, n=n, seed=seed,
                                      inst_reaction=inst_reaction, literal_sign=literal_sign,
                                      stop_indices=stop_indices, score_top_k=score_top_k)
    return _profile_search_host_driven(source, table, total, i=i, n=n, seed=seed,
                                       inst_reaction=inst_reaction, literal_sign=literal_sign,
                                       stop_indices=stop_indices, score_top_k=score_top_k)


def _profile_search_device(source, table, *, i, n, seed, inst_reaction, literal_sign,
                           stop_indices, score_top_k=None) -> SearchTrace:
    ds = source.dataset
    N = len(source.space)
    rt, th, req, hr = replay_arrays(ds)
    missing = missing_required(ds)
    if missing:
        c0 = int(np.random.default_rng(seed).integers(0, N))
        if not hr[c0]:
            raise CounterTuneError(f"dataset holds no measurement for configuration {c0}")
        raise AnalysisError(f"counter map is missing {', '.join(missing)}")
    _check_inst_reaction(inst_reaction)
    stop = stop_mask_of(stop_indices, N)
    ctx = _ctx()
    ctx.upload_table(table.matrix, key=table.matrix)
    ctx.upload_replay(rt, th, req, hr, stop)
    if score_top_k is not None:
        ctx.upload_space(assignments_of(source.space), key=source.space)
    params = search_params(table, source.arch, i=i, n=n, inst_reaction=inst_reaction,
                           literal_sign=literal_sign, score_top_k=score_top_k,
                           use_stop=stop is not None)
    ctx.launch_profile(params, _native.SeedWords(seed, child_per_rep=False), 1)
    idx, prof, nst, status, err, _ = ctx.fetch(1)
    if status[0] == _native.CT_STATUS_ERROR:
        failing = int(idx[0, nst[0]]) if nst[0] < idx.shape[1] else -1
        raise rep_error(int(err[0]), failing)
    return trace_from_row(idx[0], prof[0], nst[0], status[0], rt, seed)


def _counters23(m: Measurement) -> np.ndarray:
    missing = [c for c in cc.REQUIRED_COUNTERS if c not in (m.counters or {})]
    if missing:
        raise AnalysisError(f"counter map is missing {', '.join(missing)}")
    return np.array([m.counters[c] for c in cc.REQUIRED_COUNTERS], dtype=np.float64)


def _profile_search_host_driven(source, table, total, *, i, n, seed, inst_reaction,
                                literal_sign, stop_indices, score_top_k) -> SearchTrace:
    """Live sources: the host owns measurement and the numpy Generator; the
    device runs the expert system, scoring, normalisation and every draw."""
    steps = _profile_search_steps(source.space, source.arch, table, total, i=i, n=n, seed=seed,
                                  inst_reaction=inst_reaction, literal_sign=literal_sign,
                                  stop_indices=stop_indices, score_top_k=score_top_k)
    try:
        request = next(steps)
        while True:
            request = steps.send(source.measure(*request))
    except StopIteration as done:
        return done.value


def _profile_search_batches(space, arch, table, total, *, i, n, seed, inst_reaction,
                            literal_sign, stop_indices, score_top_k, score_fn=None):
    """run_profile_search (search.py:338-399) as a generator of measurement
    batches: it yields ``(indices, profiled)`` -- the profiled configuration
    alone, then the n draws of the outer iteration together -- and is sent the
    Measurements of a prefix of the batch (all of it, or up to and including
    a configuration of the stop set); it returns the SearchTrace.

    The n draws of an iteration depend only on that iteration's weights and
    the Generator, not on the runtimes measured in between (search.py:388-398),
    so they can be made before any of them is measured: the RNG is consumed
    exactly as the reference's loop consumes it up to the end of the search
    (a stop ends the search before the extra draws could matter), and the
    recorded steps, the stop test and the later-ties-win argmin follow the
    reference's order.  That is what lets several GPUs time one iteration's
    candidates concurrently (dist_live.py)."""
    # A caller-owned Generator is drawn from through a private copy: the n
    # draws of an iteration are made before any is measured, so on an early
    # stop the copy has consumed draws the reference never makes.  The
    # caller's Generator is advanced by exactly the reference's draws when
    # the search ends (one integers(), then one random() per recorded draw;
    # random(k) consumes the stream as k single calls do).
    caller = seed if isinstance(seed, np.random.Generator) else None
    rng = (np.random.Generator(copy.deepcopy(caller.bit_generator)) if caller is not None
           else np.random.default_rng(seed))
    explored = np.zeros(total, dtype=bool)
    steps: List[TraceStep] = []
    c_profile = space.configurations[int(rng.integers(0, total))]
    ctx = _ctx()
    gen = cc.generation_code(arch)

    def record(idx: int, runtime: float, profiled: bool) -> bool:
        steps.append(TraceStep(step=len(steps) + 1, config_index=idx, runtime_us=runtime,
                               profiled=profiled))
        explored[idx] = True
        return stop_indices is not None and idx in stop_indices

    def finish(status: str) -> SearchTrace:
        if caller is not None:
            caller.integers(0, total)
            drawn = sum(1 for s in steps if not s.profiled)
            if drawn:
                caller.random(drawn)
        return SearchTrace(steps=steps, seed=seed, status=status)

    for _ in range(i):
        m = (yield ([c_profile.index], True))[0]
        if record(c_profile.index, m.runtime_us, True):
            return finish(STATUS_STOPPED)
        _check_inst_reaction(inst_reaction)
        _, deltas, _ = ctx.analyze_react(_counters23(m), gen, arch.cores,
                                         m.global_threads, inst_reaction)
        delta = dict(zip(cc.DELTA_KEYS, map(float, deltas)))
        if not (~explored).any():
            return finish(STATUS_EXHAUSTED)
        scores = (score_fn or score_configurations)(table, c_profile, delta, space, explored,
                                      literal_sign=literal_sign, score_top_k=score_top_k)
        scores = normalize_scores(scores)
        chosen: List[int] = []
        exhausted = False
        for _ in range(n):
            try:
                # zero total mass == norm.max() <= 0 (weights are 0 or >= 1e-4);
                # the draw is not consumed in that case
                c = weighted_select(scores, rng)
            except SpaceExhaustedError:
                exhausted = True
                break
            scores.norm[c] = 0.0
            chosen.append(c)
        got = (yield (chosen, False)) if chosen else []
        t_best = np.inf
        for c, meas in zip(chosen, got):
            if record(c, meas.runtime_us, False):
                return finish(STATUS_STOPPED)
            if meas.runtime_us <= t_best:
                t_best = meas.runtime_us
                c_profile = space.configurations[c]
        if len(got) < len(chosen):
            raise CounterTuneError("a measurement batch was cut short before a stop configuration")
        if exhausted:
            return finish(STATUS_EXHAUSTED)
    return finish(STATUS_BUDGET)


def _profile_search_steps(space, arch, table, total, *, i, n, seed, inst_reaction,
                          literal_sign, stop_indices, score_top_k):
    """The batch generator one empirical test at a time: yields
    (config_index, profiled), is sent each Measurement, returns the trace.
    Draws after a stop configuration are never measured."""
    core = _profile_search_batches(space, arch, table, total, i=i, n=n, seed=seed,
                                   inst_reaction=inst_reaction, literal_sign=literal_sign,
                                   stop_indices=stop_indices, score_top_k=score_top_k)
    try:
        batch, profiled = next(core)
        while True:
            got = []
            for idx in batch:
                got.append((yield (idx, profiled)))
                if stop_indices is not None and idx in stop_indices:
                    break
            batch, profiled = core.send(got)
    except StopIteration as done:
        return done.value


class ProfileSearcher:
    """Ask/tell form of the profile searcher (north_star's
    ``searcher.next_config`` / ``add_result``) for callers that own the
    measurement loop -- e.g. a tuner that times candidates itself, or the
    original KTT stub that talked "via files and sockets".

        s = ProfileSearcher(models, space, arch, i=40)
        while (req := s.next_config()) is not None:
            idx, profiled = req
            s.add_result(measure(idx, profiled))
        trace = s.trace

    It is the inversion of control of run_profile_search (same arguments,
    same RNG consumption, same trajectory); every numeric step runs on the
    GPU through libct_b200.so.
    """

    def __init__(self, models, space, arch, *, i: int, n: int = DEFAULT_INNER_STEPS, seed=0,
                 inst_reaction: float = DEFAULT_INST_REACTION, literal_sign: bool = False,
                 stop_indices: Optional[Set[int]] = None, score_top_k: Optional[int] = None):
        if i < 1:
            raise ValueError(f"need at least one outer iteration, got i={i}")
        if n < 0:
            raise ValueError(f"inner step count must be >= 0, got n={n}")
        self.space = space
        self.arch = arch
        table = _as_table(models, space)
        self._gen = _profile_search_steps(space, arch, table, len(space), i=i, n=n, seed=seed,
                                          inst_reaction=inst_reaction, literal_sign=literal_sign,
                                          stop_indices=stop_indices, score_top_k=score_top_k)
        self._pending = None
        self._trace: Optional[SearchTrace] = None
        self._advance(None, first=True)

    def _advance(self, value, first=False):
        try:
            self._pending = next(self._gen) if first else self._gen.send(value)
        except StopIteration as done:
            self._pending = None
            self._trace = done.value

    def next_config(self):
        """(config_index, profiled) of the next empirical test, or None when
        the search has finished (budget, stop set or exhausted space)."""
        return self._pending

    def add_result(self, measurement: Measurement) -> None:
        """Report the measurement of the configuration next_config() named.
        A profiled request needs runtime_us, global_threads and counters."""
        if self._pending is None:
            raise CounterTuneError("the search has finished; no measurement is pending")
        self._advance(measurement)

    @property
    def finished(self) -> bool:
        return self._pending is None

    @property
    def trace(self) -> SearchTrace:
        if self._trace is None:
            raise CounterTuneError("the search has not finished yet")
        return self._trace
