"""ctypes binding of libct_b200.so (include/countertune_b200.h).

The library is the only compute path: importing this module fails loudly if
it has not been built (``python -c "import __graft_entry__ as g; g.build()"``)
and every call that needs a GPU raises if no CUDA device is present.  There is
no CPU fallback.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import (CounterTuneError, SpaceExhaustedError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libct_b200.so"
LIB_PATH = os.environ.get("CT_LIB_PATH") or os.path.join(_HERE, LIB_NAME)

CT_OK = 0
CT_ERR_CUDA = -1
CT_ERR_VALUE = -2
CT_ERR_EXHAUSTED = -3
CT_ERR_NO_RECORD = -4
CT_ERR_MISMATCH = -5
CT_ERR_STATE = -6
CT_ERR_NONFINITE = -7
CT_ERR_UNSUPPORTED = -8

CT_STATUS_BUDGET = 0
CT_STATUS_STOPPED = 1
CT_STATUS_EXHAUSTED = 2
CT_STATUS_ERROR = 3

N_DELTA = 18
N_REQUIRED = 23

_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_P = ctypes.POINTER


class SearchParams(ctypes.Structure):
    """ct_search_params"""
    _fields_ = [
        ("outer_iterations", _i32),
        ("inner_steps", _i32),
        ("inst_reaction", _dbl),
        ("issue_delta_sign", _dbl),
        ("gamma", _dbl),
        ("literal_sign", _i32),
        ("score_top_k", _i64),
        ("use_stop", _i32),
        ("generation", _i32),
        ("cores", _i64),
        ("delta_columns", _i32 * N_DELTA),
    ]


class SeedSpec(ctypes.Structure):
    """ct_seed_spec"""
    _fields_ = [
        ("entropy", _P(ctypes.c_uint32)),
        ("n_entropy", _i32),
        ("spawn_prefix", _P(ctypes.c_uint32)),
        ("n_prefix", _i32),
        ("child_per_rep", _i32),
        ("rep_offset", _i64),
    ]


class BatchStats(ctypes.Structure):
    """ct_batch_stats"""
    _fields_ = [
        ("configs_scored", _i64),
        ("draws", _i64),
        ("uncertified", _i64),
        ("outer_iterations", _i64),
        ("algorithmic_bytes", _i64),
    ]


class ModelProgramC(ctypes.Structure):
    """ct_model_program"""
    _fields_ = [
        ("n_cols", _i32), ("n_nodes", _i32), ("n_models", _i32), ("n_terms", _i32),
        ("n_binary", _i32),
        ("node_feature", _vp), ("node_left", _vp), ("node_right", _vp),
        ("node_threshold", _vp), ("node_value", _vp), ("col_root", _vp),
        ("col_model_first", _vp), ("col_model_count", _vp), ("model_key", _vp),
        ("model_term_first", _vp), ("model_term_count", _vp), ("term_kind", _vp),
        ("term_p1", _vp), ("term_p2", _vp), ("term_coef", _vp), ("binary_pos", _vp),
    ]


# name -> (restype, argtypes); the exported surface of include/countertune_b200.h
SIGNATURES = {
    "ct_abi_version": (ctypes.c_int, []),
    "ct_last_error": (ctypes.c_char_p, []),
    "ct_device_count": (ctypes.c_int, [_P(ctypes.c_int)]),
    "ct_create": (ctypes.c_int, [ctypes.c_int, _P(_vp)]),
    "ct_destroy": (ctypes.c_int, [_vp]),
    "ct_set_stream": (ctypes.c_int, [_vp, _vp]),
    "ct_synchronize": (ctypes.c_int, [_vp]),
    "ct_table_upload": (ctypes.c_int, [_vp, _vp, _i64, _i32]),
    "ct_space_upload": (ctypes.c_int, [_vp, _vp, _i64, _i32]),
    "ct_replay_upload": (ctypes.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "ct_score": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i32, _vp, _i32, _i64, _vp, _vp,
                                _P(_i32)]),
    "ct_normalize": (ctypes.c_int, [_vp, _vp, _vp, _i64, _dbl, _vp]),
    "ct_select": (ctypes.c_int, [_vp, _vp, _i64, _dbl, _P(_i64), _P(_i32)]),
    "ct_profile_search_launch": (ctypes.c_int, [_vp, _P(SearchParams), _P(SeedSpec), _i32]),
    "ct_random_search_launch": (ctypes.c_int, [_vp, _P(SeedSpec), _i32, _i64, _i32]),
    "ct_result_max_steps": (ctypes.c_int, [_vp, _P(_i64)]),
    "ct_fetch_results": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _P(BatchStats)]),
    "ct_result_device_ptrs": (ctypes.c_int, [_vp, _P(_vp), _P(_vp), _P(_vp), _P(_vp)]),
    "ct_analyze_react": (ctypes.c_int, [_vp, _vp, _i32, _i64, _i64, _dbl, _dbl, _vp]),
    "ct_check_division": (ctypes.c_int, [_vp, _i64, ctypes.c_uint64, _P(_i64), _vp]),
    "ct_model_predict": (ctypes.c_int, [_vp, _P(ModelProgramC), _vp, _i64, _i32, _vp]),
    "ct_aggregate_steps": (ctypes.c_int, [_vp, _dbl, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ct_aggregate_time": (ctypes.c_int, [_vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp]),
    "ct_report": (ctypes.c_int, [_vp, _dbl, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp, _vp]),
}

_lib = None
_lib_lock = threading.Lock()


def library(path: str = LIB_PATH):
    """Load libct_b200.so (no GPU needed to load it)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(path):
                raise CounterTuneError(
                    f"CUDA extension {LIB_NAME} is not built at {path}; run "
                    f"`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def _raise(code: int, exc_map=None):
    msg = library().ct_last_error().decode("utf-8", "replace")
    if exc_map and code in exc_map:
        raise exc_map[code](msg)
    if code == CT_ERR_VALUE:
        raise ValueError(msg)
    if code == CT_ERR_EXHAUSTED:
        raise SpaceExhaustedError(msg)
    raise CounterTuneError(msg)


def check(code: int, exc_map=None) -> None:
    if code != CT_OK:
        _raise(code, exc_map)


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


class Context:
    """One ct_ctx (one GPU).  Not thread-safe; one per device per thread."""

    def __init__(self, device: int = 0):
        lib = library()
        count = ctypes.c_int(0)
        rc = lib.ct_device_count(ctypes.byref(count))
        if rc != CT_OK or count.value < 1:
            raise CounterTuneError(
                "no CUDA device available: the countertune-b200 hot path runs only on the GPU")
        handle = ctypes.c_void_p()
        check(lib.ct_create(device, ctypes.byref(handle)))
        self.device = device
        self.handle = handle
        self._table_key = None
        self._replay_key = None
        self._space_key = None

    def close(self):
        if self.handle:
            library().ct_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- stream ----------------------------------------------------------
    def set_stream(self, cuda_stream_ptr):
        check(library().ct_set_stream(self.handle, ctypes.c_void_p(cuda_stream_ptr or 0)))

    def synchronize(self):
        check(library().ct_synchronize(self.handle))

    # -- resident inputs ---------------------------------------------------
    def upload_table(self, matrix: np.ndarray, key=None):
        """key: an object identifying the contents (e.g. the array itself);
        a call with the object the last upload was keyed by is a no-op.  The
        context holds the key, so its identity cannot be reused meanwhile."""
        if key is not None and key is self._table_key:
            return
        m = np.ascontiguousarray(matrix, dtype=np.float64)
        check(library().ct_table_upload(self.handle, ptr(m), m.shape[0], m.shape[1]))
        self._table_key = key

    def upload_space(self, assignments: np.ndarray, key=None):
        if key is not None and key is self._space_key:
            return
        a = np.ascontiguousarray(assignments, dtype=np.float64)
        check(library().ct_space_upload(self.handle, ptr(a), a.shape[0], a.shape[1]))
        self._space_key = key

    def upload_replay(self, runtime, threads, counters, has_record, stop_mask=None, key=None):
        if key is not None and key is self._replay_key:
            return
        rt = np.ascontiguousarray(runtime, dtype=np.float64)
        th = np.ascontiguousarray(threads, dtype=np.int64)
        cm = np.ascontiguousarray(counters, dtype=np.float64)
        hr = np.ascontiguousarray(has_record, dtype=np.uint8)
        sm = None if stop_mask is None else np.ascontiguousarray(stop_mask, dtype=np.uint8)
        if cm.shape != (rt.size, N_REQUIRED):
            raise ValueError(f"counters must be n x {N_REQUIRED}")
        check(library().ct_replay_upload(self.handle, rt.size, ptr(rt), ptr(th), ptr(cm),
                                         ptr(hr), ptr(sm)))
        self._replay_key = key

    # -- single-call hot path -----------------------------------------------
    def score(self, profile_index, delta_columns, delta_values, explored, literal_sign,
              score_top_k, n):
        cols = np.ascontiguousarray(delta_columns, dtype=np.int32)
        vals = np.ascontiguousarray(delta_values, dtype=np.float64)
        expl = np.ascontiguousarray(explored, dtype=np.uint8)
        raw = np.empty(n, dtype=np.float64)
        scoreable = np.empty(n, dtype=np.uint8)
        has = ctypes.c_int32(0)
        check(library().ct_score(self.handle, int(profile_index), ptr(cols), ptr(vals),
                                 cols.size, ptr(expl), int(bool(literal_sign)),
                                 -1 if score_top_k is None else int(score_top_k),
                                 ptr(raw), ptr(scoreable), ctypes.byref(has)))
        return raw, (scoreable.astype(bool) if has.value else None)

    def normalize(self, raw, pool, gamma):
        r = np.ascontiguousarray(raw, dtype=np.float64)
        p = np.ascontiguousarray(pool, dtype=np.uint8)
        out = np.empty_like(r)
        check(library().ct_normalize(self.handle, ptr(r), ptr(p), r.size, float(gamma),
                                     ptr(out)))
        return out

    def select(self, norm, u):
        w = np.ascontiguousarray(norm, dtype=np.float64)
        chosen = ctypes.c_int64(-1)
        cert = ctypes.c_int32(0)
        check(library().ct_select(self.handle, ptr(w), w.size, float(u), ctypes.byref(chosen),
                                  ctypes.byref(cert)))
        return int(chosen.value), bool(cert.value)

    def analyze_react(self, counters23, generation, cores, global_threads, inst_reaction,
                      issue_sign=-1.0):
        c = np.ascontiguousarray(counters23, dtype=np.float64)
        out = np.empty(2 * N_DELTA + 1, dtype=np.float64)
        check(library().ct_analyze_react(self.handle, ptr(c), int(generation), int(cores),
                                         int(global_threads), float(inst_reaction),
                                         float(issue_sign), ptr(out)))
        return out[:N_DELTA], out[N_DELTA:2 * N_DELTA], bool(out[2 * N_DELTA])

    def check_division(self, n: int, seed: int = 1, samples: bool = False):
        out = ctypes.c_int64(-1)
        first = np.zeros(16)
        check(library().ct_check_division(self.handle, int(n), int(seed), ctypes.byref(out),
                                          ptr(first)))
        return (int(out.value), first.reshape(4, 4)) if samples else int(out.value)

    # -- batched replay searches ----------------------------------------------
    def launch_profile(self, params: SearchParams, seeds: "SeedWords", n_reps: int):
        spec = seeds.spec()
        check(library().ct_profile_search_launch(self.handle, ctypes.byref(params),
                                                 ctypes.byref(spec), int(n_reps)))

    def launch_random(self, seeds: "SeedWords", n_reps: int, max_steps=None, use_stop=True):
        spec = seeds.spec()
        check(library().ct_random_search_launch(self.handle, ctypes.byref(spec), int(n_reps),
                                                -1 if max_steps is None else int(max_steps),
                                                int(bool(use_stop))))

    def fetch(self, n_reps: int, want_profiled=True):
        ms = ctypes.c_int64(0)
        check(library().ct_result_max_steps(self.handle, ctypes.byref(ms)))
        m = ms.value
        idx = np.empty((n_reps, m), dtype=np.int32)
        prof = np.empty((n_reps, m), dtype=np.uint8) if want_profiled else None
        nst = np.empty(n_reps, dtype=np.int32)
        status = np.empty(n_reps, dtype=np.int32)
        err = np.empty(n_reps, dtype=np.int32)
        stats = BatchStats()
        check(library().ct_fetch_results(self.handle, ptr(idx), ptr(prof), ptr(nst),
                                         ptr(status), ptr(err), ctypes.byref(stats)))
        return idx, prof, nst, status, err, stats

    def model_predict(self, prog, assignments: np.ndarray) -> np.ndarray:
        """ct_model_predict: the n x n_cols table (also left resident on the
        device as the context's prediction table)."""
        a = np.ascontiguousarray(assignments, dtype=np.float64)
        arrays = {f: np.ascontiguousarray(getattr(prog, f)) for f in (
            "node_feature", "node_left", "node_right", "node_threshold", "node_value",
            "col_root", "col_model_first", "col_model_count", "model_key", "model_term_first",
            "model_term_count", "term_kind", "term_p1", "term_p2", "term_coef", "binary_pos")}
        c = ModelProgramC()
        c.n_cols, c.n_nodes = prog.n_cols, arrays["node_feature"].size
        c.n_models, c.n_terms = arrays["model_key"].size, arrays["term_kind"].size
        c.n_binary = arrays["binary_pos"].size
        for f, arr in arrays.items():
            setattr(c, f, arr.ctypes.data if arr.size else None)
        out = np.empty((a.shape[0], prog.n_cols), dtype=np.float64)
        check(library().ct_model_predict(self.handle, ctypes.byref(c), ptr(a), a.shape[0],
                                         a.shape[1], ptr(out)))
        self._table_key = None
        return out

    def fetch_status(self, n_reps: int):
        """n_steps, status, rep_error and stats of the last launch (no trajectories)."""
        nst = np.empty(n_reps, dtype=np.int32)
        status = np.empty(n_reps, dtype=np.int32)
        err = np.empty(n_reps, dtype=np.int32)
        stats = BatchStats()
        check(library().ct_fetch_results(self.handle, None, None, ptr(nst), ptr(status),
                                         ptr(err), ctypes.byref(stats)))
        return nst, status, err, stats

    def failing_index(self, rep: int, n_reps: int) -> int:
        """Configuration index a repetition stopped on with an error."""
        idx, _, nst, _, _, _ = self.fetch(n_reps, want_profiled=False)
        return int(idx[rep, nst[rep]]) if nst[rep] < idx.shape[1] else -1

    def aggregate_steps(self, overhead: float, n_reps: int, max_len: int, sum0=None, sq0=None):
        """(col_sum, col_sq, total_times, first_times) of the last launch."""
        col_sum = np.empty(max_len)
        col_sq = np.empty(max_len)
        total = np.empty(n_reps)
        first = np.empty(n_reps)
        s0 = None if sum0 is None else np.ascontiguousarray(sum0, dtype=np.float64)
        q0 = None if sq0 is None else np.ascontiguousarray(sq0, dtype=np.float64)
        check(library().ct_aggregate_steps(self.handle, float(overhead), int(max_len), ptr(s0),
                                           ptr(q0), ptr(col_sum), ptr(col_sq), ptr(total),
                                           ptr(first)))
        return col_sum, col_sq, total, first

    def aggregate_time(self, time_reps: int, grid: np.ndarray, sum0=None, sq0=None):
        g = np.ascontiguousarray(grid, dtype=np.float64)
        out_s = np.empty(g.size)
        out_q = np.empty(g.size)
        s0 = None if sum0 is None else np.ascontiguousarray(sum0, dtype=np.float64)
        q0 = None if sq0 is None else np.ascontiguousarray(sq0, dtype=np.float64)
        check(library().ct_aggregate_time(self.handle, int(time_reps), ptr(g), g.size, ptr(s0),
                                          ptr(q0), ptr(out_s), ptr(out_q)))
        return out_s, out_q

    def report(self, overhead: float, n_reps: int, time_reps: int):
        """ct_report: everything harness.simulate aggregates, one sync."""
        msv = ctypes.c_int64(0)
        check(library().ct_result_max_steps(self.handle, ctypes.byref(msv)))
        ms = msv.value
        nst = np.empty(n_reps, dtype=np.int32)
        status = np.empty(n_reps, dtype=np.int32)
        err = np.empty(n_reps, dtype=np.int32)
        stats = BatchStats()
        max_len = ctypes.c_int32()
        n_grid = ctypes.c_int32()
        col_sum = np.empty(ms)
        col_sq = np.empty(ms)
        total = np.empty(n_reps)
        grid = np.empty(100)
        tcs = np.empty(100)
        tcq = np.empty(100)
        check(library().ct_report(self.handle, float(overhead), int(time_reps), ptr(nst),
                                  ptr(status), ptr(err), ctypes.byref(stats),
                                  ctypes.byref(max_len), ptr(col_sum), ptr(col_sq), ptr(total),
                                  ctypes.byref(n_grid), ptr(grid), ptr(tcs), ptr(tcq)))
        ml, ng = max_len.value, n_grid.value
        return dict(n_steps=nst, status=status, rep_error=err, stats=stats, max_len=ml,
                    col_sum=col_sum[:ml], col_sq=col_sq[:ml], total=total, grid=grid[:ng],
                    tc_sum=tcs[:ng], tc_sq=tcq[:ng])

    def fetch_stats(self):
        stats = BatchStats()
        check(library().ct_fetch_results(self.handle, None, None, None, None, None,
                                         ctypes.byref(stats)))
        return stats


class SeedWords:
    """A numpy SeedSequence expressed as the words the device mixes.

    seed: int / sequence of ints / SeedSequence.  child_per_rep=True means
    repetition r uses SeedSequence(entropy, spawn_key + (rep_offset + r,)),
    i.e. seed.spawn(R)[r] of a fresh SeedSequence (harness.py:135-136).
    """

    def __init__(self, seed, child_per_rep: bool, rep_offset: int = 0):
        if isinstance(seed, np.random.SeedSequence):
            ss = seed
        elif isinstance(seed, (np.random.Generator, np.random.BitGenerator)):
            raise TypeError("a Generator seed cannot be regenerated on the device")
        else:
            ss = np.random.SeedSequence(seed)
        if ss.n_children_spawned and child_per_rep:
            raise ValueError("per-repetition children assume a fresh SeedSequence")
        if ss.pool_size != 4:
            raise ValueError("only the default SeedSequence pool size (4) is supported")
        self.entropy = _uint32_words(ss.entropy)
        self.prefix = _uint32_words(tuple(ss.spawn_key))
        self.child_per_rep = bool(child_per_rep)
        self.rep_offset = int(rep_offset)

    def spec(self) -> SeedSpec:
        s = SeedSpec()
        s.entropy = self.entropy.ctypes.data_as(_P(ctypes.c_uint32))
        s.n_entropy = self.entropy.size
        s.spawn_prefix = self.prefix.ctypes.data_as(_P(ctypes.c_uint32))
        s.n_prefix = self.prefix.size
        s.child_per_rep = int(self.child_per_rep)
        s.rep_offset = self.rep_offset
        return s


def _int_words(v: int):
    if v < 0:
        raise ValueError("seed entropy must be non-negative")
    if v == 0:
        return [0]
    out = []
    while v > 0:
        out.append(v & 0xFFFFFFFF)
        v >>= 32
    return out


def _uint32_words(x) -> np.ndarray:
    """numpy's _coerce_to_uint32_array for the int / sequence / array cases."""
    if x is None:
        raise ValueError("SeedSequence entropy is None")
    if isinstance(x, np.ndarray):
        if x.dtype == np.uint32:
            return np.ascontiguousarray(x)
        return np.concatenate([np.asarray(_int_words(int(v)), dtype=np.uint32) for v in x.ravel()]
                              ) if x.size else np.zeros(0, dtype=np.uint32)
    if isinstance(x, (int, np.integer)):
        return np.asarray(_int_words(int(x)), dtype=np.uint32)
    words = []
    for v in x:
        words.extend(_uint32_words(v).tolist())
    return np.asarray(words, dtype=np.uint32)


_ctx_lock = threading.Lock()
_contexts = {}


def context(device: int = 0, slot: int = 0) -> Context:
    """Process-wide context for one device; distinct slots are independent
    contexts on the same GPU (own buffers, own stream)."""
    with _ctx_lock:
        ctx = _contexts.get((device, slot))
        if ctx is None:
            ctx = Context(device)
            _contexts[(device, slot)] = ctx
        return ctx
