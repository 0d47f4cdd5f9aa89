"""Live measurement path: the five tunable benchmark kernels of the paper
(Table 2), compiled per configuration with NVRTC for the
B200, timed with CUDA events and profiled with the CUPTI range profiler.

This is the in-process B200 runner behind the reference's measurement plug
point (the ``MeasurementSource`` duck type, search.py:188-217; its
out-of-process form is the line protocol of search.py:220-275):

    src = CudaMeasurementSource(benchmark("transpose"))
    trace = run_profile_search(src, models, i=40)        # live Alg. 1
    ds = sweep(src)                                       # exhaustive B200 dataset

* ``src.space`` is the same configuration set as the synthetic stand-in of the
  same name (``spaces.space_of``), so models, datasets and traces line up.
* ``measure(idx, profiled=False)`` compiles the variant on first use (cached),
  times it (median of ``reps`` launches, L2 flushed between them) and returns
  ``Measurement(runtime_us)``; ``profiled=True`` also collects the paper's
  counter set (Table 1; ``counters.VOLTA_METRICS``, 24 metrics, 5 replay passes
  on GB100) and canonicalises it (``counters.canonicalize``,
  counters.py:161-180) as the reference's runner protocol does
  (search.py:262).
* Benchmark inputs are deterministic functions of ``seed``; outputs can be
  fetched for checking against the numpy oracles (tests only).
"""

import ctypes
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import counters as cc
from . import spaces
from .counters import ArchProfile
from .errors import CounterTuneError
from .search import Measurement
from .space import Dataset
from .tuner import CompileError, Launch, LaunchError, Tuner

_KDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "kernels")

# Table-1 metric names in catalog order (the counters the profiled step reports)
TABLE1_ABBRS: Sequence[str] = tuple(a for a in cc.ABBREVIATIONS if a in cc.VOLTA_METRICS)
TABLE1_METRICS: Sequence[str] = tuple(cc.VOLTA_METRICS[a][0] for a in TABLE1_ABBRS)

# The largest single-replay-pass subset of Table 1 on GB100 (SURVEY F13 group
# 1, 13 metrics): DRAM / L2 sectors, global load requests, executed and
# issued instructions, the four utilisations, warp / predication efficiency.
GROUP1_ABBRS: Sequence[str] = ("DRAM_RT", "DRAM_WT", "L2_RT", "L2_WT", "TEX_RWT", "INST_EXE",
                               "INST_ISSUE_U", "DRAM_U", "L2_U", "TEX_U", "SM_E", "WARP_E",
                               "WARP_NP_E")
GROUP1_METRICS: Sequence[str] = tuple(cc.VOLTA_METRICS[a][0] for a in GROUP1_ABBRS)

_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_f32 = ctypes.c_float


def clamp_counter(abbr: str, value: float) -> float:
    """A canonical reading inside the catalog's value range (the reference's
    dataset format rejects anything else, space.py:286-350): CUPTI's
    pct_of_peak ratios can read a few percent above 100 (e.g. SM_E 101.03
    on a kernel shorter than the sampling window), counts are >= 0."""
    from .formats import VALUE_RANGES
    lo, hi = VALUE_RANGES.get(abbr, (0.0, None))
    v = max(lo, value)
    return min(hi, v) if hi is not None else v


def b200_arch(sm_count: int = spaces.B200_SMS) -> ArchProfile:
    """ArchProfile of the device: Volta+ counter dialect, 128 FP32 cores/SM
    (the b_paral saturation rule of bottlenecks.py:172-173 counts cores)."""
    return ArchProfile(name="b200", generation=cc.VOLTA_PLUS, cores=int(sm_count) * 128)


class Benchmark:
    """One tunable kernel: its space, NVRTC source, inputs and launch geometry."""

    name = ""
    kernel = ""
    bound = ""        # roofline the kernel is judged against
    unit = ""

    def __init__(self, seed: int = 0):
        self.seed = seed
        with open(os.path.join(_KDIR, self.kernel + ".cu")) as f:
            self.source = f.read()
        self._space = None

    @property
    def space(self):
        if self._space is None:
            self._space = spaces.space_of(self.name)
        return self._space

    def values(self, config_index: int) -> Dict[str, int]:
        row = self.space.assignments[config_index]
        return {p.name: int(v) for p, v in zip(self.space.parameters, row)}

    def options(self, values: Dict[str, int]) -> List[str]:
        return [f"-D{k}={v}" for k, v in values.items()] + self.extra_options()

    def extra_options(self) -> List[str]:
        return []

    def valid(self, values: Dict[str, int]) -> bool:
        """Whether the configuration can run on this input (a configuration
        that does not tile the input is not part of the input's space)."""
        return True

    def restrict_space(self) -> None:
        """Keep only the configurations valid for this input, in the space's
        order (the KTT/CLTune constraint pass on the input sizes)."""
        keep = [i for i in range(len(self.space)) if self.valid(self.values(i))]
        if len(keep) < len(self.space):
            self._space = spaces.TuningSpace.from_assignments(
                self.space.parameters, self.space.assignments[keep])

    # per subclass -----------------------------------------------------------
    def host_inputs(self) -> Dict[str, np.ndarray]:
        raise NotImplementedError

    def setup(self, tuner: Tuner) -> Dict[str, int]:
        """Device buffers (inputs uploaded, outputs allocated)."""
        raise NotImplementedError

    def launch(self, values: Dict[str, int], bufs: Dict[str, int]) -> Launch:
        raise NotImplementedError

    def output(self, tuner: Tuner, bufs: Dict[str, int]) -> np.ndarray:
        raise NotImplementedError

    def work(self) -> float:
        """Algorithmic bytes (HBM-bound) or flops / interactions per launch."""
        raise NotImplementedError


class TransposeBenchmark(Benchmark):
    name, kernel, bound, unit = "transpose", "transpose", "hbm", "bytes"

    def __init__(self, width: int = 8192, height: int = 8192, seed: int = 0):
        super().__init__(seed)
        if width % 128 or height % 64:
            raise ValueError("transpose sizes must be multiples of 128 (width) and 64 (height)")
        self.width, self.height = width, height

    def host_inputs(self):
        rng = np.random.default_rng(self.seed)
        return {"in": rng.standard_normal((self.height, self.width), dtype=np.float32)}

    def setup(self, tuner):
        x = self.host_inputs()["in"]
        return {"in": tuner.upload(x), "out": tuner.alloc(x.nbytes)}

    def launch(self, v, bufs):
        tile, work_x = v["TILE"], v["WORK_X"]
        return Launch((self.width // (tile * work_x), self.height // tile),
                      (tile // v["VEC"], v["BLOCK_Y"]),
                      [_u64(bufs["in"]), _u64(bufs["out"]), _i32(self.width), _i32(self.height)])

    def output(self, tuner, bufs):
        return tuner.d2h(bufs["out"], np.empty((self.width, self.height), np.float32))

    def work(self):
        return 2.0 * 4.0 * self.width * self.height


class CoulombBenchmark(Benchmark):
    name, kernel, bound, unit = "coulomb", "coulomb", "mufu", "interactions"

    def __init__(self, grid: int = 256, atoms: int = 256, spacing: float = 0.5, seed: int = 0):
        super().__init__(seed)
        if grid % 32 or atoms % 256:
            raise ValueError("coulomb needs grid % 32 == 0 and atoms % 256 == 0")
        self.grid, self.atoms, self.spacing = grid, atoms, float(np.float32(spacing))

    def host_inputs(self):
        rng = np.random.default_rng(self.seed)
        extent = self.grid * self.spacing
        a = np.empty((self.atoms, 4), np.float32)
        # atoms between grid planes (never on a grid point)
        a[:, :3] = (rng.integers(0, self.grid, (self.atoms, 3)) + rng.uniform(0.2, 0.8, (self.atoms, 3))
                    ) * self.spacing
        a[:, :3] = np.minimum(a[:, :3], extent)
        a[:, 3] = rng.uniform(-1.0, 1.0, self.atoms)
        return {"atoms": a}

    def setup(self, tuner):
        a = self.host_inputs()["atoms"]
        soa = np.ascontiguousarray(a.T)
        out = {"atoms": tuner.upload(a)}
        for k, name in enumerate("xyzw"):
            out[name] = tuner.upload(soa[k])
        out["energy"] = tuner.alloc(4 * self.grid ** 3)
        return out

    def launch(self, v, bufs):
        by = v["BLOCK"] // 32
        z = v["Z_ITERATIONS"]
        return Launch((self.grid // 32, self.grid // by, -(-self.grid // z)), (32, by),
                      [_u64(bufs["atoms"]), _u64(bufs["x"]), _u64(bufs["y"]), _u64(bufs["z"]),
                       _u64(bufs["w"]), _i32(self.atoms), _f32(self.spacing), _i32(self.grid),
                       _u64(bufs["energy"])])

    def output(self, tuner, bufs):
        g = self.grid
        return tuner.d2h(bufs["energy"], np.empty((g, g, g), np.float32))

    def work(self):
        return float(self.grid) ** 3 * self.atoms


class NBodyBenchmark(Benchmark):
    name, kernel, bound, unit = "nbody", "nbody", "fp32", "interactions"

    def __init__(self, bodies: int = 16384, eps2: float = 0.01, seed: int = 0):
        super().__init__(seed)
        if bodies % 1024:
            raise ValueError("nbody needs bodies % 1024 == 0")
        self.bodies, self.eps2 = bodies, float(np.float32(eps2))

    def host_inputs(self):
        rng = np.random.default_rng(self.seed)
        pm = np.empty((self.bodies, 4), np.float32)
        pm[:, :3] = rng.standard_normal((self.bodies, 3))
        pm[:, 3] = rng.uniform(0.5, 1.5, self.bodies)
        return {"pm": pm}

    def setup(self, tuner):
        self.SMS = tuner.sm_count          # the device's SMs (148 on B200) for split()
        pm = self.host_inputs()["pm"]
        soa = np.ascontiguousarray(pm.T)
        out = {"pm": tuner.upload(pm)}
        for k, name in enumerate(("x", "y", "z", "m")):
            out[name] = tuner.upload(soa[k])
        out["acc"] = tuner.alloc(16 * self.bodies)
        out["partial"] = tuner.alloc(16 * self.bodies * self.MAX_JB)
        groups = -(-self.bodies // 32)
        out["arrivals"] = tuner.alloc(4 * groups)
        tuner.memset(out["arrivals"], 0, 4 * groups)
        return out

    # the kernel's launch bounds cap it at 64 registers for 1024 resident
    # threads per SM (32 warps: 8 per scheduler for the MUFU/FMA latencies)
    SM_THREADS = 1024
    SMS = 148                         # replaced by the device's count in setup()
    MAX_JB = 16

    def split(self, v):
        """(JS, JB): thread rows per block and blocks the j range is split
        over, minimising waves of resident blocks x j tiles per thread row
        (a partial extra wave costs a whole one); ties go to fewer splits
        (less reduction), then to more thread rows (reduced in shared memory,
        not through global partials)."""
        B = v["BLOCK"]
        gx = -(-self.bodies // (B * v["OUTER"]))
        tiles = -(-self.bodies // B)
        best = None
        js = 1
        while B * js <= 1024:
            slots = self.SMS * max(1, self.SM_THREADS // (B * js))
            for jb in range(1, self.MAX_JB + 1):
                waves = -(-(gx * jb) // slots)
                key = (waves * -(-tiles // (js * jb)), js * jb, -js)
                if best is None or key < best[0]:
                    best = (key, js, jb)
            js *= 2
        return best[1], best[2]

    def jb(self, v) -> int:
        return self.split(v)[1]

    def js(self, v) -> int:
        return self.split(v)[0]

    def options(self, values):
        return super().options(values) + [f"-DJS={self.js(values)}"]

    def launch(self, v, bufs):
        per_block = v["BLOCK"] * v["OUTER"]
        return Launch((-(-self.bodies // per_block), self.jb(v)), (v["BLOCK"], self.js(v)),
                      [_u64(bufs["pm"]), _u64(bufs["x"]), _u64(bufs["y"]), _u64(bufs["z"]),
                       _u64(bufs["m"]), _i32(self.bodies), _f32(self.eps2), _u64(bufs["acc"]),
                       _u64(bufs["partial"]), _u64(bufs["arrivals"])])

    def output(self, tuner, bufs):
        return tuner.d2h(bufs["acc"], np.empty((self.bodies, 4), np.float32))[:, :3]

    def work(self):
        return float(self.bodies) ** 2


def _conv_filter_arg(filt: np.ndarray):
    """conv.cu's by-value Filter: the taps, then every tap as a packed pair
    (f, f) for the FFMA2 path's broadcast operand."""
    n = filt.size

    class Filter(ctypes.Structure):
        _fields_ = [("f", ctypes.c_float * n), ("f2", ctypes.c_uint64 * n)]

    taps = np.ascontiguousarray(filt.ravel(), dtype=np.float32)
    bits = taps.view(np.uint32).astype(np.uint64)
    return Filter((ctypes.c_float * n)(*taps.tolist()),
                  (ctypes.c_uint64 * n)(*((bits << np.uint64(32)) | bits).tolist()))


class ConvBenchmark(Benchmark):
    name, kernel, bound, unit = "conv", "conv", "fp32", "flops"

    def __init__(self, width: int = 4096, height: int = 4096, filt: int = 7, seed: int = 0):
        super().__init__(seed)
        if width % 512 or height % 128:
            raise ValueError("conv sizes must be multiples of 512 (width) and 128 (height)")
        self.width, self.height, self.filt = width, height, filt

    def extra_options(self):
        return [f"-DFILTER={self.filt}"]

    def host_inputs(self):
        rng = np.random.default_rng(self.seed)
        return {"in": rng.standard_normal((self.height, self.width), dtype=np.float32),
                "filt": rng.uniform(-1, 1, (self.filt, self.filt)).astype(np.float32)}

    def setup(self, tuner):
        h = self.host_inputs()
        self._filt_host = h["filt"]
        return {"in": tuner.upload(h["in"]), "filt": tuner.upload(h["filt"]),
                "out": tuner.alloc(h["in"].nbytes)}

    def smem_bytes(self, v) -> int:
        f = self.filt
        tw, th = v["TBX"] * v["WPTX"], v["TBY"] * v["WPTY"]
        # conv.cu PAIRED: two tile copies and (CACHE_F) the taps duplicated
        # as packed pairs, where that still fits 227 KB
        filt2 = ((f * f + 1) // 2 * 2 + 2 * f * f) if v["CACHE_F"] else 0
        paired = (v["LOCAL"] == 2 and v["WPTX"] % 2 == 0
                  and 4 * (2 * (th + f - 1) * (tw + 8 + 2 * v["PAD"]) + filt2) <= 227 * 1024)
        filt = (filt2 if paired else f * f) if v["CACHE_F"] else 0
        tile = ((th + f - 1) * (tw + 8 + v["PAD"] * (2 if paired else 1)) * (2 if paired else 1)
                if v["LOCAL"] else 0)
        return 4 * (tile + filt)

    def launch(self, v, bufs):
        tw, th = v["TBX"] * v["WPTX"], v["TBY"] * v["WPTY"]
        # the filter also travels by value (kernel parameter bank, CACHE_F = 0)
        if getattr(self, "_filt_host", None) is None:
            self._filt_host = self.host_inputs()["filt"]
        kf = _conv_filter_arg(self._filt_host)
        return Launch((self.width // tw, self.height // th), (v["TBX"], v["TBY"]),
                      [_u64(bufs["in"]), _u64(bufs["filt"]), kf, _u64(bufs["out"]),
                       _i32(self.width), _i32(self.height)], dynamic_smem=self.smem_bytes(v))

    def output(self, tuner, bufs):
        return tuner.d2h(bufs["out"], np.empty((self.height, self.width), np.float32))

    def work(self):
        return 2.0 * self.filt ** 2 * self.width * self.height


class GemmBenchmark(Benchmark):
    name, kernel, bound, unit = "gemm", "gemm", "fp32", "flops"

    def __init__(self, m: int = 2048, n: int = 2048, k: int = 2048, seed: int = 0):
        super().__init__(seed)
        if m % 16 or n % 16 or k % 16 or min(m, n, k) < 16:
            raise ValueError("gemm sizes must be positive multiples of 16")
        self.m, self.n, self.k = m, n, k

    def valid(self, v) -> bool:
        # the kernel has no edge tiles (CLBlast's xgemm pads instead): the
        # block tile must divide C and the k-slice must divide K
        return self.m % v["MWG"] == 0 and self.n % v["NWG"] == 0 and self.k % v["KWG"] == 0

    def host_inputs(self):
        rng = np.random.default_rng(self.seed)
        return {"at": rng.uniform(-1, 1, (self.k, self.m)).astype(np.float32),
                "b": rng.uniform(-1, 1, (self.k, self.n)).astype(np.float32)}

    def setup(self, tuner):
        h = self.host_inputs()
        self._tuner = tuner
        self._maps = {}
        return {"at": tuner.upload(h["at"]), "b": tuner.upload(h["b"]),
                "c": tuner.alloc(4 * self.m * self.n)}

    @staticmethod
    def tc5(v) -> bool:
        """TC=1 variants that run on the 5th-generation tensor cores
        (tcgen05.mma, M = 128, >= 4 warps); other TC=1 variants use mma.sync."""
        return v["TC"] == 1 and v["MWG"] == 128 and v["MDIMC"] * v["NDIMC"] >= 128

    def smem_bytes(self, v) -> int:
        # tcgen05 pipeline (gemm.cu): two raw fp32 stages of A^T (KWG x 128)
        # and B (KWG x NWG) for the TMA, two stages of tf32 big/small operand
        # tiles, after 1 KB of alignment for the static barriers
        if not self.tc5(v):
            return 0
        return 1024 + 8 * v["KWG"] * (384 + 3 * v["NWG"])

    def tensor_maps(self, v, bufs):
        """TMA descriptors of A^T (box 128 x KWG) and B (box NWG x KWG)."""
        key = (v["KWG"], v["NWG"])
        if key not in self._maps:
            t = self._tuner
            self._maps[key] = (
                t.tensor_map_2d(bufs["at"], self.m, self.k, 4 * self.m, 128, v["KWG"]),
                t.tensor_map_2d(bufs["b"], self.n, self.k, 4 * self.n, v["NWG"], v["KWG"]))
        return self._maps[key]

    def launch(self, v, bufs):
        args = [_u64(bufs["at"]), _u64(bufs["b"]), _u64(bufs["c"]), _i32(self.m), _i32(self.n),
                _i32(self.k)]
        if self.tc5(v):
            args += list(self.tensor_maps(v, bufs))
        return Launch((self.m // v["MWG"], self.n // v["NWG"]), (v["MDIMC"] * v["NDIMC"],),
                      args, dynamic_smem=self.smem_bytes(v))

    def output(self, tuner, bufs):
        return tuner.d2h(bufs["c"], np.empty((self.m, self.n), np.float32))

    def work(self):
        return 2.0 * self.m * self.n * self.k


BENCHMARKS = {
    "transpose": TransposeBenchmark,
    "coulomb": CoulombBenchmark,
    "nbody": NBodyBenchmark,
    "conv": ConvBenchmark,
    "gemm": GemmBenchmark,
}


def benchmark(name: str, **sizes) -> Benchmark:
    try:
        return BENCHMARKS[name](**sizes)
    except KeyError:
        raise ValueError(f"unknown benchmark {name!r}; known: {sorted(BENCHMARKS)}")


class CudaMeasurementSource:
    """MeasurementSource over one GPU (search.py:188-217 duck type)."""

    def __init__(self, bench: Benchmark, device: int = 0, tuner: Optional[Tuner] = None,
                 warmup: int = 1, reps: int = 3, flush_l2: bool = True,
                 metrics: Sequence[str] = TABLE1_METRICS, slow_us: float = 5000.0,
                 fill_from=None):
        """metrics: the CUPTI metric set of a profiled step (Table 1, 24
        metrics, 5 replay passes on B200).  With a reduced set --
        GROUP1_METRICS, the largest single-pass subset -- the
        Table-1 counters not collected are taken from fill_from for the
        profiled configuration (mode "group1+model"), a labelled
        approximation of the reference's full profile: a PredictionTable
        (its model's prediction; the exact/tree models do not predict the
        utilisations, so SHR_U -- outside group 1, a second pass on B200 --
        needs the next source) or a Dataset (a recorded sweep of the space,
        which is what the exact model replays)."""
        self.bench = bench
        self.tuner = tuner if tuner is not None else Tuner(device)
        self._own_tuner = tuner is None
        self.space = bench.space
        self.arch = b200_arch(self.tuner.sm_count)
        self.warmup, self.reps, self.flush_l2 = warmup, reps, flush_l2
        self.slow_us = slow_us
        self.metrics = tuple(metrics)
        self.fill_from = fill_from
        collected = {cc.canonicalize(m, 1.0, self.arch)[0] for m in self.metrics}
        self.filled = tuple(a for a in TABLE1_ABBRS if a not in collected)
        if self.filled:
            if fill_from is None:
                raise ValueError("a reduced metric set needs fill_from (the model that predicts "
                                 f"{', '.join(self.filled)})")
            names = (fill_from.column if hasattr(fill_from, "column")
                     else {a: j for j, a in enumerate(fill_from.counter_names)})
            missing = [a for a in self.filled if a not in names]
            if missing:
                raise ValueError(f"fill_from does not provide {', '.join(missing)}")
            self._fill_col = {a: names[a] for a in self.filled}
            self._fill_rows = (fill_from.matrix if hasattr(fill_from, "column")
                               else fill_from.counter_matrix)
        self.mode = "full" if not self.filled else "group1+model"
        self._bufs = bench.setup(self.tuner)
        self._variants: Dict[int, int] = {}
        self.profile_passes = 0
        self.compile_failures: Dict[int, str] = {}

    # -- variants ---------------------------------------------------------
    def compile_all(self, indices: Optional[Sequence[int]] = None, threads: int = 0) -> int:
        """Compile the variants of `indices` (default: the whole space)
        concurrently on host threads; returns how many failed."""
        idx = [i for i in (range(len(self.space)) if indices is None else indices)
               if i not in self._variants]
        if not idx:
            return 0
        opts = [self.bench.options(self.bench.values(i)) for i in idx]
        handles, status = self.tuner.compile_batch(self.bench.source, self.bench.kernel, opts,
                                                   threads)
        bad = 0
        for i, h, st in zip(idx, handles, status):
            if st == 0:
                self._variants[i] = int(h)
            else:
                self.compile_failures[i] = f"status {int(st)}"
                bad += 1
        return bad

    def reset_variants(self) -> None:
        """Unload the compiled variants (the next measure() compiles again,
        as a fresh tuning session would).  The modules are unloaded, not just
        forgotten: every module left loaded in the context would stay there
        for the rest of the process."""
        for v in self._variants.values():
            self.tuner.unload(v)
        self._variants.clear()

    def variant(self, config_index: int) -> int:
        v = self._variants.get(config_index)
        if v is None:
            try:
                v = self.tuner.compile(self.bench.source, self.bench.kernel,
                                       self.bench.options(self.bench.values(config_index)))
            except CompileError as e:
                raise CounterTuneError(f"configuration {config_index} does not compile: {e}")
            self._variants[config_index] = v
        return v

    def launch_of(self, config_index: int) -> Launch:
        return self.bench.launch(self.bench.values(config_index), self._bufs)

    # -- MeasurementSource ------------------------------------------------
    def measure(self, config_index: int, profiled: bool) -> Measurement:
        v = self.variant(config_index)
        launch = self.launch_of(config_index)
        try:
            times = self.tuner.time(v, launch, warmup=self.warmup, reps=1, flush_l2=self.flush_l2)
            # a slow variant (>= slow_us) is timed once: its run-to-run spread
            # is far below the gaps the search distinguishes, and a sweep of a
            # space full of pathological variants stays affordable
            if self.reps > 1 and times[0] < self.slow_us:
                more = self.tuner.time(v, launch, warmup=0, reps=self.reps - 1,
                                       flush_l2=self.flush_l2)
                times = np.concatenate([times, more])
        except LaunchError as e:
            raise CounterTuneError(f"configuration {config_index} failed to launch: {e}")
        runtime = float(np.median(times))
        if not profiled:
            return Measurement(runtime_us=runtime)
        vals, passes = self.tuner.profile(v, launch, self.metrics)
        self.profile_passes = passes
        counter_map: Dict[str, float] = {}
        for name, value in zip(self.metrics, vals):
            abbr, canonical = cc.canonicalize(name, float(value), self.arch)
            counter_map[abbr] = clamp_counter(abbr, canonical)
        if self.filled:
            row = self._fill_rows[config_index]
            for abbr in self.filled:
                counter_map[abbr] = clamp_counter(abbr, float(row[self._fill_col[abbr]]))
        return Measurement(runtime_us=runtime, global_threads=launch.threads,
                           counters=counter_map)

    def profile_many(self, indices: Sequence[int]):
        """The profiled half of measure() for several configurations in ONE
        CUPTI collection (ct_tuner_profile_batch: one range per launch, the
        per-collection cost paid once) -> [(global_threads, counters)]."""
        vs = [self.variant(i) for i in indices]
        launches = [self.launch_of(i) for i in indices]
        vals, passes = self.tuner.profile_batch(vs, launches, self.metrics)
        self.profile_passes = passes
        out = []
        for i, launch, row in zip(indices, launches, vals):
            counter_map: Dict[str, float] = {}
            for name, value in zip(self.metrics, row):
                abbr, canonical = cc.canonicalize(name, float(value), self.arch)
                counter_map[abbr] = clamp_counter(abbr, canonical)
            if self.filled:
                frow = self._fill_rows[i]
                for abbr in self.filled:
                    counter_map[abbr] = clamp_counter(abbr, float(frow[self._fill_col[abbr]]))
            out.append((launch.threads, counter_map))
        return out

    def output(self, config_index: int) -> np.ndarray:
        """Run the variant once and fetch its output (for oracle checks)."""
        v = self.variant(config_index)
        self.tuner.time(v, self.launch_of(config_index), warmup=1, reps=0, flush_l2=False)
        return self.bench.output(self.tuner, self._bufs)

    def close(self) -> None:
        if self._own_tuner and self.tuner is not None:
            self.tuner.close()
        self.tuner = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


@dataclass
class SweepResult:
    dataset: Dataset
    failures: Dict[int, str]
    seconds_compile: float
    seconds_measure: float


def sweep(source: CudaMeasurementSource, profiled: bool = True, checkpoint: Optional[str] = None,
          compile_threads: int = 0, progress=None,
          budget_s: Optional[float] = None, batch: int = 32) -> SweepResult:
    """Exhaustive sweep of the source's space -> a replay Dataset in the
    reference's layout (runtime, threads, the Table-1 counters canonicalised).

    With ``checkpoint`` the partial results are kept in an .npz every 64
    configurations and a rerun resumes from it (config_index order).  With
    ``budget_s`` measuring stops after that many seconds; configurations not
    reached carry no record (a later run with the same checkpoint resumes)."""
    import time
    n = len(source.space)
    names = TABLE1_ABBRS
    runtime = np.full(n, np.nan)
    threads = np.zeros(n, dtype=np.int64)
    cm = np.full((n, len(names)), np.nan)
    done = np.zeros(n, dtype=bool)
    if checkpoint and os.path.exists(checkpoint):
        z = np.load(checkpoint)
        runtime, threads, cm, done = z["runtime"], z["threads"], z["counters"], z["done"]
    t0 = time.perf_counter()
    source.compile_all([i for i in range(n) if not done[i]], threads=compile_threads)
    t1 = time.perf_counter()
    failures = dict(source.compile_failures)
    todo = [i for i in range(n) if not done[i] and i not in failures]
    # chunks of `batch` configurations: each timed on its own (median of the
    # source's reps, L2 flushed), then profiled together in one CUPTI
    # collection (profile_many); a chunk whose collection fails is profiled
    # one configuration at a time
    for c0 in range(0, len(todo), batch):
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
        timed = []
        for i in todo[c0:c0 + batch]:
            try:
                runtime[i] = source.measure(i, profiled=False).runtime_us
                timed.append(i)
            except CounterTuneError as e:
                failures[i] = str(e)
        if profiled and timed:
            try:
                got = source.profile_many(timed)
            except CounterTuneError:
                got = []
                for i in list(timed):
                    try:
                        got.append(source.profile_many([i])[0])
                    except CounterTuneError as e:
                        failures[i] = str(e)
                        timed.remove(i)
            for i, (th, counters) in zip(timed, got):
                threads[i] = th
                cm[i] = [counters[a] for a in names]
        for i in timed:
            done[i] = True
        if checkpoint:
            np.savez(checkpoint, runtime=runtime, threads=threads, counters=cm, done=done)
        if progress and timed:
            progress(timed[-1], n)
    if checkpoint:
        np.savez(checkpoint, runtime=runtime, threads=threads, counters=cm, done=done)
    t2 = time.perf_counter()
    # configurations that failed to build or launch carry no record: replaying
    # them raises, as the reference's replay source does (search.py:205-214)
    ds = Dataset(source.space, source.arch, f"{source.bench.name}-b200",
                 runtime_us=np.where(done, runtime, 1.0), global_threads=np.maximum(1, threads),
                 counter_names=names if profiled else (),
                 counter_matrix=np.where(done[:, None], cm, 0.0) if profiled
                 else np.zeros((n, 0)), has_record=done)
    return SweepResult(ds, failures, t1 - t0, t2 - t1)
