"""Benchmark of the searcher hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (configs[1] of BASELINE.json): the matrix-transpose tuning space
(1,784 configurations, 8 parameters) replayed from its exhaustive B200 sweep
(datasets/transpose-b200: every configuration of the NVRTC transpose kernel
timed and profiled on a B200 by scripts/live_sweep.py, 24 CUPTI counters,
reference on-disk format), profile-guided searcher with the exact model, R = 1000 repetitions per GPU (SeedSequence(42) children), n = 5,
i = 40 outer iterations, throughput mode (stop_indices = {}).  One step = one
batched device search over all R repetitions.  value = configurations scored
per second over the whole job (sum over ranks / max rank time).

Also reported: the steps metric (mean empirical steps to a configuration
within 1.1x of the best, profile vs random search, simulated wall-s) for the
same space, e2e through the public API (harness.simulate with host buffers),
the roofline of the search kernel and the CPU oracle baseline.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "configs scored/s (profile searcher hot path); steps & wall-s to <=1.1x best"
UNIT = "configs/s"
REPS = 1000
OUTER = 40
INNER = 5
SEED = 42


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    in-process every 2 ms (nvidia-smi as a fallback, ~10 Hz)."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.samples = []          # (sm_mhz, max_mhz, reason names)
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            try:
                uuid = str(torch.cuda.get_device_properties(device).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self._nvml = (pynvml, h, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _run_nvml(self):
        nv, h, mx = self._nvml
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), [n for n, b in self.REASONS if r & b]))
            except Exception:
                return
            self._stop.wait(0.002)

    def _run_smi(self):
        self.source = "nvidia-smi"
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                c = [x.strip() for x in out.split(",")]
                if len(c) >= 2 and c[0].replace(".", "").isdigit():
                    self.samples.append((float(c[0]), float(c[1]),
                                         [names[k] for k in range(4)
                                          if len(c) > 2 + k and c[2 + k].lower() == "active"]))
            except Exception:
                return
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run_nvml if self._nvml else self._run_smi, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted({n for s in self.samples for n in s[2]}),
                "samples": len(self.samples), "source": self.source}


def _traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)["k_profile_search"]
        return int(t["dram_bytes_per_launch"]), t["source"], t
    except Exception:
        return None, None, {}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


DATASET = os.path.join(ROOT, "datasets", "transpose-b200")
DATA = "B200-measured replay dataset (datasets/transpose-b200)"
# the workload, identical in both arms' lines
CONFIG = {"workload": "transpose tuning space (1,784 configs, 8 params) replay of its "
                      "exhaustive B200 sweep; profile searcher, exact model, throughput mode "
                      "(stop_indices = {})",
          "dataset": "datasets/transpose-b200", "repetitions_per_gpu": REPS,
          "outer_iterations": OUTER, "inner_steps": INNER, "seed": SEED,
          "l2": "GPU arm: 256 MiB buffer written between timed steps (table 271 KB)"}


def load_dataset():
    from paper_2102_05297_b200 import formats
    return formats.load_dataset_dir(DATASET)


def workload(reps=REPS, stop=False):
    from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec
    ds = load_dataset()
    spec = ExperimentSpec(dataset=ds, searcher="profile", model=ExactModelSet(ds),
                          name="profile-search", repetitions=reps, inner_steps=INNER,
                          outer_iterations=OUTER, seed=SEED, stop_at_well_performing=stop)
    return ds, spec


# ------------------------------------------------------------- CPU baseline
def _oracle_chunk(args):
    rep_lo, rep_hi, reps_total = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import countertune_oracle as oracle
    from paper_2102_05297_b200 import ExactModelSet
    from paper_2102_05297_b200.space import replay_arrays
    ds = load_dataset()
    ms = ExactModelSet(ds)
    matrix = ms.prediction_matrix(ds.space)
    column = {n: j for j, n in enumerate(ms.counters)}
    rt, th, req, hr = replay_arrays(ds)
    seeds = np.random.SeedSequence(SEED).spawn(reps_total)
    scored = 0
    t0 = time.perf_counter()
    for r in range(rep_lo, rep_hi):
        _, _, s = oracle.profile_search(matrix, column, rt, th, req, hr, pre_volta=False,
                                        cores=ds.arch.cores, i=OUTER, n=INNER, seed=seeds[r],
                                        stop=None)
        scored += s
    return scored, time.perf_counter() - t0


def cpu_baseline(reps: int, cores: int):
    """The oracle (numpy restatement of the reference) over `reps` repetitions
    of the same workload, fanned out over `cores` processes as the reference's
    harness does (COUNTERTUNE_WORKERS)."""
    from concurrent.futures import ProcessPoolExecutor
    chunks = [(k * reps // cores, (k + 1) * reps // cores, max(REPS, reps)) for k in range(cores)]
    t0 = time.perf_counter()
    if cores == 1:
        out = [_oracle_chunk(chunks[0])]
    else:
        with ProcessPoolExecutor(max_workers=cores) as pool:
            out = list(pool.map(_oracle_chunk, chunks))
    wall = time.perf_counter() - t0
    scored = sum(o[0] for o in out)
    return scored / wall, scored, wall


# ------------------------------------------------------- reference arm
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_REF = {}


def _ref_init():
    """Worker: the unmodified reference package (baseline/_ref, installed from
    /root/reference/pkg) loads the dataset with its own loader and builds its
    own PredictionTable, as harness._run_repetitions does per worker."""
    sys.path.insert(0, REF_DIR)
    from countertune import models, search, space
    ds = space.load_dataset_dir(DATASET)
    _REF["src"] = search.DatasetReplaySource(ds)
    _REF["table"] = search.PredictionTable.from_model_set(models.ExactModelSet(ds), ds.space)
    _REF["n"] = len(ds.space)


def _ref_chunk(reps):
    """run_profile_search (the reference's public API, stock code path) over
    the given repetitions in throughput mode; configurations scored = the
    unexplored pool at each scoring call (search.py:380-385)."""
    from countertune import search
    seeds = np.random.SeedSequence(SEED).spawn(REPS)
    n = _REF["n"]
    scored = 0
    for r in reps:
        tr = search.run_profile_search(_REF["src"], _REF["table"], i=OUTER, n=INNER,
                                       seed=seeds[r], stop_indices=frozenset())
        idx = [s.config_index for s in tr.steps]
        for k in range(OUTER):
            first = k * (INNER + 1) + 1          # steps recorded when iteration k scores
            if first > len(idx):
                break
            scored += n - len(set(idx[:first]))
    return scored


def run_reference(args):
    """The reference's own CPU implementation of the path, on all host cores
    (worker processes with strided repetition chunks, as its harness fans
    out with COUNTERTUNE_WORKERS), same workload, metric and unit."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    if not os.path.isdir(os.path.join(REF_DIR, "countertune")):
        print(json.dumps({"impl": "reference", "unavailable":
                          "baseline/_ref holds no countertune install"}), flush=True)
        return
    from concurrent.futures import ProcessPoolExecutor
    cores = os.cpu_count() or 1
    sample = min(REPS, 32 * cores)               # repetitions per step (bounded CPU time)
    chunks = [list(range(k, sample, cores)) for k in range(cores)]
    vals = []
    with ProcessPoolExecutor(max_workers=cores, initializer=_ref_init) as pool:
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            scored = sum(pool.map(_ref_chunk, chunks))
            wall = time.perf_counter() - t0
            if k >= args.warmup:
                vals.append((scored / wall, scored, wall))
    value = float(np.median([v for v, _, _ in vals]))
    ms = float(np.median([w for _, _, w in vals])) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": dict(CONFIG),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{sample} of the {REPS} repetitions per step "
                                   f"({vals[0][1]} configs scored), countertune.search."
                                   f"run_profile_search from baseline/_ref in {cores} worker "
                                   f"processes"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    # CT_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0 over gloo, to
    # exercise the multi-rank path on a one-GPU box; timings are meaningless
    shared = os.environ.get("CT_BENCH_SHARED_GPU") == "1"
    if world > 1:
        if shared:
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = 0 if (world == 1 or shared) else local
    torch.cuda.set_device(device)

    from paper_2102_05297_b200 import _native, harness
    from paper_2102_05297_b200.space import replay_arrays
    ds, spec = workload()
    ctx = _native.context(device)
    # a dedicated stream: the kernels, the L2 flush and the timing events
    # all live on it (torch's legacy default stream has handle 0, which the
    # C ABI reads as "the context's own stream")
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    params, _ = harness.prepare_device(ctx, spec)
    rep_offset = rank * REPS                  # weak scaling: R repetitions per GPU

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)

    def one_step():
        harness.launch(ctx, spec, params, rep_offset, REPS)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize(device)
    stats0 = ctx.fetch_stats()
    configs_per_step = stats0.configs_scored
    bytes_per_step = stats0.algorithmic_bytes

    times = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    with ClockSampler(device) as clocks:
        for _ in range(args.steps):
            flush.add_(1.0)                   # evict the table from L2 between steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            one_step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    stats = ctx.fetch_stats()
    assert stats.configs_scored == configs_per_step, "steps must be identical"
    t_total = float(sum(times))
    if world > 1:
        t = torch.tensor([t_total], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_total = float(t.item())
    value = world * configs_per_step * args.steps / t_total
    per_launch = t_total / args.steps
    hbm, peak_kind = _peaks()
    traffic, traffic_src, kprof = _traffic()
    achieved_gbs = bytes_per_step / per_launch / 1e9
    print(f"[bench] rank {rank}: {configs_per_step} configs/step, {per_launch * 1e3:.3f} ms/step, "
          f"{value:.4g} configs/s, {achieved_gbs:.1f} GB/s algorithmic, "
          f"uncertified {stats0.uncertified}", file=sys.stderr, flush=True)
    if args.kernel_only:
        if world > 1:
            dist.destroy_process_group()
        return

    # e2e through the public API with host buffers in and the report out:
    # harness.simulate (N=1) / dist.simulate_distributed (N>1, one experiment
    # of world*R repetitions sharded over the ranks).  Inside the timed
    # region every step: H2D of the prediction table (padded column-major),
    # the replay arrays and stop mask; the search; the on-device aggregation;
    # D2H of the per-repetition status/step counts/times and the report sums.
    import dataclasses
    from paper_2102_05297_b200.dist import simulate_distributed
    espec = dataclasses.replace(spec, repetitions=REPS * world)
    e2e_times = []
    rt, th, req, hr = replay_arrays(ds)
    n = len(ds.space)
    ld = (n + 2047) // 2048 * 2048
    h2d_rank = ld * 19 * 8 + rt.nbytes + th.nbytes + req.nbytes + hr.nbytes + (n + 31) // 32 * 4
    max_len = OUTER * (INNER + 1)
    d2h_rank = REPS * (4 + 4 + 4 + 8 + 8) + 2 * 8 * max_len + 2 * 8 * 100 + 40
    for k in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        if world > 1:
            rep = simulate_distributed(espec, device=device)
        else:
            rep = harness.simulate(espec, devices=[device])
        torch.cuda.synchronize(device)
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        if k >= args.warmup:
            e2e_times.append(dt)
    e2e_value = rep.configs_scored / float(np.median(e2e_times))
    h2d = h2d_rank * world
    d2h = d2h_rank * world

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # the BASELINE.md section 3 stress size where the table (152 MB) no
    # longer fits the L2: the same search at N = 2^20 on the default (tiled)
    # path, CUDA events on the context's stream, for the HBM-bound roofline
    large = None
    if not args.no_large_space:
        try:
            from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec, spaces
            lds = spaces.stress(1 << 20)
            lspec = ExperimentSpec(dataset=lds, searcher="profile", model=ExactModelSet(lds),
                                   repetitions=444, outer_iterations=10, seed=SEED,
                                   stop_at_well_performing=False)
            lparams, _ = harness.prepare_device(ctx, lspec)
            harness.launch(ctx, lspec, lparams, 0, 444)            # warm-up
            lt = []
            for _ in range(3):
                flush.add_(1.0)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                harness.launch(ctx, lspec, lparams, 0, 444)
                e1.record(stream)
                e1.synchronize()
                lt.append(e0.elapsed_time(e1) / 1e3)
            lst = ctx.fetch_stats()
            lsec = float(np.median(lt))
            lgbs = lst.algorithmic_bytes / lsec / 1e9
            large = {"workload": "stress space, 1,048,576 configurations x 19 counter columns "
                                 "(table 152 MB > L2), R = 444, i = 10, n = 5, default "
                                 "dispatch (tiled path)",
                     "ms_per_step": lsec * 1e3, "configs_per_s": lst.configs_scored / lsec,
                     "roofline": {"bound": "hbm", "achieved": lgbs, "peak": hbm, "unit": "GB/s",
                                  "frac": lgbs / hbm,
                                  "algorithmic_bytes_per_launch": int(lst.algorithmic_bytes),
                                  "traffic_source": "profiles/r02/r02s_tiled_score.md, "
                                                    "r02s_tiled_weights.md (ncu, per kernel)"},
                     "uncertified_draws": int(lst.uncertified)}
            params, _ = harness.prepare_device(ctx, spec)         # restore the bench space
        except Exception as exc:  # report, never hide
            large = {"error": repr(exc)}

    # steps metric on the same space: profile vs random, stop at <= 1.1x best
    steps_info = {}
    try:
        from paper_2102_05297_b200 import ExperimentSpec, pair_with_baseline
        _, sspec = workload(stop=True)
        sspec.outer_iterations = None
        # simulated wall-s with the MEASURED profiling overhead of this space
        # (not the reference's invented 3.0)
        with open(os.path.join(DATASET, "profiling_overhead.json")) as fh:
            ovh = json.load(fh)
        sspec.profiling_overhead = float(ovh["profiling_overhead"])
        prof = harness.simulate(sspec, devices=[device])
        rspec = ExperimentSpec(dataset=ds, searcher="random", name="random-search",
                               repetitions=REPS, seed=SEED,
                               profiling_overhead=sspec.profiling_overhead)
        rnd = harness.simulate(rspec, devices=[device])
        pair_with_baseline(prof, rnd)
        steps_info = {"profile_mean_steps": prof.mean_steps, "random_mean_steps": rnd.mean_steps,
                      "improvement": prof.improvement,
                      "profile_mean_sim_wall_s": prof.mean_time_seconds,
                      "random_mean_sim_wall_s": rnd.mean_time_seconds,
                      "profile_censored": prof.censored, "uncertified_draws": prof.uncertified_draws,
                      "profiling_overhead": sspec.profiling_overhead,
                      "profiling_overhead_source": ovh["source"]}
    except Exception as exc:  # report, never hide
        steps_info = {"error": repr(exc)}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        sample = 64 * cores
        v, scored, wall = cpu_baseline(sample, cores)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{sample} repetitions ({scored} configs scored) of the same workload, "
                         f"oracle/countertune_oracle.py in {cores} processes, {wall:.1f} s wall"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_launch * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": dict(CONFIG),
        "configs_scored_per_step_per_gpu": configs_per_step,
        "parallelism": f"reps sharded over {world} GPU(s)",
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "api": "harness.simulate" if world == 1 else "dist.simulate_distributed",
                "timing": "host wall clock around the API call, median of steps, max over ranks"},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": achieved_gbs / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": bytes_per_step,
                     "note": "8*C_used+16 B per scored config (BASELINE.md); the 271 KB table "
                             "is L2-resident across repetitions, so HBM does not bind here: "
                             "the kernel is FP64-issue bound (fp64_pipe)",
                     "fp64_pipe": {"active_frac": kprof.get("fp64_pipe_active"),
                                   "issue_active_frac": kprof.get("issue_active"),
                                   "source": kprof.get("fp64_source")}},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "gpu_launches": args.steps,
        "steps_metric": steps_info,
        "uncertified_draws_per_step": stats0.uncertified,
        "large_space": large,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-large-space", action="store_true",
                    help="skip the 1M-configuration stress measurement")
    ap.add_argument("--kernel-only", action="store_true",
                    help="time the search kernel only (for ncu captures)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
