"""Where a profiled step's wall time goes.

For each benchmark, on the best configuration of its B200 dataset: the wall
time of a timed step (CudaMeasurementSource.measure(profiled=False)) and of a
profiled step (24 Table-1 metrics, CUPTI range profiler), the profiled
step's phases (ct_tuner_profile_timing), and the collection cost of metric
subsets: the SASS-instrumented per-class instruction counts (group 4 of
SURVEY F13), the 13-metric single-pass group 1, and the rest.

    python scripts/profile_cost.py [--benches coulomb,transpose,...] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--benches", default="coulomb,transpose,nbody,conv,gemm")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from paper_2102_05297_b200 import formats, live
    from paper_2102_05297_b200 import counters as cc
    sass = [m for m, _ in cc.VOLTA_METRICS.values() if "sass" in m]
    group1 = list(live.GROUP1_METRICS)
    for name in a.benches.split(","):
        ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", f"{name}-b200"))
        best = int(np.argmin(np.where(ds.has_record, ds.runtime_us, np.inf)))
        src = live.CudaMeasurementSource(live.benchmark(name))
        src.measure(best, profiled=True)           # compile, host configs, warm
        t = src.tuner
        out = {"bench": name, "best": best}
        t0 = time.perf_counter()
        for _ in range(a.reps):
            src.measure(best, profiled=False)
        out["timed_step_s"] = (time.perf_counter() - t0) / a.reps
        t.profile_timing(reset=True)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            src.measure(best, profiled=True)
        out["profiled_step_s"] = (time.perf_counter() - t0) / a.reps
        out["profiled_phases_us_per_call"] = {k: v / a.reps for k, v in
                                              t.profile_timing(reset=True).items()}
        v = src.variant(best)
        launch = src.launch_of(best)
        for label, ms in (("sass_group4", sass), ("group1_13", group1),
                          ("non_sass", [m for m in live.TABLE1_METRICS if m not in sass]),
                          ("all24", list(live.TABLE1_METRICS))):
            print(f"[profile_cost] {name}: {label}", file=sys.stderr, flush=True)
            t.profile(v, launch, ms)                 # host config built outside the timing
            t.profile_timing(reset=True)
            t0 = time.perf_counter()
            for _ in range(a.reps):
                _, passes = t.profile(v, launch, ms)
            out[f"{label}_s"] = (time.perf_counter() - t0) / a.reps
            out[f"{label}_passes"] = passes
            out[f"{label}_phases_us"] = {k: round(v_ / a.reps, 1) for k, v_ in
                                         t.profile_timing(reset=True).items()}
        if name in ("coulomb", "transpose"):
            # the same profiled step with the whole space's modules loaded
            # in the context (the state a session without unloads reaches)
            t0 = time.perf_counter()
            bad = src.compile_all()
            out["compile_all_s"] = time.perf_counter() - t0
            out["modules_loaded"] = len(src._variants)
            t0 = time.perf_counter()
            for _ in range(a.reps):
                src.measure(best, profiled=True)
            out["profiled_step_all_modules_s"] = (time.perf_counter() - t0) / a.reps
            out["profiled_all_modules_phases_us"] = {k: round(v_ / a.reps, 1) for k, v_ in
                                                     t.profile_timing(reset=True).items()}
            del bad
        src.close()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
