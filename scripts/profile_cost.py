"""Where a profiled step's wall time goes.

For each benchmark, on the best configuration of its B200 dataset: the wall
time of a timed step (CudaMeasurementSource.measure(profiled=False)) and of a
profiled step (24 Table-1 metrics, CUPTI range profiler), the profiled
step's phases (ct_tuner_profile_timing), and the collection cost of metric
subsets: the SASS-instrumented per-class instruction counts (group 4 of
SURVEY F13), the 13-metric single-pass group 1, and the rest.  Every
measurement runs in its own process with its own tuner (one metric set per
process, as a live search uses one), and prints one JSON line.

    python scripts/profile_cost.py [--benches coulomb,transpose,...] [--reps 5]
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SETS = ("steps", "sass_group4", "group1_13", "non_sass", "all24")


def metric_set(label):
    from paper_2102_05297_b200 import counters as cc, live
    sass = [m for m, _ in cc.VOLTA_METRICS.values() if "sass" in m]
    return {"sass_group4": sass, "group1_13": list(live.GROUP1_METRICS),
            "non_sass": [m for m in live.TABLE1_METRICS if m not in sass],
            "all24": list(live.TABLE1_METRICS)}[label]


def one(name, label, reps):
    from paper_2102_05297_b200 import formats, live
    ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", f"{name}-b200"))
    best = int(np.argmin(np.where(ds.has_record, ds.runtime_us, np.inf)))
    src = live.CudaMeasurementSource(live.benchmark(name))
    t = src.tuner
    out = {"bench": name, "best": best, "what": label}
    if label == "steps":
        src.measure(best, profiled=True)           # compile, host configuration, warm
        t0 = time.perf_counter()
        for _ in range(reps):
            src.measure(best, profiled=False)
        out["timed_step_s"] = (time.perf_counter() - t0) / reps
        t.profile_timing(reset=True)
        t0 = time.perf_counter()
        for _ in range(reps):
            src.measure(best, profiled=True)
        out["profiled_step_s"] = (time.perf_counter() - t0) / reps
        out["overhead"] = out["profiled_step_s"] / out["timed_step_s"]
        # a live step of a search also compiles the configuration (NVRTC +
        # module load; every search starts with no variant loaded)
        cs = []
        for _ in range(reps):
            src.reset_variants()
            t0 = time.perf_counter()
            src.variant(best)
            cs.append(time.perf_counter() - t0)
        out["compile_s"] = float(np.median(cs))
        out["overhead_with_compile"] = ((out["compile_s"] + out["profiled_step_s"])
                                        / (out["compile_s"] + out["timed_step_s"]))
        out["profiled_phases_us_per_call"] = {k: round(v / reps, 1) for k, v in
                                              t.profile_timing(reset=True).items()}
    else:
        ms = metric_set(label)
        v = src.variant(best)
        launch = src.launch_of(best)
        t.profile(v, launch, ms)                 # host configuration built outside the timing
        t.profile_timing(reset=True)
        t0 = time.perf_counter()
        for _ in range(reps):
            _, passes = t.profile(v, launch, ms)
        out["collect_s"] = (time.perf_counter() - t0) / reps
        out["metrics"] = len(ms)
        out["passes"] = passes
        out["phases_us"] = {k: round(v_ / reps, 1) for k, v_ in t.profile_timing(reset=True).items()}
    src.close()
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--benches", default="coulomb,transpose,nbody,conv,gemm")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--one", default=None, help="internal: bench:label")
    a = ap.parse_args()
    if a.one:
        name, label = a.one.split(":")
        one(name, label, a.reps)
        return
    for name in a.benches.split(","):
        for label in SETS:
            r = subprocess.run([sys.executable, "-X", "faulthandler", __file__, "--one",
                                f"{name}:{label}", "--reps", str(a.reps)],
                               capture_output=True, text=True, timeout=600)
            if r.returncode == 0:
                print(r.stdout.strip().splitlines()[-1], flush=True)
            else:
                print(json.dumps({"bench": name, "what": label, "rc": r.returncode,
                                  "stderr": r.stderr.strip()[-600:]}), flush=True)


if __name__ == "__main__":
    main()
