"""Wall cost of a live step (compile + load + time) in each CUPTI state.

    python scripts/debug/load_cost.py datasets/gemm-b200 gemm

Phases, 12 fresh variants each: no profiler yet; after one group-1 profiled
step (range-profiler object alive); after reset_variants (object disabled);
after one full-set profiled step; after reset again.  Prints the per-step
split compile / time."""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    from paper_2102_05297_b200 import formats
    from paper_2102_05297_b200.live import GROUP1_METRICS, CudaMeasurementSource, benchmark
    ds = formats.load_dataset_dir(sys.argv[1])
    bench = benchmark(sys.argv[2])
    g1 = CudaMeasurementSource(bench, metrics=GROUP1_METRICS, fill_from=ds)
    full = CudaMeasurementSource(bench, tuner=g1.tuner)
    ok = np.flatnonzero(ds.has_record)
    order = iter(np.random.default_rng(0).permutation(ok).tolist())

    def steps(src, label, k=12):
        c_s, t_s = [], []
        for _ in range(k):
            i = next(order)
            t0 = time.perf_counter()
            src.variant(i)
            t1 = time.perf_counter()
            src.measure(i, profiled=False)
            t2 = time.perf_counter()
            c_s.append(t1 - t0)
            t_s.append(t2 - t1)
        out = {"phase": label, "compile_load_ms": 1e3 * float(np.median(c_s)),
               "time_ms": 1e3 * float(np.median(t_s)),
               "compile_load_ms_max": 1e3 * float(np.max(c_s))}
        print(json.dumps(out), flush=True)

    def profiled(src, label):
        i = next(order)
        src.variant(i)
        t0 = time.perf_counter()
        src.measure(i, profiled=True)
        t1 = time.perf_counter()
        src.measure(i, profiled=True)
        t2 = time.perf_counter()
        print(json.dumps({"phase": label, "first_profiled_ms": 1e3 * (t1 - t0),
                          "second_profiled_ms": 1e3 * (t2 - t1)}), flush=True)

    steps(g1, "no profiler yet")
    profiled(g1, "group1 profiled")
    steps(g1, "group1 object alive")
    g1.reset_variants()
    steps(g1, "after reset (disabled)")
    profiled(g1, "group1 profiled again")
    steps(g1, "group1 object alive again")
    full.reset_variants()
    profiled(full, "full profiled")
    steps(full, "full object alive")
    full.reset_variants()
    steps(full, "after reset from full")
    g1.close()


if __name__ == "__main__":
    main()
