"""Exhaustive B200 sweep of a benchmark space -> dataset directory in the
reference's on-disk format (space.csv, measurements.csv, arch.txt; SURVEY
section 8f rank 1/4), plus a JSON summary with the best configuration's
roofline fraction.

    python scripts/live_sweep.py --bench transpose --out datasets/transpose-b200 \
        [--size width=8192,height=8192] [--checkpoint gpurun_out/t.npz] [--no-profile]

Roofline denominators: HBM from MEASURED_PEAKS.json (hbm_gbs, measured copy);
FP32 pipe = SMs x 128 lanes x 2 flops x max SM clock; MUFU (rsqrt) = SMs x 16
x max SM clock (nominal, at clocks.max.sm).
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def peaks(sm_count, clock_hz=1.965e9):
    hbm = 6548.5e9
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            hbm = float(json.load(f).get("hbm_gbs", 6548.5)) * 1e9
    return {"hbm": hbm, "fp32": sm_count * 128 * 2 * clock_hz, "mufu": sm_count * 16 * clock_hz}


def roofline(bench, runtime_us, pk):
    """(achieved, peak, unit, frac) of one launch."""
    work = bench.work()
    t = runtime_us * 1e-6
    if bench.name == "transpose":
        return work / t / 1e9, pk["hbm"] / 1e9, "GB/s", work / t / pk["hbm"]
    if bench.name == "coulomb":
        return work / t / 1e9, pk["mufu"] / 1e9, "G interactions/s (MUFU rsqrt)", work / t / pk["mufu"]
    if bench.name == "nbody":
        fl = 20.0 * work
        return fl / t / 1e12, pk["fp32"] / 1e12, "TFLOP/s (20 flop/interaction)", fl / t / pk["fp32"]
    if bench.name == "conv":
        # both bounds are close at 7x7: the roofline time is the larger one
        bytes_ = 2.0 * 4.0 * bench.width * bench.height
        t_roof = max(work / pk["fp32"], bytes_ / pk["hbm"])
        return work / t / 1e12, pk["fp32"] / 1e12, \
            "TFLOP/s (frac = max(flop, HBM-byte) roofline time / time)", t_roof / t
    return work / t / 1e12, pk["fp32"] / 1e12, "TFLOP/s", work / t / pk["fp32"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--size", default="")
    ap.add_argument("--checkpoint", default=None)
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--limit", type=int, default=0, help="sweep only the first K configs")
    ap.add_argument("--budget-s", type=float, default=None,
                    help="stop measuring after this many seconds (partial dataset)")
    ap.add_argument("--update", default=None,
                    help="existing dataset dir: re-measure only --select configs, keep the rest")
    ap.add_argument("--select", default=None,
                    help="'tc5' (gemm tcgen05 variants), 'PARAM=value', or a comma list of "
                         "config indices")
    args = ap.parse_args()

    from paper_2102_05297_b200 import formats, live
    sizes = {}
    for kv in filter(None, args.size.split(",")):
        k, v = kv.split("=")
        sizes[k] = float(v) if "." in v else int(v)
    bench = live.benchmark(args.bench, **sizes)
    full_size = len(bench.space)
    bench.restrict_space()      # configurations that do not tile this input are not in its space
    src = live.CudaMeasurementSource(bench, reps=args.reps)
    t0 = time.time()
    last = [t0]

    def progress(i, n):
        if time.time() - last[0] > 30:
            last[0] = time.time()
            print(f"[sweep] {bench.name}: {i + 1}/{n} after {time.time() - t0:.0f} s", flush=True)

    if args.update:
        # re-measure a subset (variants whose kernel code changed) and merge
        ds = formats.load_dataset_dir(args.update)
        if args.select == "tc5":
            idx = [i for i in range(len(bench.space)) if bench.tc5(bench.values(i))]
        elif "=" in args.select:
            key, val = args.select.split("=")
            idx = [i for i in range(len(bench.space)) if bench.values(i)[key] == int(val)]
        else:
            idx = [int(x) for x in args.select.split(",")]
        src.compile_all(idx)
        names = list(ds.counter_names)
        for i in idx:
            m = src.measure(i, profiled=True)
            ds.runtime_us[i] = m.runtime_us
            ds.global_threads[i] = m.global_threads
            ds.counter_matrix[i] = [m.counters[a] for a in names]
            ds.has_record[i] = True
        ds._records = None
        formats.save_dataset(ds, args.out)
        rt = np.where(ds.has_record, ds.runtime_us, np.inf)
        best = int(np.argmin(rt))
        pk = peaks(src.tuner.sm_count)
        ach, peak, unit, frac = roofline(bench, float(rt[best]), pk)
        sub = np.array(idx)
        bsub = int(sub[np.argmin(rt[sub])])
        print(json.dumps({"bench": bench.name, "updated": len(idx), "best_index": best,
                          "best_values": bench.values(best), "best_us": float(rt[best]),
                          "best_updated_index": bsub, "best_updated_us": float(rt[bsub]),
                          "best_updated_values": bench.values(bsub),
                          "roofline": {"achieved": ach, "peak": peak, "unit": unit, "frac": frac}}))
        return
    if args.limit:
        # restricted sweep (smoke): measure the first K only
        idx = list(range(min(args.limit, len(bench.space))))
        src.compile_all(idx)
        rts = [src.measure(i, profiled=not args.no_profile).runtime_us for i in idx]
        print(json.dumps({"bench": bench.name, "measured": len(idx),
                          "best_us": float(min(rts)), "passes": src.profile_passes}))
        return
    res = live.sweep(src, profiled=not args.no_profile, checkpoint=args.checkpoint,
                     progress=progress, budget_s=args.budget_s)
    ds = res.dataset
    formats.save_dataset(ds, args.out)
    rt = np.where(ds.has_record, ds.runtime_us, np.inf)
    best = int(np.argmin(rt))
    pk = peaks(src.tuner.sm_count)
    ach, peak, unit, frac = roofline(bench, float(rt[best]), pk)
    well = int((rt <= 1.1 * rt[best]).sum())
    summary = {
        "bench": bench.name, "configs": len(ds.space), "space_before_input_constraints": full_size,
        "measured": int(ds.has_record.sum()),
        "failures": len(res.failures), "failure_examples": dict(list(res.failures.items())[:3]),
        "compile_s": round(res.seconds_compile, 1), "measure_s": round(res.seconds_measure, 1),
        "profile_passes": src.profile_passes, "sizes": sizes or "paper defaults",
        "best_index": best, "best_values": bench.values(best), "best_us": float(rt[best]),
        "median_us": float(np.median(rt[ds.has_record])),
        "well_performing_1.1x": well,
        "roofline": {"achieved": ach, "peak": peak, "unit": unit, "frac": frac,
                     "bound": bench.bound},
    }
    with open(os.path.join(args.out, "sweep_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
