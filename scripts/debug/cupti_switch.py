"""Which metric-set sequence crashes the CUPTI collector?  Each case in its
own process: python scripts/debug/cupti_switch.py [case]"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
CASES = {
    "sass": ["sass"], "g1": ["g1"], "all": ["all"], "nonsass": ["nonsass"],
    "all_sass": ["all", "sass"], "g1_sass": ["g1", "sass"], "nonsass_sass": ["nonsass", "sass"],
    "sass_all": ["sass", "all"], "all_g1": ["all", "g1"], "all_nonsass": ["all", "nonsass"],
    "measure_sass": ["measure", "sass"],
}

def run(seq):
    import numpy as np
    from paper_2102_05297_b200 import formats, live, counters as cc
    ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", "coulomb-b200"))
    best = int(np.argmin(np.where(ds.has_record, ds.runtime_us, np.inf)))
    src = live.CudaMeasurementSource(live.benchmark("coulomb"))
    t = src.tuner
    sass = [m for m, _ in cc.VOLTA_METRICS.values() if "sass" in m]
    sets = {"sass": sass, "g1": list(live.GROUP1_METRICS), "all": list(live.TABLE1_METRICS),
            "nonsass": [m for m in live.TABLE1_METRICS if m not in sass]}
    v = src.variant(best); launch = src.launch_of(best)
    for name in seq:
        print("step", name, flush=True)
        if name == "measure":
            m = src.measure(best, profiled=True); print("  runtime", m.runtime_us, flush=True)
            continue
        for k in range(2):
            vals, passes = t.profile(v, launch, sets[name])
            print("  passes", passes, "nan", int(np.isnan(vals).sum()), "of", len(vals), flush=True)
    src.close()
    print("ok", flush=True)

if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(CASES[sys.argv[1]]); sys.exit(0)
    for c in CASES:
        r = subprocess.run([sys.executable, __file__, c], capture_output=True, text=True, timeout=300)
        print("==", c, "rc", r.returncode, flush=True)
        print(r.stdout.strip(), flush=True)
        if r.returncode:
            print(r.stderr.strip()[-800:], flush=True)
