"""Table-1 values of one profiled step: run under CT_TUNE_REPLAY=user|kernel
and compare (prints JSON of abbr -> value, passes)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2102_05297_b200 import formats, live
name = sys.argv[1]
ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", f"{name}-b200"))
best = int(np.argmin(np.where(ds.has_record, ds.runtime_us, np.inf)))
src = live.CudaMeasurementSource(live.benchmark(name))
out = {}
for k in range(2):
    m = src.measure(best, profiled=True)
    out[f"run{k}"] = m.counters
out["passes"] = src.profile_passes
print(json.dumps(out))
