"""CUPTI DRAM metrics on the transpose best config with several metric sets."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2102_05297_b200 import formats, counters as cc
from paper_2102_05297_b200.live import CudaMeasurementSource, benchmark
from paper_2102_05297_b200.tuner import Tuner
t = Tuner(0)
ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", "transpose-b200"))
best = int(np.argmin(np.where(ds.has_record, ds.runtime_us, np.inf)))
src = CudaMeasurementSource(benchmark("transpose"), tuner=t)
v = src.variant(best); launch = src.launch_of(best)
sets = [("DRAM_RT", "DRAM_WT", "L2_RT", "L2_WT", "INST_EXE", "INST_F32"), ("DRAM_RT", "DRAM_WT"),
        ("DRAM_RT",), tuple(cc.VOLTA_METRICS)]
for s in sets:
    ms = [cc.VOLTA_METRICS[a][0] for a in s]
    for k in range(2):
        vals, passes = t.profile(v, launch, ms)
        print(len(s), "passes", passes, dict(zip(s, np.round(vals, 1).tolist())), flush=True)
