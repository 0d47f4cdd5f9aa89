"""Is a repeated NVRTC compile of the same configuration cheaper?  One
process: 12 fresh configurations (A), unload, A again, 12 new (B)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2102_05297_b200 import formats
from paper_2102_05297_b200.live import CudaMeasurementSource, benchmark
ds = formats.load_dataset_dir(sys.argv[1])
src = CudaMeasurementSource(benchmark(sys.argv[2]))
ok = np.flatnonzero(ds.has_record)
perm = np.random.default_rng(int(sys.argv[3])).permutation(ok).tolist()
A, B = perm[:12], perm[12:24]
def run(idx, label):
    ts = []
    for i in idx:
        t0 = time.perf_counter(); src.variant(i); ts.append(time.perf_counter() - t0)
    print(json.dumps({"label": label, "median_ms": 1e3 * float(np.median(ts)),
                      "ms": [round(1e3 * t) for t in ts]}), flush=True)
run(A, "A first"); src.reset_variants(); run(A, "A again"); run(B, "B first")
src.reset_variants(); run(B, "B again")
