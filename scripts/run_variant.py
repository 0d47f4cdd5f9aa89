"""Launch one benchmark variant a few times (for ncu captures of the best
configurations of the B200 sweeps).

    python scripts/run_variant.py --bench gemm --index 5664 [--launches 3]
    python scripts/run_variant.py --bench transpose --best datasets/transpose-b200
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bench", required=True)
    ap.add_argument("--index", type=int, default=None)
    ap.add_argument("--best", default=None, help="dataset dir: run its best configuration")
    ap.add_argument("--launches", type=int, default=3)
    a = ap.parse_args()
    from paper_2102_05297_b200 import formats, live
    bench = live.benchmark(a.bench)
    idx = a.index
    if a.best:
        ds = formats.load_dataset_dir(a.best)
        idx = int(np.argmin(np.where(ds.has_record, ds.runtime_us, np.inf)))
    src = live.CudaMeasurementSource(bench, flush_l2=False)
    v = src.variant(idx)
    t = src.tuner.time(v, src.launch_of(idx), warmup=0, reps=a.launches, flush_l2=True)
    print(f"{a.bench} config {idx} {bench.values(idx)}: {np.round(t, 1).tolist()} us")


if __name__ == "__main__":
    main()
