"""Cross-input model reuse (BASELINE config 4),
recorded with the reference itself (build container only).

Datasets (B200 sweeps, scripts/resweep_r02.sh + scripts/live_sweep.py):
  GEMM   datasets/gemm-b200 (2048^3), gemm-128-b200, gemm-16x4096-b200,
         gemm-4096x16-b200 (configurations that do not tile an input are
         not in its space)
  N-body datasets/nbody-b200 (16,384 bodies), nbody-32768-b200 (the paper's 131,072 costs ~3 s per configuration under the profiler on B200, 2.6 h for the space)
  conv   datasets/conv-b200 (4096^2), conv-8192-b200
For every dataset the reference trains its decision-tree model set (seed 0,
models.py:354-369); then for every (run dataset, model dataset) pair of a
family it runs harness.cross_evaluate(model, run dataset) (harness.py:292-323)
with R = 100 repetitions, seed 42, and records the per-counter errors and
both reports:

  tests/golden/cross/models/<dataset>_tree.json
  tests/golden/cross/cross_<run>__<model>.npz

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cross_golden.py
"""

import logging
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
import make_golden  # noqa: E402,F401  (puts the reference on sys.path)

OUT = os.path.join(HERE, "cross")
FAMILIES = {
    "gemm": ["gemm", "gemm-128", "gemm-16x4096", "gemm-4096x16"],
    "nbody": ["nbody", "nbody-32768"],
    "conv": ["conv", "conv-8192"],
}
REPS, SEED = 100, 42
REPORT_FIELDS = ("steps", "step_curve_mean", "step_curve_std", "time_grid_seconds",
                 "time_curve_mean", "time_curve_std")


def _dir(name):
    return os.path.join(ROOT, "datasets", f"{name}-b200")


def train(name):
    from countertune import models, space
    logging.disable(logging.WARNING)
    ds = space.load_dataset_dir(_dir(name))
    ms = models.train_model_set(ds, family="tree", seed=0)
    models.save_model_set(ms, os.path.join(OUT, "models", f"{name}_tree.json"))
    return name


def cross(pair):
    from countertune import harness, models, space
    run, model = pair
    ds = space.load_dataset_dir(_dir(run))
    ms = models.load_model_set(os.path.join(OUT, "models", f"{model}_tree.json"))
    rep = harness.cross_evaluate(ms, ds, repetitions=REPS, seed=SEED)
    out = {"model_label": np.array(rep.model_label), "dataset_label": np.array(rep.dataset_label),
           "error_names": np.array(list(rep.counter_errors)),
           "error_values": np.array(list(rep.counter_errors.values()))}
    for tag, r in (("profile", rep.profile_report), ("random", rep.random_report)):
        for f in REPORT_FIELDS:
            out[f"{tag}_{f}"] = getattr(r, f)
        out[f"{tag}_censored"] = np.int64(r.censored)
        out[f"{tag}_mean_time_seconds"] = np.float64(r.mean_time_seconds)
    out["improvement"] = np.float64(rep.profile_report.improvement)
    harness.write_counter_errors(rep.counter_errors,
                                 os.path.join(OUT, f"counter_errors_{run}__{model}.csv"))
    np.savez_compressed(os.path.join(OUT, f"cross_{run}__{model}.npz"), **out)
    return run, model, rep.profile_report.improvement


def main():
    os.makedirs(os.path.join(OUT, "models"), exist_ok=True)
    names = [n for fam in FAMILIES.values() for n in fam if os.path.isdir(_dir(n))]
    with ProcessPoolExecutor(8) as pool:
        for n in pool.map(train, names):
            print("trained", n, flush=True)
        pairs = [(r, m) for fam in FAMILIES.values() for r in fam for m in fam
                 if r in names and m in names]
        for run, model, imp in pool.map(cross, pairs):
            print(f"run {run} model {model}: improvement {imp:.3f}", flush=True)


if __name__ == "__main__":
    main()
