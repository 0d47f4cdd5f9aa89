"""The paper's input-portability study (Table 6) on the B200
datasets: for every (run dataset, model dataset) pair of a family, the
profile searcher driven by a decision-tree model trained on the model
dataset (the reference's trees, tests/golden/cross/models) against random
search on the run dataset -- harness.cross_evaluate on the GPU, R = 1000,
seed 42 -- plus the counter prediction errors.

    python scripts/cross_matrix.py [--reps 1000] [--out profiles/r02_cross_input.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
FAMILIES = {
    "gemm": ["gemm", "gemm-128", "gemm-16x4096", "gemm-4096x16"],
    "nbody": ["nbody", "nbody-32768"],
    "conv": ["conv", "conv-8192"],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=1000)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from paper_2102_05297_b200 import cross_evaluate, formats, models
    res = {}
    for fam, names in FAMILIES.items():
        for run in names:
            d = os.path.join(ROOT, "datasets", f"{run}-b200")
            if not os.path.isdir(d):
                continue
            ds = formats.load_dataset_dir(d)
            for model in names:
                mp = os.path.join(ROOT, "tests", "golden", "cross", "models", f"{model}_tree.json")
                if not os.path.exists(mp):
                    continue
                ms = models.load_model_set(mp)
                t0 = time.perf_counter()
                rep = cross_evaluate(ms, ds, repetitions=a.reps, seed=42)
                res[f"{run} <- {model}"] = {
                    "run": run, "model": model, "configs": len(ds.space),
                    "improvement": rep.profile_report.improvement,
                    "profile_mean_steps": rep.profile_report.mean_steps,
                    "random_mean_steps": rep.random_report.mean_steps,
                    "profile_censored": rep.profile_report.censored,
                    "seconds": time.perf_counter() - t0,
                    "counter_mae": {k: v[0] for k, v in rep.counter_errors.items()}}
                print(json.dumps({k: v for k, v in res[f"{run} <- {model}"].items()
                                  if k != "counter_mae"}), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
