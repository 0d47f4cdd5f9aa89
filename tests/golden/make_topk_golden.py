"""score_top_k fixtures, recorded with the reference itself (build container
only): run_profile_search trajectories with the top-K neighbourhood
(search.py:133-140) and harness.simulate reports with ExperimentSpec.score_top_k
(harness.py:155-158).

  traj_topk_<set>.npz   per K: <K>_idx / _prof / _off / _status (64 reps,
                        SeedSequence(42).spawn, i=40, n=5, exact model,
                        stop at the well-performing set)
  sim_topk.npz          gradient, profile searcher, K = 40, 50 reps, seed 7

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_topk_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import REF  # noqa: E402,F401  (puts the reference on sys.path)
from countertune import harness, models, search, synth  # noqa: E402
from countertune import space as rspace  # noqa: E402

# K below n (the pool empties mid-iteration), near n, and well inside the space
TOPK = (1, 3, 7, 40, 300)


def record(name, ds, reps=64, i=40):
    exact = search.PredictionTable.from_model_set(models.ExactModelSet(ds), ds.space)
    src = search.DatasetReplaySource(ds)
    well = rspace.well_performing_set(ds, 1.1)
    out = {"topk": np.array(TOPK, dtype=np.int64), "reps": np.int64(reps), "i": np.int64(i),
           "well": np.array(sorted(well), dtype=np.int64)}
    for K in TOPK:
        seeds = np.random.SeedSequence(42).spawn(reps)
        idx, prof, off, status = [], [], [0], []
        for r in range(reps):
            tr = search.run_profile_search(src, exact, i=i, n=5, seed=seeds[r],
                                           stop_indices=well, score_top_k=K)
            idx.extend(s.config_index for s in tr.steps)
            prof.extend(s.profiled for s in tr.steps)
            off.append(len(idx))
            status.append(tr.status)
        out[f"k{K}_idx"] = np.array(idx, dtype=np.int32)
        out[f"k{K}_prof"] = np.array(prof, dtype=bool)
        out[f"k{K}_off"] = np.array(off, dtype=np.int64)
        out[f"k{K}_status"] = np.array(status)
        print(name, K, "mean steps", np.mean(np.diff(off)), flush=True)
    np.savez_compressed(os.path.join(HERE, f"traj_topk_{name}.npz"), **out)


def record_simulate(ds):
    spec = harness.ExperimentSpec(dataset=ds, searcher="profile", model=models.ExactModelSet(ds),
                                  name="profile-topk", repetitions=50, seed=7,
                                  time_repetitions=20, score_top_k=40)
    rep = harness.simulate(spec)
    res = {}
    for f in ("steps", "step_curve_mean", "step_curve_std", "time_grid_seconds",
              "time_curve_mean", "time_curve_std"):
        res[f] = getattr(rep, f)
    res["censored"] = np.int64(rep.censored)
    res["mean_time_seconds"] = np.float64(rep.mean_time_seconds)
    np.savez_compressed(os.path.join(HERE, "sim_topk.npz"), **res)


def main():
    grad = synth.build_dataset(synth.GENERATOR_PRESETS["gradient"])
    record("gradient", grad)
    record("b200_transpose", rspace.load_dataset_dir(
        os.path.join(os.path.dirname(os.path.dirname(HERE)), "datasets", "transpose-b200")),
        reps=32)
    record_simulate(grad)


if __name__ == "__main__":
    main()
