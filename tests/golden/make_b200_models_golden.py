"""Tree- and regression-model trajectories on the B200-measured gemm / conv /
nbody datasets, recorded with the reference itself (build container only;
one process per dataset, the reference trains 19 trees per dataset).

For each dataset the reference trains its decision-tree model set (seed 0)
and its regression model set (models.py:174-369), saves both model files,
builds their PredictionTables and replays run_profile_search with each
(16 repetitions, SeedSequence(42).spawn, i=40, n=5, stop at the
well-performing set):

  tests/golden/models/b200_<name>_{tree,regression}.json
  tests/golden/traj_b200_<name>_models.npz   {tree,regression}_{matrix,names},
                                             {tree,regression}_stop_{idx,prof,off,status}

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_b200_models_golden.py
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

REPS, I = 16, 40


def record(name):
    from countertune import models, search
    from countertune import space as rspace
    logging.disable(logging.WARNING)
    ds = rspace.load_dataset_dir(os.path.join(ROOT, "datasets", f"{name}-b200"))
    src = search.DatasetReplaySource(ds)
    well = rspace.well_performing_set(ds, 1.1)
    out = {"reps": np.int64(REPS), "i": np.int64(I),
           "well": np.array(sorted(well), dtype=np.int64)}
    for family in ("tree", "regression"):
        ms = models.train_model_set(ds, family=family, seed=0)
        models.save_model_set(ms, os.path.join(HERE, "models", f"b200_{name}_{family}.json"))
        table = search.PredictionTable.from_model_set(ms, ds.space)
        out[f"{family}_matrix"] = table.matrix
        out[f"{family}_names"] = np.array(table.counter_names)
        seeds = np.random.SeedSequence(42).spawn(REPS)
        idx, prof, off, status = [], [], [0], []
        for r in range(REPS):
            tr = search.run_profile_search(src, table, i=I, n=5, seed=seeds[r], stop_indices=well)
            idx.extend(s.config_index for s in tr.steps)
            prof.extend(s.profiled for s in tr.steps)
            off.append(len(idx))
            status.append(tr.status)
        key = f"{family}_stop"
        out[key + "_idx"] = np.array(idx, dtype=np.int32)
        out[key + "_prof"] = np.array(prof, dtype=bool)
        out[key + "_off"] = np.array(off, dtype=np.int64)
        out[key + "_status"] = np.array(status)
    np.savez_compressed(os.path.join(HERE, f"traj_b200_{name}_models.npz"), **out)
    return name


def main():
    names = sys.argv[1:] or ["gemm", "conv", "nbody"]
    with ProcessPoolExecutor(len(names)) as pool:
        for name in pool.map(record, names):
            print("recorded", name, flush=True)


if __name__ == "__main__":
    main()
