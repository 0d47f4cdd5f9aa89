"""Reference trajectories on the 205,216-configuration GEMM-full space
(synthetic stand-in, spaces.gemm_full), recorded with the reference itself
(build container only; 8 worker processes, ~10 min).

At this size the device's draw certificate ((8N + 128) 2^-53 T) rejects
about 7e-5 of the draws, which the device then re-decides with the
sequential float64 cumsum over its own (correctly rounded) weights.  These
trajectories pin that fallback against numpy's cumsum over its SVML pow
weights: 256 repetitions x 40 outer iterations x 5 draws (throughput mode,
no stop set), exact model, SeedSequence(42).spawn(256).

  tests/golden/traj_gemm_full.npz   exact_nostop_{idx,prof,off,status}, reps, i

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gemmfull_golden.py
"""

import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import ref_dataset_from_mine  # noqa: E402  (puts the reference on sys.path)

REPS, I = 256, 40
_STATE = {}


def _init():
    from countertune import models, search
    from paper_2102_05297_b200 import spaces
    ds = ref_dataset_from_mine(spaces.gemm_full())
    _STATE["src"] = search.DatasetReplaySource(ds)
    _STATE["table"] = search.PredictionTable.from_model_set(models.ExactModelSet(ds), ds.space)


def _run(reps):
    from countertune import search
    seeds = np.random.SeedSequence(42).spawn(REPS)
    out = []
    for r in reps:
        tr = search.run_profile_search(_STATE["src"], _STATE["table"], i=I, n=5, seed=seeds[r],
                                       stop_indices=frozenset())
        out.append((r, [s.config_index for s in tr.steps], [s.profiled for s in tr.steps],
                    tr.status))
    return out


def main():
    workers = int(os.environ.get("WORKERS", "8"))
    chunks = [list(range(k, REPS, workers)) for k in range(workers)]
    res = []
    with ProcessPoolExecutor(workers, initializer=_init) as pool:
        for part in pool.map(_run, chunks):
            res.extend(part)
    res.sort(key=lambda x: x[0])
    idx, prof, off, status = [], [], [0], []
    for _, i_, p_, st in res:
        idx.extend(i_)
        prof.extend(p_)
        off.append(len(idx))
        status.append(st)
    np.savez_compressed(os.path.join(HERE, "traj_gemm_full.npz"),
                        exact_nostop_idx=np.array(idx, dtype=np.int32),
                        exact_nostop_prof=np.array(prof, dtype=bool),
                        exact_nostop_off=np.array(off, dtype=np.int64),
                        exact_nostop_status=np.array(status), reps=np.int64(REPS),
                        i=np.int64(I))
    print("wrote traj_gemm_full.npz", len(idx), "steps")


if __name__ == "__main__":
    main()
