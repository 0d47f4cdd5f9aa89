"""Record golden trajectories on the B200-measured datasets (datasets/*-b200,
written by scripts/live_sweep.py) with the REFERENCE implementation.

The datasets are read with the reference's own loader
(countertune.space.load_dataset_dir, space.py:376-383), which also pins our
on-disk writer, and replayed with the reference's run_profile_search /
run_random_search exactly like make_golden.py does for the synthetic spaces.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_b200_golden.py

Writes tests/golden/ds_b200_<name>.npz and traj_b200_<name>.npz.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)

import make_golden  # noqa: E402  (imports the reference from /root/reference)
from countertune import space as rspace  # noqa: E402


def main():
    import sys as _sys
    which = set(_sys.argv[1:])
    for name, tree, reps in (("transpose", True, 32), ("coulomb", True, 32), ("conv", False, 16),
                             ("gemm", False, 16), ("nbody", False, 16)):
        if which and name not in which:
            continue
        d = os.path.join(ROOT, "datasets", f"{name}-b200")
        if not os.path.isdir(d):
            print("missing", d)
            continue
        ds = rspace.load_dataset_dir(d)
        make_golden.record_dataset(f"b200_{name}", ds, tree=tree, reps=reps)
        print("recorded", name, len(ds.space))


if __name__ == "__main__":
    main()
