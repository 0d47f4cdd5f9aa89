"""Record-order fixtures, recorded with the reference itself (build container
only).

The reference keeps Dataset.records in measurements.csv order
(space.py:286-350), and model training iterates them in that order
(models.py:160-171, 237): the seeded half split, the stable sort's tie order
and the regression rows all depend on it.  This writes the B200 coulomb
dataset with its measurement rows in a seeded random order, trains the
reference's tree (seed 0) and regression model sets on it and records their
model files and counter errors:

  tests/golden/order/coulomb_shuffled/{space.csv,arch.txt,measurements.csv}
  tests/golden/order/coulomb_shuffled_{tree,regression}.json
  tests/golden/order/coulomb_shuffled_errors.json

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_order_golden.py
"""

import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from countertune import harness, models, space  # noqa: E402

OUT = os.path.join(HERE, "order")
SRC = os.path.join(ROOT, "datasets", "coulomb-b200")


def main():
    d = os.path.join(OUT, "coulomb_shuffled")
    os.makedirs(d, exist_ok=True)
    shutil.copy(os.path.join(SRC, "space.csv"), d)
    shutil.copy(os.path.join(SRC, "arch.txt"), d)
    lines = open(os.path.join(SRC, "measurements.csv")).read().splitlines()
    body = lines[1:]
    perm = np.random.default_rng(2024).permutation(len(body))
    with open(os.path.join(d, "measurements.csv"), "w", newline="\n") as f:
        f.write("\n".join([lines[0]] + [body[i] for i in perm]) + "\n")
    ds = space.load_dataset_dir(d)
    assert [r.config_index for r in ds.records][:5] != [0, 1, 2, 3, 4]
    errors = {}
    for family in ("tree", "regression"):
        ms = models.train_model_set(ds, family=family, seed=0)
        models.save_model_set(ms, os.path.join(OUT, f"coulomb_shuffled_{family}.json"))
        errors[family] = {k: [repr(a), repr(b)]
                          for k, (a, b) in harness.counter_prediction_errors(ms, ds).items()}
    with open(os.path.join(OUT, "coulomb_shuffled_errors.json"), "w") as f:
        json.dump(errors, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
