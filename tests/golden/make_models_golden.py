"""Record model fixtures with the reference itself (build container only).

For the gradient synth preset and the coulomb / conv spaces (our synthetic
B200 stand-ins, rebuilt as reference Datasets) this trains the reference's
tree (seed 0) and regression model sets, saves the JSON model files and the
PredictionTable each yields:  tests/golden/models/<space>_<family>.json and
tests/golden/models/tables.npz.

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_models_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

from countertune import models, search, synth  # noqa: E402

from make_golden import ref_dataset_from_mine  # noqa: E402
from paper_2102_05297_b200 import spaces as my_spaces  # noqa: E402

OUT = os.path.join(HERE, "models")


def main():
    os.makedirs(OUT, exist_ok=True)
    sets = {"gradient": synth.build_dataset(synth.GENERATOR_PRESETS["gradient"]),
            "coulomb": ref_dataset_from_mine(my_spaces.coulomb()),
            "conv": ref_dataset_from_mine(my_spaces.conv())}
    tables = {}
    for name, ds in sets.items():
        for family in ("tree", "regression"):
            if name == "conv" and family == "tree":
                continue   # 3,928 configs x 19 trees: minutes in the reference
            ms = models.train_model_set(ds, family=family, seed=0)
            models.save_model_set(ms, os.path.join(OUT, f"{name}_{family}.json"))
            t = search.PredictionTable.from_model_set(ms, ds.space)
            tables[f"{name}_{family}_matrix"] = t.matrix
            tables[f"{name}_{family}_names"] = np.array(t.counter_names)
            print(name, family, t.matrix.shape, flush=True)
    np.savez_compressed(os.path.join(OUT, "tables.npz"), **tables)


if __name__ == "__main__":
    main()
