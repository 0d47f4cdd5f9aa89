"""Cross-input model reuse (BASELINE config 4): harness.cross_evaluate on the
GPU against the reference's own cross_evaluate (harness.py:292-323) on the
B200 datasets at two input sizes (tests/golden/make_cross_golden.py): the
per-counter prediction errors, both reports and the improvement, bit for
bit, and the counter_errors.csv writer (harness.py:391-398) byte for byte."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

CROSS = os.path.join(GOLDEN, "cross")
CASES = sorted(os.path.basename(p)[len("cross_"):-len(".npz")]
               for p in glob.glob(os.path.join(CROSS, "cross_*.npz")))
FIELDS = ("steps", "step_curve_mean", "step_curve_std", "time_grid_seconds",
          "time_curve_mean", "time_curve_std")


@pytest.mark.parametrize("case", CASES)
def test_counter_errors_csv_matches_reference_writer(case, tmp_path):
    from paper_2102_05297_b200 import write_counter_errors
    g = np.load(os.path.join(CROSS, f"cross_{case}.npz"))
    errors = {str(k): (float(v[0]), float(v[1])) for k, v in zip(g["error_names"], g["error_values"])}
    out = tmp_path / "counter_errors.csv"
    write_counter_errors(errors, out)
    assert out.read_bytes() == open(os.path.join(CROSS, f"counter_errors_{case}.csv"), "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_cross_evaluate_matches_reference(case):
    from paper_2102_05297_b200 import cross_evaluate, formats, models
    run, model = case.split("__")
    g = np.load(os.path.join(CROSS, f"cross_{case}.npz"))
    ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", f"{run}-b200"))
    ms = models.load_model_set(os.path.join(CROSS, "models", f"{model}_tree.json"))
    rep = cross_evaluate(ms, ds, repetitions=100, seed=42)
    assert rep.model_label == str(g["model_label"])
    assert rep.dataset_label == str(g["dataset_label"])
    assert list(rep.counter_errors) == [str(x) for x in g["error_names"]]
    np.testing.assert_array_equal(np.array(list(rep.counter_errors.values())), g["error_values"])
    for tag, r in (("profile", rep.profile_report), ("random", rep.random_report)):
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(r, f), g[f"{tag}_{f}"], err_msg=f"{tag} {f}")
        assert r.censored == int(g[f"{tag}_censored"])
        assert r.mean_time_seconds == float(g[f"{tag}_mean_time_seconds"])
    assert rep.profile_report.improvement == float(g["improvement"])
