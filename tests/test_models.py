"""Model training / files against the reference (tests/golden/models, written
by make_models_golden.py with the reference itself): same trees, same
regression fits, byte-identical model files, same prediction tables."""

import filecmp
import logging
import os

import numpy as np
import pytest

from conftest import GOLDEN, dataset_from_golden

MODELS = os.path.join(GOLDEN, "models")


def _dataset(name):
    from paper_2102_05297_b200 import spaces
    if name == "gradient":
        return dataset_from_golden("gradient")
    return spaces.SPACES[name]()


@pytest.mark.parametrize("name,family", [("gradient", "tree"), ("coulomb", "tree"),
                                         ("gradient", "regression"),
                                         ("coulomb", "regression"), ("conv", "regression")])
def test_trained_model_file_is_byte_identical_to_reference(name, family, tmp_path, caplog):
    from paper_2102_05297_b200 import models
    caplog.set_level(logging.ERROR)
    ms = models.train_model_set(_dataset(name), family=family, seed=0)
    out = tmp_path / "m.json"
    models.save_model_set(ms, out)
    assert filecmp.cmp(out, os.path.join(MODELS, f"{name}_{family}.json"), shallow=False)


@pytest.mark.parametrize("name,family", [("gradient", "tree"), ("coulomb", "regression")])
def test_host_predict_matches_reference_table(name, family):
    from paper_2102_05297_b200 import models
    ms = models.load_model_set(os.path.join(MODELS, f"{name}_{family}.json"))
    tables = np.load(os.path.join(MODELS, "tables.npz"))
    want = tables[f"{name}_{family}_matrix"]
    assert ms.counters == tuple(str(x) for x in tables[f"{name}_{family}_names"])
    ds = _dataset(name)
    for conf in ds.space.configurations[::7]:
        pred = ms.predict(conf)
        row = [pred.get(c, 0.0) for c in ms.counters]
        np.testing.assert_array_equal(row, want[conf.index])


def test_model_file_round_trip_and_errors(tmp_path):
    from paper_2102_05297_b200 import models
    from paper_2102_05297_b200.errors import ModelFormatError
    src = os.path.join(MODELS, "coulomb_tree.json")
    ms = models.load_model_set(src)
    out = tmp_path / "again.json"
    models.save_model_set(ms, out)
    assert filecmp.cmp(out, src, shallow=False)
    bad = tmp_path / "bad.json"
    bad.write_text('{"format": "countertune-model", "version": 2}')
    with pytest.raises(ModelFormatError, match="unsupported version"):
        models.load_model_set(bad)
    bad.write_text('{"format": "countertune-model", "version": 1}')
    with pytest.raises(ModelFormatError, match="malformed"):
        models.load_model_set(bad)
    bad.write_text('{"format": ')
    with pytest.raises(ModelFormatError, match="not a complete model file"):
        models.load_model_set(bad)


def test_training_errors_and_family_dispatch():
    from paper_2102_05297_b200 import models
    from paper_2102_05297_b200.counters import ArchProfile
    from paper_2102_05297_b200.errors import ModelTrainingError
    from paper_2102_05297_b200.space import Dataset, TuningParameter, TuningSpace
    with pytest.raises(ValueError, match="unknown model family"):
        models.train_model_set(_dataset("coulomb"), family="forest")
    p = TuningParameter.make("x", [1, 2, 3])
    sp = TuningSpace.from_assignments([p], np.array([[1.0], [2.0], [3.0]]))
    ds = Dataset(sp, ArchProfile("a", "volta_plus", 10), "in", runtime_us=np.ones(3),
                 global_threads=np.ones(3, dtype=np.int64), counter_names=("DRAM_RT",),
                 counter_matrix=np.ones((3, 1)))
    with pytest.raises(ModelTrainingError, match="at least 4 records"):
        models.train_decision_tree(ds, "DRAM_RT")


def test_model_program_flattening():
    """The GPU programme walks the same trees: re-walk it on the host."""
    from paper_2102_05297_b200 import models
    ms = models.load_model_set(os.path.join(MODELS, "gradient_tree.json"))
    prog = models.compile_model_program(ms)
    tables = np.load(os.path.join(MODELS, "tables.npz"))
    want = tables["gradient_tree_matrix"]
    ds = _dataset("gradient")
    A = ds.space.assignments
    for i in range(0, A.shape[0], 37):
        for c in range(prog.n_cols):
            node = int(prog.col_root[c])
            while prog.node_feature[node] >= 0:
                f = prog.node_feature[node]
                node = int(prog.node_left[node] if A[i, f] <= prog.node_threshold[node]
                           else prog.node_right[node])
            v = prog.node_value[node]
            assert (v if v > 0.0 else 0.0) == want[i, c]


ORDER = os.path.join(GOLDEN, "order")


@pytest.mark.parametrize("family", ["tree", "regression"])
def test_training_follows_measurement_file_order(family, tmp_path, caplog):
    """A measurements.csv whose rows are not sorted by config_index trains the
    reference's models (make_order_golden.py): rows are used in file order,
    as the reference's Dataset.records are (models.py:160-171, 237)."""
    import json
    from paper_2102_05297_b200 import formats, models
    caplog.set_level(logging.ERROR)
    ds = formats.load_dataset_dir(os.path.join(ORDER, "coulomb_shuffled"))
    assert ds.record_order[:5].tolist() != [0, 1, 2, 3, 4]
    ms = models.train_model_set(ds, family=family, seed=0)
    out = tmp_path / "m.json"
    models.save_model_set(ms, out)
    assert filecmp.cmp(out, os.path.join(ORDER, f"coulomb_shuffled_{family}.json"),
                       shallow=False)


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["tree", "regression"])
def test_counter_errors_follow_measurement_file_order(family):
    """counter_prediction_errors (harness.py:268-289) averages over records in
    file order; the GPU prediction table reproduces the reference's values."""
    import json
    from paper_2102_05297_b200 import formats, harness, models
    ds = formats.load_dataset_dir(os.path.join(ORDER, "coulomb_shuffled"))
    ms = models.load_model_set(os.path.join(ORDER, f"coulomb_shuffled_{family}.json"))
    want = json.load(open(os.path.join(ORDER, "coulomb_shuffled_errors.json")))[family]
    got = harness.counter_prediction_errors(ms, ds)
    assert {k: [repr(a), repr(b)] for k, (a, b) in got.items()} == want


@pytest.mark.parametrize("name,family", [("gemm", "regression"), ("conv", "regression"),
                                         ("nbody", "regression"), ("nbody", "tree")])
def test_b200_model_files_are_byte_identical_to_reference(name, family, tmp_path, caplog):
    """Training on the B200-measured datasets gives the reference's model
    files (make_b200_models_golden.py; the gemm / conv trees are pinned the
    same way on the GPU box, tests/test_gpu_models.py)."""
    from paper_2102_05297_b200 import formats, models
    caplog.set_level(logging.ERROR)
    ds = formats.load_dataset_dir(os.path.join(os.path.dirname(GOLDEN), "..", "datasets",
                                               f"{name}-b200"))
    ms = models.train_model_set(ds, family=family, seed=0)
    out = tmp_path / "m.json"
    models.save_model_set(ms, out)
    assert filecmp.cmp(out, os.path.join(MODELS, f"b200_{name}_{family}.json"), shallow=False)
