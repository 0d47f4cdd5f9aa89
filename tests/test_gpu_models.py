"""Model-driven searches on the B200-measured datasets: the reference's tree
and regression model sets (make_b200_models_golden.py), their prediction
tables computed on the GPU (ct_model_predict) and the batched device search
driven by them, against the reference's tables and trajectories."""

import logging
import os

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden, ragged

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["gemm", "conv", "nbody"])
@pytest.mark.parametrize("family", ["tree", "regression"])
def test_model_tables_and_trajectories_match_reference(name, family):
    from paper_2102_05297_b200 import _native, formats, models
    from paper_2102_05297_b200.search import PredictionTable, search_params
    from paper_2102_05297_b200.space import replay_arrays
    traj = golden(f"traj_b200_{name}_models.npz")
    ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", f"{name}-b200"))
    ms = models.load_model_set(os.path.join(GOLDEN, "models", f"b200_{name}_{family}.json"))
    table = PredictionTable.from_model_set(ms, ds.space)          # GPU inference
    assert table.counter_names == tuple(str(x) for x in traj[f"{family}_names"])
    np.testing.assert_array_equal(table.matrix, traj[f"{family}_matrix"])
    reps, i = int(traj["reps"]), int(traj["i"])
    rt, th, req, hr = replay_arrays(ds)
    stop = np.zeros(len(ds.space), dtype=np.uint8)
    stop[traj["well"]] = 1
    ctx = _native.context(0)
    ctx.upload_table(table.matrix)
    ctx.upload_replay(rt, th, req, hr, stop)
    params = search_params(table, ds.arch, i=i, n=5, inst_reaction=0.7, literal_sign=False,
                           score_top_k=None, use_stop=True)
    ctx.launch_profile(params, _native.SeedWords(42, child_per_rep=True), reps)
    idx, prof, nst, status, err, stats = ctx.fetch(reps)
    key = f"{family}_stop"
    want = ragged(traj, key)
    names = {0: "budget", 1: "stopped", 2: "exhausted"}
    for r in range(reps):
        assert idx[r, :nst[r]].tolist() == want[r], f"{name}/{family} rep {r}"
        assert names[int(status[r])] == str(traj[key + "_status"][r])


@pytest.mark.parametrize("name", ["gemm", "conv"])
def test_b200_tree_training_matches_reference(name, tmp_path, caplog):
    """The slower tree trainings (gemm, conv), run on the GPU box's cores."""
    import filecmp
    from paper_2102_05297_b200 import formats, models
    caplog.set_level(logging.ERROR)
    ds = formats.load_dataset_dir(os.path.join(ROOT, "datasets", f"{name}-b200"))
    ms = models.train_model_set(ds, family="tree", seed=0)
    out = tmp_path / "m.json"
    models.save_model_set(ms, out)
    assert filecmp.cmp(out, os.path.join(GOLDEN, "models", f"b200_{name}_tree.json"),
                       shallow=False)
