"""score_top_k through the batched device search (search.py:133-140,
harness.py:155-158) against the reference's own trajectories and report
(tests/golden/make_topk_golden.py).

K below n empties the pool mid-iteration (status exhausted), K = 7 / 40 / 300
exercise the radix select with and without ties at the K-th distance (the
gradient space's parameter grid has many equidistant configurations)."""

import numpy as np
import pytest

from conftest import dataset_from_golden, golden, ragged

pytestmark = pytest.mark.gpu


def _exact_table(name):
    from paper_2102_05297_b200.search import PredictionTable
    d = golden(f"ds_{name}.npz")
    ds = dataset_from_golden(name)
    return ds, PredictionTable(ds.space, [str(x) for x in d["exact_names"]], d["exact_matrix"])


@pytest.mark.parametrize("name", ["gradient", "b200_transpose"])
def test_topk_trajectories_match_reference(name):
    from paper_2102_05297_b200 import _native
    from paper_2102_05297_b200.search import search_params
    from paper_2102_05297_b200.space import assignments_of, replay_arrays
    traj = golden(f"traj_topk_{name}.npz")
    reps, i = int(traj["reps"]), int(traj["i"])
    ds, table = _exact_table(name)
    rt, th, req, hr = replay_arrays(ds)
    stop = np.zeros(len(ds.space), dtype=np.uint8)
    stop[traj["well"]] = 1
    ctx = _native.context(0)
    ctx.upload_table(table.matrix)
    ctx.upload_replay(rt, th, req, hr, stop)
    ctx.upload_space(assignments_of(ds.space))
    names = {0: "budget", 1: "stopped", 2: "exhausted"}
    for K in traj["topk"].tolist():
        key = f"k{K}"
        params = search_params(table, ds.arch, i=i, n=5, inst_reaction=0.7, literal_sign=False,
                               score_top_k=K, use_stop=True)
        ctx.launch_profile(params, _native.SeedWords(42, child_per_rep=True), reps)
        idx, prof, nst, status, err, stats = ctx.fetch(reps)
        want = ragged(traj, key)
        off = traj[key + "_off"]
        for r in range(reps):
            assert idx[r, :nst[r]].tolist() == want[r], f"{name} K={K} rep {r}"
            assert prof[r, :nst[r]].astype(bool).tolist() == \
                traj[key + "_prof"][off[r]:off[r + 1]].tolist()
            assert names[int(status[r])] == str(traj[key + "_status"][r])


def test_topk_run_profile_search_replay_path():
    """run_profile_search(score_top_k=K) on a replay source: one-repetition
    device launch, same trajectories."""
    from paper_2102_05297_b200 import DatasetReplaySource, run_profile_search
    traj = golden("traj_topk_gradient.npz")
    ds, table = _exact_table("gradient")
    seeds = np.random.SeedSequence(42).spawn(int(traj["reps"]))
    stop = set(traj["well"].tolist())
    for K in (3, 40):
        want = ragged(traj, f"k{K}")
        for r in range(6):
            tr = run_profile_search(DatasetReplaySource(ds), table, i=int(traj["i"]), n=5,
                                    seed=seeds[r], stop_indices=stop, score_top_k=K)
            assert [s.config_index for s in tr.steps] == want[r]


def test_simulate_with_score_top_k_matches_reference():
    from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec, simulate
    gold = golden("sim_topk.npz")
    ds = dataset_from_golden("gradient")
    rep = simulate(ExperimentSpec(dataset=ds, searcher="profile", model=ExactModelSet(ds),
                                  name="profile-topk", repetitions=50, seed=7,
                                  time_repetitions=20, score_top_k=40))
    for f in ("steps", "step_curve_mean", "step_curve_std", "time_grid_seconds",
              "time_curve_mean", "time_curve_std"):
        np.testing.assert_array_equal(getattr(rep, f), gold[f], err_msg=f)
    assert rep.censored == int(gold["censored"])
    assert rep.mean_time_seconds == float(gold["mean_time_seconds"])
    # configs scored counts the K-configuration pools
    assert rep.configs_scored <= 40 * sum(int(s) // 6 + 1 for s in rep.steps)


def test_score_top_k_zero_raises_like_reference():
    """K = 0 leaves normalize_scores an empty pool: SpaceExhaustedError."""
    from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec, simulate
    from paper_2102_05297_b200.errors import SpaceExhaustedError
    ds = dataset_from_golden("gradient")
    with pytest.raises(SpaceExhaustedError, match="no unexplored configurations"):
        simulate(ExperimentSpec(dataset=ds, searcher="profile", model=ExactModelSet(ds),
                                repetitions=8, seed=7, score_top_k=0,
                                stop_at_well_performing=False))
