"""GPU parity: libct_b200.so against fixtures recorded from the reference.

Trajectories, raw scores and reports must be bit-identical; weights are the
one place the device is allowed to differ, by at most 1 ulp (correctly
rounded x**8 vs numpy's pow), and every draw must then still pick the same
configuration (certified selection).
"""

import numpy as np
import pytest

from conftest import dataset_from_golden, golden, ragged

pytestmark = pytest.mark.gpu

TRAJ_SETS = ["gradient", "calibration", "transpose", "coulomb",
             "b200_transpose", "b200_coulomb", "b200_conv", "b200_gemm", "b200_nbody"]   # B200 sweeps


def _table(name, model):
    from paper_2102_05297_b200.search import PredictionTable
    d = golden(f"ds_{name}.npz")
    ds = dataset_from_golden(name)
    return ds, PredictionTable(ds.space, [str(x) for x in d[f"{model}_names"]],
                               d[f"{model}_matrix"])


def _keys(traj):
    return sorted({k[:-4] for k in traj.files if k.endswith("_idx") and not k.startswith("random")})


@pytest.mark.parametrize("name", TRAJ_SETS)
def test_batched_profile_trajectories_match_reference(name):
    _check_trajectories(name)


# the alternative kernel builds selected by environment at launch time:
# warp-specialised two-repetition kernel, in-row prefixes stored by the
# weight pass or scanned per draw (the default picks by row count), one-warp
# and eight-warp CTA sizes, weights in a global slice instead of shared memory
@pytest.mark.parametrize("env", [{"CT_SEARCH_WS": "4"}, {"CT_SEARCH_WS": "6"},
                                 {"CT_SEARCH_PRE": "0"}, {"CT_SEARCH_PRE": "1"},
                                 {"CT_SEARCH_NT": "32"}, {"CT_SEARCH_NT": "256"},
                                 {"CT_SEARCH_SMEM": "0"}],
                         ids=["ws4", "ws6", "pre0", "pre1", "nt32", "nt256", "smem0"])
@pytest.mark.parametrize("name", ["gradient", "b200_transpose"])
def test_kernel_variants_match_reference(name, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _check_trajectories(name)


# the tiled large-space path (ct_tiled.cuh: grid-wide Eq. 16 / Eq. 17 kernels
# per outer iteration, one warp per repetition for the draws), forced on every
# trajectory set (tiles of 4096 configurations: one partial tile here)
@pytest.mark.parametrize("name", TRAJ_SETS)
def test_tiled_path_matches_reference(name, monkeypatch):
    monkeypatch.setenv("CT_SEARCH_TILED", "1")
    _check_trajectories(name)


def test_tiled_path_small_batches_match_reference(monkeypatch):
    """A scratch budget of 1 MB forces repetition batches of a few each."""
    monkeypatch.setenv("CT_SEARCH_TILED", "1")
    monkeypatch.setenv("CT_TILED_BUDGET_MB", "1")
    _check_trajectories("b200_gemm")


def _check_trajectories(name):
    from paper_2102_05297_b200 import _native
    from paper_2102_05297_b200.search import search_params
    from paper_2102_05297_b200.space import replay_arrays
    traj = golden(f"traj_{name}.npz")
    reps, i = int(traj["reps"]), int(traj["i"])
    well = traj["well"]
    for key in _keys(traj):
        model, stop_name = key.split("_")[0], key.split("_")[1]
        literal = key.endswith("_literal")
        ds, table = _table(name, model)
        rt, th, req, hr = replay_arrays(ds)
        stop = np.zeros(len(ds.space), dtype=np.uint8)
        stop[well] = 1
        ctx = _native.context(0)
        ctx.upload_table(table.matrix)
        ctx.upload_replay(rt, th, req, hr, stop)
        params = search_params(table, ds.arch, i=i, n=5, inst_reaction=0.7,
                               literal_sign=literal, score_top_k=None,
                               use_stop=(stop_name == "stop"))
        ctx.launch_profile(params, _native.SeedWords(42, child_per_rep=True), reps)
        idx, prof, nst, status, err, stats = ctx.fetch(reps)
        want = ragged(traj, key)
        want_prof = [traj[key + "_prof"][traj[key + "_off"][r]:traj[key + "_off"][r + 1]].tolist()
                     for r in range(reps)]
        names = {0: "budget", 1: "stopped", 2: "exhausted"}
        for r in range(reps):
            got = idx[r, :nst[r]].tolist()
            assert got == want[r], f"{name}/{key} rep {r}: first divergence at " \
                f"{next((k for k, (a, b) in enumerate(zip(got, want[r])) if a != b), min(len(got), len(want[r])))}"
            assert prof[r, :nst[r]].astype(bool).tolist() == want_prof[r]
            assert names[int(status[r])] == str(traj[key + "_status"][r])
        assert stats.configs_scored > 0


@pytest.mark.parametrize("name", TRAJ_SETS)
def test_random_search_matches_reference(name):
    from paper_2102_05297_b200 import _native
    from paper_2102_05297_b200.space import replay_arrays
    traj = golden(f"traj_{name}.npz")
    reps = int(traj["reps"])
    ds = dataset_from_golden(name)
    rt, th, req, hr = replay_arrays(ds)
    stop = np.zeros(len(ds.space), dtype=np.uint8)
    stop[traj["well"]] = 1
    ctx = _native.context(0)
    ctx.upload_replay(rt, th, req, hr, stop)
    ctx.launch_random(_native.SeedWords(42, child_per_rep=True), reps, None, use_stop=True)
    idx, _, nst, status, _, _ = ctx.fetch(reps)
    want = ragged(traj, "random_stop")
    for r in range(reps):
        assert idx[r, :nst[r]].tolist() == want[r]


def test_score_raw_bit_exact_and_norm_within_one_ulp():
    from paper_2102_05297_b200 import normalize_scores, score_configurations
    from paper_2102_05297_b200.counters import DELTA_KEYS
    s = golden("scores.npz")
    ds, table = _table("gradient", "exact")
    for k in range(int(s["cases"])):
        delta = dict(zip(DELTA_KEYS, map(float, s[f"delta_{k}"])))
        top_k = int(s[f"topk_{k}"])
        sv = score_configurations(table, ds.space.configurations[int(s[f"prof_{k}"])], delta,
                                  ds.space, s[f"explored_{k}"].astype(bool),
                                  literal_sign=bool(s[f"literal_{k}"]),
                                  score_top_k=None if top_k < 0 else top_k)
        np.testing.assert_array_equal(sv.raw.view(np.uint64), s[f"raw_{k}"].view(np.uint64))
        if s[f"scoreable_{k}"].size:
            np.testing.assert_array_equal(sv.scoreable, s[f"scoreable_{k}"])
        else:
            assert sv.scoreable is None
        nv = normalize_scores(sv)
        ulps = np.abs(nv.norm.view(np.int64) - s[f"norm_{k}"].view(np.int64))
        assert ulps.max() <= 1, f"case {k}: {ulps.max()} ulp"


def test_weighted_select_statistics_and_errors():
    """search tests: test_weighted_select_matches_weights / _requires_weight."""
    from paper_2102_05297_b200 import ScoreVector, SpaceExhaustedError, weighted_select
    weights = np.array([4.0, 0.0, 1.0, 3.0])
    sv = ScoreVector(raw=np.zeros(4), explored=np.zeros(4, dtype=bool), norm=weights.copy())
    rng = np.random.default_rng(0)
    counts = np.zeros(4)
    draws = 3000
    for _ in range(draws):
        counts[weighted_select(sv, rng)] += 1
    assert counts[1] == 0
    probs = weights / weights.sum()
    for i in (0, 2, 3):
        sigma = np.sqrt(draws * probs[i] * (1 - probs[i]))
        assert abs(counts[i] - draws * probs[i]) < 4 * sigma
    with pytest.raises(SpaceExhaustedError):
        weighted_select(ScoreVector(raw=np.zeros(3), explored=np.zeros(3, dtype=bool),
                                    norm=np.zeros(3)), np.random.default_rng(0))
    with pytest.raises(ValueError):
        weighted_select(ScoreVector(raw=np.zeros(3), explored=np.zeros(3, dtype=bool)),
                        np.random.default_rng(0))


def test_weighted_select_same_index_as_numpy():
    """Random weight vectors in Eq. 17's range: device == np.cumsum/searchsorted."""
    from paper_2102_05297_b200 import _native
    ctx = _native.context(0)
    rng = np.random.default_rng(5)
    for trial in range(200):
        n = int(rng.integers(1, 5000))
        w = np.where(rng.random(n) < 0.5, rng.uniform(1.0, 256.0, n), rng.uniform(1e-4, 1.0, n))
        w[rng.random(n) < 0.1] = 0.0
        if w.sum() == 0:
            w[0] = 1.0
        u = rng.random()
        c = np.cumsum(w)
        want = int(np.searchsorted(c, u * c[-1], side="right"))
        got, _ = ctx.select(w, u)
        assert got == want


def test_simulate_report_byte_identical():
    from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec, simulate
    sim = golden("sim_gradient.npz")
    ds = dataset_from_golden("gradient")
    for searcher in ("profile", "random"):
        spec = ExperimentSpec(dataset=ds, searcher=searcher,
                              model=ExactModelSet(ds) if searcher == "profile" else None,
                              name=f"{searcher}-search", repetitions=50, seed=7,
                              time_repetitions=20)
        rep = simulate(spec)
        for f in ("steps", "step_curve_mean", "step_curve_std", "time_grid_seconds",
                  "time_curve_mean", "time_curve_std"):
            np.testing.assert_array_equal(getattr(rep, f), sim[f"{searcher}_{f}"], err_msg=f)
        assert rep.censored == int(sim[f"{searcher}_censored"])
        assert rep.mean_time_seconds == float(sim[f"{searcher}_mean_time_seconds"])


def test_run_profile_search_single_api_matches_reference():
    from paper_2102_05297_b200 import DatasetReplaySource, run_profile_search
    traj = golden("traj_gradient.npz")
    ds, table = _table("gradient", "tree")
    seeds = np.random.SeedSequence(42).spawn(int(traj["reps"]))
    want = ragged(traj, "tree_stop")
    stop = set(traj["well"].tolist())
    src = DatasetReplaySource(ds)
    for r in range(8):
        tr = run_profile_search(src, table, i=int(traj["i"]), n=5, seed=seeds[r],
                                stop_indices=stop)
        assert [s.config_index for s in tr.steps] == want[r]


def test_host_driven_profile_search_matches_reference():
    """A non-replay source: host measures, device scores/normalises/draws."""
    from paper_2102_05297_b200 import DatasetReplaySource, run_profile_search

    class LiveLike(DatasetReplaySource):
        pass  # a different type: forces the host-driven path

    traj = golden("traj_gradient.npz")
    ds, table = _table("gradient", "exact")
    seeds = np.random.SeedSequence(42).spawn(int(traj["reps"]))
    want = ragged(traj, "exact_stop")
    stop = set(traj["well"].tolist())
    src = LiveLike(ds)
    for r in range(4):
        tr = run_profile_search(src, table, i=int(traj["i"]), n=5, seed=seeds[r],
                                stop_indices=stop)
        assert [s.config_index for s in tr.steps] == want[r]


def test_host_driven_generator_seed_advances_like_reference():
    """A caller-owned numpy Generator as the seed: the searcher draws a whole
    iteration's candidates before measuring them, but on an early stop the
    caller's Generator must end where the reference leaves it (one
    integers() plus one random() per recorded draw)."""
    from paper_2102_05297_b200 import DatasetReplaySource, run_profile_search

    class LiveLike(DatasetReplaySource):
        pass

    traj = golden("traj_gradient.npz")
    ds, table = _table("gradient", "exact")
    seeds = np.random.SeedSequence(42).spawn(int(traj["reps"]))
    want = ragged(traj, "exact_stop")
    stop = set(traj["well"].tolist())
    for r in range(4):
        g = np.random.default_rng(seeds[r])
        tr = run_profile_search(LiveLike(ds), table, i=int(traj["i"]), n=5, seed=g,
                                stop_indices=stop)
        assert [s.config_index for s in tr.steps] == want[r]
        n = len(want[r])
        drawn = n - ((n - 1) // 6 + 1)
        ref = np.random.default_rng(seeds[r])
        ref.integers(0, len(ds.space))
        ref.random(drawn)
        assert g.bit_generator.state == ref.bit_generator.state


def test_large_space_properties():
    """GEMM-full (205,216 configurations): global-scratch path; cadence, no
    redraw, later-ties-win argmin, and identical results for any rep split."""
    from paper_2102_05297_b200 import ExactModelSet, harness, spaces
    ds = spaces.gemm_full()
    spec = harness.ExperimentSpec(dataset=ds, searcher="profile", model=ExactModelSet(ds),
                                  repetitions=6, outer_iterations=6, seed=1, slack=1.0)
    res, rt = harness.run_batch(spec)
    for r in range(6):
        n = int(res.n_steps[r])
        idx = res.step_index[r, :n]
        prof = res.step_profiled[r, :n].astype(bool)
        for k in range(n):
            assert prof[k] == (k % 6 == 0)
        drawn = idx[~prof]
        assert len(set(drawn.tolist())) == drawn.size
        for o in range(1, n // 6):
            batch = idx[(o - 1) * 6 + 1: o * 6]
            times = rt[batch]
            winner = max(j for j, t in enumerate(times) if t == times.min())
            assert idx[o * 6] == batch[winner]
    # rep_offset sharding reproduces the same rows
    from paper_2102_05297_b200 import _native
    ctx = _native.context(0)
    params, _ = harness.prepare_device(ctx, spec)
    harness.launch(ctx, spec, params, 3, 3)
    idx2, _, nst2, _, _, _ = ctx.fetch(3)
    for r in range(3):
        assert idx2[r, :nst2[r]].tolist() == res.step_index[3 + r, :res.n_steps[3 + r]].tolist()


@pytest.mark.parametrize("tiled,slack,force", [("0", "1", "0"), ("0", "4", "0"), ("1", "1", "0"),
                                               ("1", "4", "0"), ("0", "1", "1"), ("1", "1", "1")],
                         ids=["persistent", "persistent-slack4", "tiled", "tiled-slack4",
                              "persistent-all-sequential", "tiled-all-sequential"])
def test_gemm_full_trajectories_match_reference_with_uncertified_draws(tiled, slack, force,
                                                                        monkeypatch):
    """N = 205,216 (GEMM-full): 256 repetitions x 40 iterations x 5 draws
    against the reference's own trajectories (make_gemmfull_golden.py).  At
    this size the certificate rejects some draws, which the device re-decides
    with the sequential cumsum: the run must still match the reference
    everywhere -- with the per-repetition persistent kernel and with the
    tiled large-space path, under the proven half-width and under 4x it
    (CT_SEARCH_CERT_SLACK, about round 1's (8N + 128) u T), which must leave
    draws to the re-decision."""
    monkeypatch.setenv("CT_SEARCH_TILED", tiled)
    monkeypatch.setenv("CT_SEARCH_CERT_SLACK", slack)
    monkeypatch.setenv("CT_SEARCH_FORCE_SEQUENTIAL", force)
    from paper_2102_05297_b200 import ExactModelSet, _native, spaces
    from paper_2102_05297_b200.search import PredictionTable, search_params
    from paper_2102_05297_b200.space import replay_arrays
    traj = golden("traj_gemm_full.npz")
    reps, i = int(traj["reps"]), int(traj["i"])
    ds = spaces.gemm_full()
    table = PredictionTable.from_model_set(ExactModelSet(ds), ds.space)
    rt, th, req, hr = replay_arrays(ds)
    ctx = _native.context(0)
    ctx.upload_table(table.matrix)
    ctx.upload_replay(rt, th, req, hr, np.zeros(len(ds.space), dtype=np.uint8))
    params = search_params(table, ds.arch, i=i, n=5, inst_reaction=0.7, literal_sign=False,
                           score_top_k=None, use_stop=False)
    ctx.launch_profile(params, _native.SeedWords(42, child_per_rep=True), reps)
    idx, prof, nst, status, err, stats = ctx.fetch(reps)
    want = ragged(traj, "exact_nostop")
    for r in range(reps):
        got = idx[r, :nst[r]].tolist()
        assert got == want[r], f"rep {r}: first divergence at " \
            f"{next((k for k, (a, b) in enumerate(zip(got, want[r])) if a != b), min(len(got), len(want[r])))}"
    print(f"gemm_full: {stats.draws} draws, {stats.uncertified} uncertified")
    if slack != "1":
        assert stats.uncertified > 0
    if force == "1":
        assert stats.uncertified == stats.draws > 0


def test_inline_division_is_ddiv_rn():
    """dvd_fast (ct_hd.cuh) == __ddiv_rn bit for bit on 2^28 operand pairs."""
    from paper_2102_05297_b200 import _native
    ctx = _native.context(0)
    assert ctx.check_division(1 << 28, seed=12345) == 0


@pytest.mark.parametrize("name", ["gradient", "transpose"])
def test_device_aggregation_matches_host_aggregate(name):
    """simulate() sums on the device; aggregate() on fetched trajectories is
    the reference's harness.py:187-244 arithmetic.  Both must agree bit for bit,
    also with the repetitions split over two contexts (chained partial sums)."""
    from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec, harness
    ds = dataset_from_golden(name)
    for searcher, tr in (("profile", None), ("profile", 7), ("random", 13)):
        spec = ExperimentSpec(dataset=ds, searcher=searcher,
                              model=ExactModelSet(ds) if searcher == "profile" else None,
                              name="x", repetitions=40, seed=3, time_repetitions=tr,
                              profiling_overhead=2.5)
        want = harness.simulate_host_aggregate(spec)
        for devices in ([0], [0, 0]):
            got = harness.simulate(spec, devices=devices)
            for f in ("steps", "step_curve_mean", "step_curve_std", "time_grid_seconds",
                      "time_curve_mean", "time_curve_std"):
                np.testing.assert_array_equal(getattr(got, f), getattr(want, f), err_msg=f)
            assert got.censored == want.censored
            assert got.mean_time_seconds == want.mean_time_seconds


def test_sequential_redecision_path_matches_reference(monkeypatch):
    """Every draw forced through the uncertified path (sequential float
    cumsum over the weights recovered from the exact prefixes): the
    trajectories must still be the reference's."""
    from paper_2102_05297_b200 import _native
    from paper_2102_05297_b200.search import search_params
    from paper_2102_05297_b200.space import replay_arrays
    monkeypatch.setenv("CT_SEARCH_FORCE_SEQUENTIAL", "1")
    traj = golden("traj_gradient.npz")
    reps, i = 8, int(traj["i"])
    ds, table = _table("gradient", "exact")
    rt, th, req, hr = replay_arrays(ds)
    stop = np.zeros(len(ds.space), dtype=np.uint8)
    stop[traj["well"]] = 1
    ctx = _native.context(0)
    ctx.upload_table(table.matrix)
    ctx.upload_replay(rt, th, req, hr, stop)
    params = search_params(table, ds.arch, i=i, n=5, inst_reaction=0.7, literal_sign=False,
                           score_top_k=None, use_stop=True)
    ctx.launch_profile(params, _native.SeedWords(42, child_per_rep=True), reps)
    idx, _, nst, _, _, stats = ctx.fetch(reps)
    want = ragged(traj, "exact_stop")
    for r in range(reps):
        assert idx[r, :nst[r]].tolist() == want[r]
    assert stats.uncertified == stats.draws > 0


@pytest.mark.parametrize("name", TRAJ_SETS)
def test_every_draw_sequential_matches_reference(name, monkeypatch):
    """Every draw of every trajectory set forced through the re-decision
    (the warp's binade-exact emulation of np.cumsum's sequential adds)."""
    monkeypatch.setenv("CT_SEARCH_FORCE_SEQUENTIAL", "1")
    _check_trajectories(name)


@pytest.mark.parametrize("name,family", [("gradient", "tree"), ("coulomb", "tree"),
                                         ("gradient", "regression"),
                                         ("coulomb", "regression"), ("conv", "regression")])
def test_gpu_model_inference_matches_reference_table(name, family):
    """ct_model_predict == the reference's PredictionTable.from_model_set."""
    import os
    from conftest import GOLDEN
    from paper_2102_05297_b200 import models, spaces
    from paper_2102_05297_b200.search import PredictionTable
    ms = models.load_model_set(os.path.join(GOLDEN, "models", f"{name}_{family}.json"))
    want = np.load(os.path.join(GOLDEN, "models", "tables.npz"))[f"{name}_{family}_matrix"]
    ds = dataset_from_golden("gradient") if name == "gradient" else spaces.SPACES[name]()
    table = PredictionTable.from_model_set(ms, ds.space)
    np.testing.assert_array_equal(table.matrix.view(np.uint64), want.view(np.uint64))


def test_device_expert_system_bit_exact():
    """The search kernel's warp expert system (analyze_component_warp, run by
    ct_analyze_react) against the 3,020 reference-recorded cases, bit for bit."""
    from paper_2102_05297_b200 import _native
    e = golden("expert.npz")
    ctx = _native.context(0)
    for k in range(e["counters"].shape[0]):
        b, d, deg = ctx.analyze_react(e["counters"][k], int(e["generation"][k]),
                                      int(e["cores"][k]), int(e["threads"][k]),
                                      float(e["inst_reaction"][k]))
        np.testing.assert_array_equal(b, e["b"][k], err_msg=f"case {k}")
        np.testing.assert_array_equal(d, e["delta"][k], err_msg=f"case {k}")
        assert deg == bool(e["degenerate"][k])


def test_reference_acceptance_criteria_3_and_4():
    """The reference's own acceptance gate (pkg/tests/test_acceptance.py:104-142)
    on the GPU harness.  Trajectories are bit-exact, so the numbers are the
    ones the reference itself computes in this container,
    to the last bit: C3 random-baseline calibration 48.3443 mean steps
    (N=1000, k=20, 10,000 repetitions); C4 exact-model improvement
    13.824442820606503x, literal sign 0.06455974815939666x (values from
    countertune.harness.simulate / pair_with_baseline with the same specs,
    recorded with PYTHONPATH=/root/reference/pkg/src)."""
    from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec, pair_with_baseline, simulate
    calib = dataset_from_golden("calibration")
    rep = simulate(ExperimentSpec(dataset=calib, searcher="random", name="rand",
                                  repetitions=10_000, seed=42, time_repetitions=10))
    expected = 1001.0 / 21.0
    assert abs(rep.mean_steps - expected) / expected <= 0.05
    assert rep.mean_steps == 48.3443
    grad = dataset_from_golden("gradient")
    exact = ExactModelSet(grad)
    prof = simulate(ExperimentSpec(dataset=grad, searcher="profile", model=exact, name="profile",
                                   repetitions=1000, seed=42, time_repetitions=10))
    rand = simulate(ExperimentSpec(dataset=grad, searcher="random", name="random",
                                   repetitions=1000, seed=42, time_repetitions=10))
    improvement = pair_with_baseline(prof, rand).improvement
    literal = simulate(ExperimentSpec(dataset=grad, searcher="profile", model=exact,
                                      name="literal", repetitions=1000, seed=42,
                                      literal_sign=True, time_repetitions=10))
    degraded = pair_with_baseline(literal, rand).improvement
    assert improvement >= 2.0 and degraded < 1.2
    assert improvement == 13.824442820606503
    assert degraded == 0.06455974815939666


def test_reference_acceptance_criterion_6_portability():
    """C6 (pkg/tests/test_acceptance.py:178-196): a tree model trained on
    gradient (seed 0) steers the 3x-rescaled gradient3x space; the GPU
    harness reproduces the reference's improvement to the last bit
    (tests/golden/make_c6_golden.py)."""
    from paper_2102_05297_b200 import ExperimentSpec, pair_with_baseline, simulate
    from paper_2102_05297_b200.models import train_model_set
    g = golden("ds_gradient3x.npz")
    train_ds = dataset_from_golden("gradient")
    target_ds = dataset_from_golden("gradient3x")
    ms = train_model_set(train_ds, "tree", 0)
    prof = simulate(ExperimentSpec(dataset=target_ds, searcher="profile", model=ms, name="ported",
                                   repetitions=1000, seed=7, time_repetitions=10))
    rand = simulate(ExperimentSpec(dataset=target_ds, searcher="random", name="random",
                                   repetitions=1000, seed=7, time_repetitions=10))
    improvement = pair_with_baseline(prof, rand).improvement
    assert improvement > 1.5
    assert prof.mean_steps == float(g["c6_prof_mean"])
    assert rand.mean_steps == float(g["c6_rand_mean"])
    assert improvement == float(g["c6_improvement"])


@pytest.mark.parametrize("tiled", ["0", "1"], ids=["persistent", "tiled"])
def test_stress_space_global_row_index_matches_oracle(tiled, monkeypatch):
    """N = 1,048,576 (BASELINE.md stress size): the row index no longer fits
    shared memory, so row totals, explored bits and weights live in global
    scratch (HG kernel) and the draw walks long row chunks with the whole
    warp.  Trajectories against the oracle (numpy restatement of the
    reference, pinned by the golden tests) for a few repetitions; with the
    persistent kernel and with the tiled large-space path."""
    monkeypatch.setenv("CT_SEARCH_TILED", tiled)
    import countertune_oracle as oracle
    from paper_2102_05297_b200 import ExactModelSet, harness, spaces
    from paper_2102_05297_b200.space import replay_arrays
    ds = spaces.stress(1 << 20)
    spec = harness.ExperimentSpec(dataset=ds, searcher="profile", model=ExactModelSet(ds),
                                  repetitions=3, outer_iterations=5, seed=9,
                                  stop_at_well_performing=False)
    res, rt = harness.run_batch(spec)
    ms = ExactModelSet(ds)
    matrix = ms.prediction_matrix(ds.space)
    column = {c: j for j, c in enumerate(ms.counters)}
    _, th, req, hr = replay_arrays(ds)
    seeds = np.random.SeedSequence(9).spawn(3)
    for r in range(3):
        steps, status, _ = oracle.profile_search(matrix, column, rt, th, req, hr, pre_volta=False,
                                                 cores=ds.arch.cores, i=5, n=5, seed=seeds[r],
                                                 stop=None)
        assert res.step_index[r, :res.n_steps[r]].tolist() == [s[0] for s in steps]
