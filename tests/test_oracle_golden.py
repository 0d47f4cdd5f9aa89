"""The CPU oracle (oracle/countertune_oracle.py) pinned to reference fixtures.

The fixtures were recorded from the reference itself (tests/golden/
make_golden.py); the expert-system cases also include the reference's own
hand-evaluated fixture (pkg/tests/data/bottleneck_cases.json) at its 1e-9
tolerance.
"""

import numpy as np
import pytest

import countertune_oracle as oracle
from conftest import golden, ragged


def test_expert_system_bit_exact():
    e = golden("expert.npz")
    for k in range(e["counters"].shape[0]):
        b, deg = oracle.analyze(e["counters"][k], int(e["generation"][k]) == 0,
                                int(e["cores"][k]), int(e["threads"][k]))
        d = oracle.react(b, float(e["inst_reaction"][k]))
        np.testing.assert_array_equal(np.array(b), e["b"][k])
        np.testing.assert_array_equal(np.array(d), e["delta"][k])
        assert deg == bool(e["degenerate"][k])


def test_expert_system_hand_evaluated_fixture():
    e = golden("expert.npz")
    for k in range(int(e["n_fixture"])):
        b, _ = oracle.analyze(e["counters"][k], int(e["generation"][k]) == 0,
                              int(e["cores"][k]), int(e["threads"][k]))
        d = oracle.react(b, float(e["inst_reaction"][k]))
        np.testing.assert_allclose(b, e["fixture_b"][k], atol=1e-9, rtol=0)
        np.testing.assert_allclose(d, e["fixture_delta"][k], atol=1e-9, rtol=0)


def test_scores_and_weights_match_reference():
    s = golden("scores.npz")
    d = golden("ds_gradient.npz")
    matrix = d["exact_matrix"]
    column = {str(n): j for j, n in enumerate(d["exact_names"])}
    for k in range(int(s["cases"])):
        deltas = list(zip(oracle.DELTA_KEYS, map(float, s[f"delta_{k}"])))
        top_k = int(s[f"topk_{k}"])
        explored = s[f"explored_{k}"].astype(bool)
        raw, scoreable = oracle.score(matrix, column, int(s[f"prof_{k}"]), deltas, explored,
                                      bool(s[f"literal_{k}"]), None if top_k < 0 else top_k,
                                      d["assignments"])
        np.testing.assert_array_equal(raw.view(np.uint64), s[f"raw_{k}"].view(np.uint64))
        pool = ~explored if scoreable is None else (scoreable & ~explored)
        w = oracle.normalize(raw, pool)
        # numpy's pow may be SVML or glibc depending on the host: <= 1 ulp
        assert np.abs(w.view(np.int64) - s[f"norm_{k}"].view(np.int64)).max() <= 1


@pytest.mark.parametrize("name", ["gradient", "calibration", "transpose", "coulomb",
                                  "b200_transpose", "b200_coulomb", "b200_conv", "b200_gemm",
                                  "b200_nbody"])
def test_trajectories_match_reference(name):
    d = golden(f"ds_{name}.npz")
    traj = golden(f"traj_{name}.npz")
    reps, i = int(traj["reps"]), int(traj["i"])
    stop = np.zeros(d["runtime"].size, dtype=bool)
    stop[traj["well"]] = True
    hr = np.ones(d["runtime"].size, dtype=bool)
    seeds = np.random.SeedSequence(42).spawn(reps)
    keys = sorted({k[:-4] for k in traj.files if k.endswith("_idx") and not k.startswith("random")})
    for key in keys:
        model = key.split("_")[0]
        matrix = d[f"{model}_matrix"]
        column = {str(n): j for j, n in enumerate(d[f"{model}_names"])}
        want = ragged(traj, key)
        for r in range(min(reps, 16)):
            steps, status, _ = oracle.profile_search(
                matrix, column, d["runtime"], d["threads"], d["required"], hr,
                pre_volta=int(d["generation"]) == 0, cores=int(d["cores"]), i=i, n=5,
                seed=seeds[r], stop=stop if "_stop" in key else None,
                literal_sign=key.endswith("_literal"))
            assert [s[0] for s in steps] == want[r], (key, r)
            assert status == str(traj[key + "_status"][r])
    want = ragged(traj, "random_stop")
    for r in range(min(reps, 16)):
        got, _ = oracle.random_search(d["runtime"].size, seed=seeds[r], stop=stop)
        assert got == want[r]
