"""Record golden fixtures from the reference implementation (run in the build
container, where /root/reference exists; the fixtures travel, the reference
does not).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.npz:
  expert.npz        analyze()/react() on the reference's 20-case bottleneck
                    fixture inputs + 3000 random counter maps
  ds_<name>.npz     replay arrays, exact + tree prediction tables
  traj_<name>.npz   run_profile_search / run_random_search trajectories
  scores.npz        score_configurations / normalize_scores vectors
  sim_gradient.npz  harness.simulate reports (profile + random)
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from countertune import bottlenecks, harness, models, search, synth  # noqa: E402
from countertune import space as rspace  # noqa: E402
from countertune.counters import ArchProfile as RArch  # noqa: E402

from paper_2102_05297_b200 import spaces as my_spaces  # noqa: E402

REQ = bottlenecks.REQUIRED_COUNTERS
DELTA_KEYS = [c for _, c in bottlenecks.MEMORY_TARGETS + bottlenecks.INSTRUCTION_TARGETS] + [
    "SM_E", "GLOBAL_THREADS"]


def expert():
    cases = json.load(open("/root/reference/pkg/tests/data/bottleneck_cases.json"))
    rows = []
    fixture_b, fixture_d = [], []
    for case in cases:
        rows.append((dict(case["counters"]), case["generation"], int(case["cores"]),
                     int(case["threads"]), float(case["inst_reaction"])))
        fixture_b.append([case["expected_b"][n] for n in bottlenecks.COMPONENT_NAMES])
        fixture_d.append([case["expected_delta"][k] for k in DELTA_KEYS])
    n_fixture = len(rows)
    rng = np.random.default_rng(7)
    for _ in range(3000):
        c = {}
        for k in REQ:
            c[k] = float(rng.choice([0.0, rng.uniform(0, 1e7), rng.uniform(0, 100)]))
        for k in ("DRAM_U", "TEX_U", "SHR_U"):
            c[k] = float(rng.uniform(0, 10)) if rng.random() < 0.9 else 0.0
        for k in ("L2_U", "SM_E", "WARP_E", "WARP_NP_E", "INST_ISSUE_U"):
            c[k] = float(rng.uniform(0, 100)) if rng.random() < 0.95 else 0.0
        rows.append((c, str(rng.choice(["pre_volta", "volta_plus"])), int(rng.integers(1, 30000)),
                     int(rng.integers(1, 300000)), float(rng.choice([0.7, 0.5, rng.uniform(0.05, 0.95)]))))
    counters, gen, cores, thr, reac, B, D, deg = [], [], [], [], [], [], [], []
    for c, g, cr, t, r in rows:
        b = bottlenecks.analyze(c, RArch("x", g, cr), t)
        d = bottlenecks.react(b, r)
        assert list(d) == DELTA_KEYS
        counters.append([c[k] for k in REQ])
        gen.append(0 if g == "pre_volta" else 1)
        cores.append(cr)
        thr.append(t)
        reac.append(r)
        B.append([getattr(b, n) for n in bottlenecks.COMPONENT_NAMES])
        D.append(list(d.values()))
        deg.append(b.degenerate_instructions)
    np.savez_compressed(os.path.join(HERE, "expert.npz"), counters=np.array(counters),
                        generation=np.array(gen, dtype=np.int32), cores=np.array(cores),
                        threads=np.array(thr), inst_reaction=np.array(reac), b=np.array(B),
                        delta=np.array(D), degenerate=np.array(deg),
                        n_fixture=np.int64(n_fixture), fixture_b=np.array(fixture_b),
                        fixture_delta=np.array(fixture_d))


def ref_dataset_from_mine(ds):
    """Build the reference's Dataset from one of our synthetic spaces."""
    params = tuple(rspace.TuningParameter(name=p.name, values=p.values, is_binary=p.is_binary)
                   for p in ds.space.parameters)
    confs = tuple(rspace.TuningConfiguration(assignment=tuple(map(float, row)), index=i)
                  for i, row in enumerate(ds.space.assignments))
    sp = rspace.TuningSpace(parameters=params, configurations=confs)
    recs = tuple(rspace.MeasurementRecord(
        config_index=i, runtime_us=float(ds.runtime_us[i]),
        global_threads=int(ds.global_threads[i]),
        counters=dict(zip(ds.counter_names, map(float, ds.counter_matrix[i]))))
        for i in range(len(sp)))
    return rspace.Dataset(space=sp, arch=RArch(ds.arch.name, ds.arch.generation, ds.arch.cores),
                          input_label=ds.input_label, records=recs)


def arrays_of(ds):
    n = len(ds.space)
    rt = np.array([ds.record_for(i).runtime_us for i in range(n)])
    th = np.array([ds.record_for(i).global_threads for i in range(n)], dtype=np.int64)
    names = ds.counter_names
    cm = np.array([[ds.record_for(i).counters[k] for k in names] for i in range(n)])
    req = np.array([[ds.record_for(i).counters[k] for k in REQ] for i in range(n)])
    assign = np.array([c.assignment for c in ds.space.configurations])
    return rt, th, cm, req, assign, names


def record_dataset(name, ds, tree=True, reps=64, i=40):
    rt, th, cm, req, assign, names = arrays_of(ds)
    exact = search.PredictionTable.from_model_set(models.ExactModelSet(ds), ds.space)
    out = dict(runtime=rt, threads=th, counter_matrix=cm, counter_names=np.array(names),
               required=req, assignments=assign,
               param_names=np.array(ds.space.parameter_names),
               param_binary=np.array([p.is_binary for p in ds.space.parameters]),
               generation=np.int32(0 if ds.arch.generation == "pre_volta" else 1),
               cores=np.int64(ds.arch.cores), arch_name=np.array(ds.arch.name),
               input_label=np.array(ds.input_label),
               exact_matrix=exact.matrix, exact_names=np.array(exact.counter_names))
    tables = {"exact": exact}
    if tree:
        ms = models.train_model_set(ds, family="tree", seed=0)
        t = search.PredictionTable.from_model_set(ms, ds.space)
        out["tree_matrix"] = t.matrix
        out["tree_names"] = np.array(t.counter_names)
        tables["tree"] = t
    np.savez_compressed(os.path.join(HERE, f"ds_{name}.npz"), **out)

    src = search.DatasetReplaySource(ds)
    well = rspace.well_performing_set(ds, 1.1)
    traj = {}
    for tname, table in tables.items():
        for stop_name, stop in (("stop", well), ("nostop", frozenset())):
            for lit in (False, True) if tname == "exact" and stop_name == "nostop" else (False,):
                seeds = np.random.SeedSequence(42).spawn(reps)
                idx, prof, off, status = [], [], [0], []
                for r in range(reps):
                    tr = search.run_profile_search(src, table, i=i, n=5, seed=seeds[r],
                                                   stop_indices=stop, literal_sign=lit)
                    idx.extend(s.config_index for s in tr.steps)
                    prof.extend(s.profiled for s in tr.steps)
                    off.append(len(idx))
                    status.append(tr.status)
                key = f"{tname}_{stop_name}" + ("_literal" if lit else "")
                traj[key + "_idx"] = np.array(idx, dtype=np.int32)
                traj[key + "_prof"] = np.array(prof, dtype=bool)
                traj[key + "_off"] = np.array(off, dtype=np.int64)
                traj[key + "_status"] = np.array(status)
    seeds = np.random.SeedSequence(42).spawn(reps)
    idx, off, status = [], [0], []
    for r in range(reps):
        tr = search.run_random_search(src, seed=seeds[r], stop_indices=well)
        idx.extend(s.config_index for s in tr.steps)
        off.append(len(idx))
        status.append(tr.status)
    traj["random_stop_idx"] = np.array(idx, dtype=np.int32)
    traj["random_stop_off"] = np.array(off, dtype=np.int64)
    traj["random_stop_status"] = np.array(status)
    traj["well"] = np.array(sorted(well), dtype=np.int64)
    traj["reps"] = np.int64(reps)
    traj["i"] = np.int64(i)
    np.savez_compressed(os.path.join(HERE, f"traj_{name}.npz"), **traj)


def record_scores(ds):
    """score_configurations + normalize_scores on random (profile, delta, explored)."""
    exact = search.PredictionTable.from_model_set(models.ExactModelSet(ds), ds.space)
    n = len(ds.space)
    rng = np.random.default_rng(11)
    out = {"cases": np.int64(60)}
    for k in range(60):
        prof = int(rng.integers(0, n))
        vals = rng.uniform(-1, 1, len(DELTA_KEYS))
        vals[rng.random(len(DELTA_KEYS)) < 0.3] = 0.0
        delta = dict(zip(DELTA_KEYS, map(float, vals)))
        explored = rng.random(n) < rng.choice([0.0, 0.01, 0.3])
        lit = bool(k % 7 == 3)
        top_k = int(rng.integers(1, 200)) if k % 5 == 4 else None
        sv = search.score_configurations(exact, ds.space.configurations[prof], delta, ds.space,
                                         explored, literal_sign=lit, score_top_k=top_k)
        nv = search.normalize_scores(sv)
        out[f"prof_{k}"] = np.int64(prof)
        out[f"delta_{k}"] = vals
        out[f"explored_{k}"] = explored
        out[f"literal_{k}"] = np.bool_(lit)
        out[f"topk_{k}"] = np.int64(-1 if top_k is None else top_k)
        out[f"raw_{k}"] = sv.raw
        out[f"scoreable_{k}"] = (sv.scoreable if sv.scoreable is not None
                                 else np.zeros(0, dtype=bool))
        out[f"norm_{k}"] = nv.norm
    np.savez_compressed(os.path.join(HERE, "scores.npz"), **out)


def record_simulate(ds):
    exact = models.ExactModelSet(ds)
    res = {}
    for searcher in ("profile", "random"):
        spec = harness.ExperimentSpec(dataset=ds, searcher=searcher,
                                      model=exact if searcher == "profile" else None,
                                      name=f"{searcher}-search", repetitions=50, seed=7,
                                      time_repetitions=20)
        rep = harness.simulate(spec)
        for f in ("steps", "step_curve_mean", "step_curve_std", "time_grid_seconds",
                  "time_curve_mean", "time_curve_std"):
            res[f"{searcher}_{f}"] = getattr(rep, f)
        res[f"{searcher}_censored"] = np.int64(rep.censored)
        res[f"{searcher}_mean_time_seconds"] = np.float64(rep.mean_time_seconds)
        res[f"{searcher}_outer"] = np.int64(rep.outer_iterations)
    np.savez_compressed(os.path.join(HERE, "sim_gradient.npz"), **res)


def main():
    expert()
    grad = synth.build_dataset(synth.GENERATOR_PRESETS["gradient"])
    calib = synth.build_dataset(synth.GENERATOR_PRESETS["calibration"])
    record_dataset("gradient", grad, tree=True)
    record_dataset("calibration", calib, tree=False)
    record_dataset("transpose", ref_dataset_from_mine(my_spaces.transpose()), tree=False,
                   reps=32)
    record_dataset("coulomb", ref_dataset_from_mine(my_spaces.coulomb()), tree=True, reps=32)
    record_scores(grad)
    record_simulate(grad)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
