"""Record the reference's acceptance criterion C6 (model portability,
pkg/tests/test_acceptance.py:178-196) for the GPU test: the gradient3x
dataset arrays and the improvement the reference computes.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c6_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from countertune import harness, models, synth  # noqa: E402


def main():
    train_ds = synth.build_dataset(synth.GENERATOR_PRESETS["gradient"])
    target_ds = synth.build_dataset(synth.GENERATOR_PRESETS["gradient3x"])
    ms = models.train_model_set(train_ds, seed=0)
    prof = harness.simulate(harness.ExperimentSpec(dataset=target_ds, searcher="profile", model=ms,
                                                   name="ported", repetitions=1000, seed=7,
                                                   time_repetitions=10))
    rand = harness.simulate(harness.ExperimentSpec(dataset=target_ds, searcher="random",
                                                   name="random", repetitions=1000, seed=7,
                                                   time_repetitions=10))
    improvement = harness.pair_with_baseline(prof, rand).improvement
    ds = target_ds
    n = len(ds.space)
    names = tuple(a for a in ds.records[0].counters)
    rt = np.array([ds.record_for(i).runtime_us for i in range(n)])
    th = np.array([ds.record_for(i).global_threads for i in range(n)], dtype=np.int64)
    cm = np.array([[ds.record_for(i).counters[k] for k in names] for i in range(n)])
    np.savez_compressed(
        os.path.join(HERE, "ds_gradient3x.npz"), runtime=rt, threads=th, counter_matrix=cm,
        counter_names=np.array(names), assignments=np.array([c.assignment for c in ds.space.configurations]),
        param_names=np.array(ds.space.parameter_names),
        param_binary=np.array([p.is_binary for p in ds.space.parameters]),
        generation=np.int32(0 if ds.arch.generation == "pre_volta" else 1),
        cores=np.int64(ds.arch.cores), arch_name=np.array(ds.arch.name),
        input_label=np.array(ds.input_label),
        c6_improvement=np.float64(improvement), c6_prof_mean=np.float64(prof.mean_steps),
        c6_rand_mean=np.float64(rand.mean_steps))
    print("C6 improvement", improvement, prof.mean_steps, rand.mean_steps)


if __name__ == "__main__":
    main()
