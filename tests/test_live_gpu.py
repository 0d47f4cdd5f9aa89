"""Live measurement path on the GPU: every benchmark kernel against its numpy
oracle (oracle/benchmarks_oracle.py) on a seeded sample of its tuning space,
the CUPTI collector's counter set, and the ask/tell searcher against the
batched device search.

Tolerances (stated FP32 bounds, relative to the magnitude sum of the terms,
see benchmarks_oracle.within): transpose bit-exact; coulomb / nbody 2e-6
(rsqrtf is within 2^-22.9 relative, per-term); conv 1e-6; gemm 1e-6 (FFMA
path and the 3xTF32 tensor-core path).
"""

import numpy as np
import pytest

import benchmarks_oracle as bo

pytestmark = pytest.mark.gpu

SAMPLE = 14


def _sample(n, seed):
    rng = np.random.default_rng(seed)
    return sorted({0, n - 1, *rng.choice(n, size=min(n, SAMPLE), replace=False).tolist()})


@pytest.fixture(scope="module")
def tuner():
    from paper_2102_05297_b200.tuner import Tuner
    t = Tuner(0)
    yield t
    t.close()


def _check(src, idxs, got_want):
    bad = src.compile_all(idxs)
    assert bad == 0, src.compile_failures
    worst = 0.0
    for i in idxs:
        worst = max(worst, got_want(i))
    return worst


def test_device_info(tuner):
    assert tuner.arch.startswith("sm_10")
    assert tuner.sm_count >= 100


def test_transpose_matches_oracle(tuner):
    from paper_2102_05297_b200.live import CudaMeasurementSource, benchmark
    b = benchmark("transpose", width=1024, height=512)
    src = CudaMeasurementSource(b, tuner=tuner)
    want = bo.transpose(b.host_inputs()["in"])
    for i in _sample(len(b.space), 1):
        src.compile_all([i])
        got = src.output(i)
        assert np.array_equal(got, want), (i, b.values(i))


@pytest.mark.parametrize("name,sizes,rtol", [
    ("coulomb", dict(grid=64, atoms=256), 2e-6),
    ("nbody", dict(bodies=2048), 2e-6),
    ("conv", dict(width=1024, height=256), 1e-6),
    ("gemm", dict(m=256, n=256, k=128), 1e-6),
])
def test_benchmark_matches_oracle(tuner, name, sizes, rtol):
    from paper_2102_05297_b200.live import CudaMeasurementSource, benchmark
    b = benchmark(name, **sizes)
    src = CudaMeasurementSource(b, tuner=tuner)
    h = b.host_inputs()
    if name == "coulomb":
        want, mag = bo.coulomb(h["atoms"], b.spacing, b.grid)
    elif name == "nbody":
        want, mag = bo.nbody(h["pm"], b.eps2)
    elif name == "conv":
        want, mag = bo.conv(h["in"], h["filt"])
    else:
        want, mag = bo.gemm(h["at"], h["b"])
    idxs = _sample(len(b.space), 2)
    # the packed-FP32 (FFMA2) paths in the sample: nbody OUTER even, conv
    # LOCAL = 2 with WPTX even (two tile copies), both filter placements
    if name == "nbody":
        paired = [i for i in range(len(b.space)) if b.values(i)["OUTER"] % 2 == 0]
        idxs = sorted(set(idxs) | set(paired[:: max(1, len(paired) // 6)][:6]))
    if name == "conv":
        paired = [i for i in range(len(b.space))
                  if b.values(i)["LOCAL"] == 2 and b.values(i)["WPTX"] % 2 == 0]
        idxs = sorted(set(idxs) | set(paired[:: max(1, len(paired) // 8)][:8]))
    if name == "gemm":   # both tensor-core paths (mma.sync, tcgen05) in the sample
        tc = [i for i in range(len(b.space)) if b.values(i)["TC"] == 1 and not b.tc5(b.values(i))]
        tc5 = [i for i in range(len(b.space)) if b.tc5(b.values(i))]
        assert tc5, "no tcgen05 variant in the space"
        idxs = sorted(set(idxs) | set(tc[:: max(1, len(tc) // 4)][:4])
                      | set(tc5[:: max(1, len(tc5) // 8)][:8]))
    worst = _check(src, idxs, lambda i: bo.within(src.output(i), want, mag, 1.0))
    assert worst <= rtol, f"{name}: worst relative error {worst:.3g} > {rtol}"


def test_profiled_measurement_has_table1_counters(tuner):
    from paper_2102_05297_b200 import counters as cc
    from paper_2102_05297_b200.live import CudaMeasurementSource, TABLE1_METRICS, benchmark
    b = benchmark("transpose", width=2048, height=2048)
    src = CudaMeasurementSource(b, tuner=tuner)
    i = 0
    m = src.measure(i, profiled=True)
    assert m.runtime_us > 0
    assert m.global_threads == src.launch_of(i).threads
    assert set(m.counters) >= set(cc.REQUIRED_COUNTERS)
    assert src.profile_passes >= 1
    assert tuner.profile_passes(TABLE1_METRICS) == src.profile_passes
    # transpose reads and writes every element once: DRAM/L2 sectors are at
    # least the algorithmic 2 x 4 B x n / 32 B
    sectors = 2 * 4 * 2048 * 2048 / 32
    assert m.counters["L2_RT"] + m.counters["L2_WT"] >= 0.9 * sectors
    for k, v in m.counters.items():
        assert np.isfinite(v) and v >= 0, (k, v)


def test_ask_tell_matches_batched_device_search():
    """ProfileSearcher driven by a replay source == the batched device search."""
    from paper_2102_05297_b200 import (DatasetReplaySource, ExactModelSet, ProfileSearcher,
                                       run_profile_search, spaces)
    from paper_2102_05297_b200.space import well_performing_set
    ds = spaces.coulomb()
    src = DatasetReplaySource(ds)
    model = ExactModelSet(ds)
    stop = set(well_performing_set(ds, 1.1))
    total = 0
    for seed in range(6):
        st = stop if seed % 2 else None      # budget runs and stop-set runs
        want = run_profile_search(src, model, i=8, seed=seed, stop_indices=st)
        s = ProfileSearcher(model, ds.space, ds.arch, i=8, seed=seed, stop_indices=st)
        while (req := s.next_config()) is not None:
            s.add_result(src.measure(*req))
        got = s.trace
        assert [x.config_index for x in got.steps] == [x.config_index for x in want.steps]
        assert [x.profiled for x in got.steps] == [x.profiled for x in want.steps]
        assert got.status == want.status
        total += len(got.steps)
    assert total >= 3 * 8 * 6                # the budget runs went the full 8 iterations
    with pytest.raises(Exception):
        s.add_result(src.measure(0, False))  # nothing pending after the end


def test_live_profile_search_runs(tuner):
    """Alg. 1 against real kernels: a live search on the coulomb space with a
    model from a live sweep of the same space (small grid)."""
    from paper_2102_05297_b200 import ExactModelSet, run_profile_search
    from paper_2102_05297_b200.live import CudaMeasurementSource, benchmark, sweep
    b = benchmark("coulomb", grid=64, atoms=256)
    src = CudaMeasurementSource(b, tuner=tuner, reps=2)
    res = sweep(src)
    ds = res.dataset
    assert not res.failures, res.failures
    assert ds.has_record.all()
    model = ExactModelSet(ds)
    trace = run_profile_search(src, model, i=4, seed=1)
    assert len(trace.steps) == 4 * 6
    assert [s.profiled for s in trace.steps[::6]] == [True] * 4
    # no configuration drawn twice within an outer iteration
    for k in range(4):
        inner = [s.config_index for s in trace.steps[6 * k + 1:6 * k + 6]]
        assert len(set(inner)) == 5


def test_group1_single_pass_profiled_step(tuner):
    """The labelled single-pass mode: a profiled step collects the 13-metric
    group 1 in ONE CUPTI pass and takes the other Table-1 counters from the
    recorded sweep of the space (what the exact model replays; SHR_U is in
    no model and not in group 1); a live search runs on it, and the
    collected counters agree with a full 24-metric profile of the same
    launch (L2 sectors and executed instructions within 5%)."""
    from paper_2102_05297_b200 import ExactModelSet, run_profile_search
    from paper_2102_05297_b200.live import (GROUP1_ABBRS, GROUP1_METRICS, CudaMeasurementSource,
                                            benchmark, sweep)
    from paper_2102_05297_b200.search import PredictionTable
    b = benchmark("transpose", width=1024, height=1024)
    full = CudaMeasurementSource(b, tuner=tuner, reps=2)
    ds = sweep(full, profiled=True).dataset
    table = PredictionTable.from_model_set(ExactModelSet(ds), ds.space)
    with pytest.raises(ValueError, match="SHR_U"):       # no model predicts it
        CudaMeasurementSource(b, tuner=tuner, metrics=GROUP1_METRICS, fill_from=table)
    g1 = CudaMeasurementSource(b, tuner=tuner, reps=2, metrics=GROUP1_METRICS, fill_from=ds)
    assert g1.mode == "group1+model" and full.mode == "full"
    best = int(np.argmin(ds.runtime_us))
    m1 = g1.measure(best, profiled=True)
    assert g1.profile_passes == 1
    mf = full.measure(best, profiled=True)
    assert full.profile_passes > 1
    assert set(m1.counters) == set(mf.counters)
    for a in ("L2_RT", "L2_WT", "INST_EXE"):     # (DRAM reads: the 4 MB input sits in L2)
        assert a in GROUP1_ABBRS
        assert abs(m1.counters[a] - mf.counters[a]) <= 0.05 * max(mf.counters[a], 1.0), a
    col = {a: j for j, a in enumerate(ds.counter_names)}
    for a in set(mf.counters) - set(GROUP1_ABBRS):   # from the recorded sweep
        assert m1.counters[a] == pytest.approx(ds.counter_matrix[best, col[a]]), a
    trace = run_profile_search(g1, ExactModelSet(ds), i=3, seed=2)
    assert len(trace.steps) == 3 * 6


def test_distributed_live_search_world1_matches_device_search():
    """dist_live with the device searcher core (world size 1, gloo) gives the
    batched device search's trajectory on a replayed dataset."""
    import socket
    import torch.distributed as dist
    from paper_2102_05297_b200 import (DatasetReplaySource, ExactModelSet, run_profile_search,
                                       spaces)
    from paper_2102_05297_b200.dist_live import run_profile_search_distributed
    from paper_2102_05297_b200.space import well_performing_set
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        ds = spaces.transpose()
        src = DatasetReplaySource(ds)
        model = ExactModelSet(ds)
        stop = set(well_performing_set(ds, 1.1))
        for seed in range(3):
            want = run_profile_search(src, model, i=10, seed=seed, stop_indices=stop)
            got = run_profile_search_distributed(src, model, i=10, seed=seed, stop_indices=stop)
            assert [s.config_index for s in got.steps] == [s.config_index for s in want.steps]
            assert got.status == want.status
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,rtol", [("coulomb", 2e-6), ("nbody", 2e-6), ("conv", 1e-6),
                                       ("gemm", 1.1e-5), ("transpose", 0.0)])
def test_best_configuration_at_paper_size_matches_oracle(tuner, name, rtol):
    """The exhaustive sweep's best configuration of every space, at the
    paper's input size, against the oracle.

    GEMM at K = 2048: FP32 accumulation of 2048 products, tolerance
    4 sqrt(K) 2^-24 = 1.1e-5 of the magnitude sum (the rigorous worst case of
    a K-term FP32 sum is K 2^-24 = 1.2e-4; the K = 128 tests use 1e-6)."""
    import os
    from paper_2102_05297_b200 import formats
    from paper_2102_05297_b200.live import CudaMeasurementSource, benchmark
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ds = formats.load_dataset_dir(os.path.join(root, "datasets", f"{name}-b200"))
    best = int(np.argmin(np.where(ds.has_record, ds.runtime_us, np.inf)))
    b = benchmark(name)
    src = CudaMeasurementSource(b, tuner=tuner)
    h = b.host_inputs()
    got = src.output(best)
    if name == "transpose":
        assert np.array_equal(got, bo.transpose(h["in"]))
        return
    if name == "coulomb":
        want, mag = bo.coulomb(h["atoms"], b.spacing, b.grid)
    elif name == "nbody":
        want, mag = bo.nbody(h["pm"], b.eps2)
    elif name == "conv":
        want, mag = bo.conv(h["in"], h["filt"])
    else:
        want, mag = bo.gemm(h["at"], h["b"])
    err = bo.within(got, want, mag, 1.0)
    assert err <= rtol, f"{name} best config {best}: relative error {err:.3g}"
