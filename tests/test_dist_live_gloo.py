"""Multi-process protocol of the live multi-GPU search (dist_live.py) with
the gloo backend on CPU, world sizes 2 and 3.

Every rank runs the searcher over a replayed dataset (the stand-in for its
GPU's live source; the numeric steps come from the oracle, a host-side
stand-in for the device kernels -- test infrastructure only), measures the
profiled configuration on one rank and its share of each iteration's draws,
and exchanges measurements through broadcast / all-gather.  The trace every
rank ends with must be the reference's sequential trajectory
(oracle.profile_search, pinned to the reference by test_oracle_golden.py),
and each rank must have measured only its own share of the draws.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def oracle_core(ds, matrix, column):
    """A host stand-in of search._profile_search_batches built from the
    oracle's primitives (same batch protocol)."""
    import countertune_oracle as oracle
    from paper_2102_05297_b200.search import SearchTrace, TraceStep
    from paper_2102_05297_b200.space import replay_arrays

    rt, th, req, hr = replay_arrays(ds)

    def factory(space, arch, *, i, n, seed, inst_reaction, literal_sign, stop_indices,
                score_top_k):
        N = len(space)
        rng = np.random.default_rng(seed)
        explored = np.zeros(N, dtype=bool)
        steps = []

        def rec(idx, runtime, profiled):
            steps.append(TraceStep(len(steps) + 1, idx, runtime, profiled))
            explored[idx] = True
            return stop_indices is not None and idx in stop_indices

        prof = int(rng.integers(0, N))
        for _ in range(i):
            m = (yield ([prof], True))[0]
            if rec(prof, m.runtime_us, True):
                return SearchTrace(steps, seed, "stopped")
            c = np.array([m.counters[k] for k in oracle.REQ])
            b, _ = oracle.analyze(c, False, arch.cores, m.global_threads)
            deltas = list(zip(oracle.DELTA_KEYS, oracle.react(b, inst_reaction)))
            if explored.all():
                return SearchTrace(steps, seed, "exhausted")
            raw, _ = oracle.score(matrix, column, prof, deltas, explored, literal_sign)
            w = oracle.normalize(raw, ~explored)
            chosen, exhausted = [], False
            for _ in range(n):
                if w.max() <= 0.0:
                    exhausted = True
                    break
                pick = oracle.select(w, rng)
                w[pick] = 0.0
                chosen.append(pick)
            got = (yield (chosen, False)) if chosen else []
            best = np.inf
            for pick, meas in zip(chosen, got):
                if rec(pick, meas.runtime_us, False):
                    return SearchTrace(steps, seed, "stopped")
                if meas.runtime_us <= best:
                    best, prof = meas.runtime_us, pick
            if exhausted:
                return SearchTrace(steps, seed, "exhausted")
        return SearchTrace(steps, seed, "budget")

    return factory


class CountingReplay:
    def __init__(self, ds):
        from paper_2102_05297_b200.search import DatasetReplaySource
        self.inner = DatasetReplaySource(ds)
        self.space, self.arch = ds.space, ds.arch
        self.calls = []

    def measure(self, idx, profiled):
        self.calls.append((int(idx), bool(profiled)))
        return self.inner.measure(idx, profiled)


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_05297_b200 import ExactModelSet, spaces
        from paper_2102_05297_b200.dist_live import run_profile_search_distributed
        from paper_2102_05297_b200.space import well_performing_set
        ds = spaces.coulomb()
        ms = ExactModelSet(ds)
        matrix = ms.prediction_matrix(ds.space)
        column = {c: j for j, c in enumerate(ms.counters)}
        stop = set(well_performing_set(ds, 1.1))
        res = {}
        for seed in range(6):
            for use_stop in (False, True):
                src = CountingReplay(ds)
                tr = run_profile_search_distributed(
                    src, None, i=12, n=5, seed=seed, stop_indices=stop if use_stop else None,
                    profile_rank=seed % world, core_factory=oracle_core(ds, matrix, column))
                key = f"s{seed}_{int(use_stop)}"
                res[key + "_idx"] = np.array([s.config_index for s in tr.steps])
                res[key + "_prof"] = np.array([s.profiled for s in tr.steps])
                res[key + "_status"] = np.array(tr.status)
                res[key + "_calls"] = np.array(src.calls, dtype=np.int64).reshape(-1, 2)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_live_search_is_the_reference_trajectory(world, tmp_path):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import countertune_oracle as oracle
    from paper_2102_05297_b200 import ExactModelSet, spaces
    from paper_2102_05297_b200.space import replay_arrays, well_performing_mask
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ds = spaces.coulomb()
    ms = ExactModelSet(ds)
    matrix = ms.prediction_matrix(ds.space)
    column = {c: j for j, c in enumerate(ms.counters)}
    rt, th, req, hr = replay_arrays(ds)
    stopm = well_performing_mask(ds, 1.1)
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for seed in range(6):
        for use_stop in (False, True):
            key = f"s{seed}_{int(use_stop)}"
            steps, status, _ = oracle.profile_search(
                matrix, column, rt, th, req, hr, pre_volta=False, cores=ds.arch.cores, i=12,
                n=5, seed=seed, stop=stopm if use_stop else None)
            for r, got in enumerate(ranks):
                assert got[key + "_idx"].tolist() == [s for s, _ in steps], (key, r)
                assert got[key + "_prof"].tolist() == [p for _, p in steps], (key, r)
                assert str(got[key + "_status"]) == status, (key, r)
            # measurement ownership: profiled steps only on profile_rank, and
            # each draw measured by exactly one rank (k mod world)
            calls = [got[key + "_calls"] for got in ranks]
            owner = seed % world
            for r in range(world):
                prof_calls = calls[r][calls[r][:, 1] == 1]
                assert (r == owner) == (len(prof_calls) > 0), (key, r)
            timed = sorted(int(c) for r in range(world) for c in calls[r][calls[r][:, 1] == 0][:, 0])
            drawn = [s for s, p in steps if not p]
            # every recorded draw was timed once; extra timed draws are the
            # ones past a stop configuration inside the last batch
            assert set(drawn) <= set(timed)
            assert len(timed) == len(set(timed)) or not use_stop


def _bcast_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_05297_b200 import ExactModelSet, spaces
        from paper_2102_05297_b200.dist_live import broadcast_table
        ds = spaces.coulomb()
        model = ExactModelSet(ds) if rank == 0 else None
        t = broadcast_table(model, ds.space, src=0)
        np.savez(os.path.join(out_dir, f"t{rank}.npz"), m=t.matrix,
                 names=np.array(t.counter_names))
    finally:
        dist.destroy_process_group()


def test_model_broadcast(tmp_path):
    from paper_2102_05297_b200 import ExactModelSet, spaces
    mp.spawn(_bcast_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    ds = spaces.coulomb()
    ms = ExactModelSet(ds)
    want = ms.prediction_matrix(ds.space)
    for r in range(3):
        got = np.load(tmp_path / f"t{r}.npz")
        np.testing.assert_array_equal(got["m"], want)
        assert got["names"].tolist() == list(ms.counters)
