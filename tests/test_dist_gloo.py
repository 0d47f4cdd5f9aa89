"""Multi-process host logic of the sharded harness (dist.simulate_distributed)
with the gloo backend on CPU, world sizes 2 and 3.

Each rank owns a contiguous repetition range; its trajectories come from the
oracle (a host-side stand-in for the rank's GPU, test infrastructure only)
and its partial report sums follow the device kernels' arithmetic
(k_agg_cols / k_agg_time_sums: sequential over repetitions, seeded with the
predecessor rank's sums).  The distributed report must be byte-identical to
the reference's own harness.simulate (tests/golden/sim_gradient.npz).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT, dataset_from_golden


class HostShard:
    """DeviceShard's interface over oracle trajectories of reps [first, first+n)."""

    def __init__(self, spec, first, n):
        import countertune_oracle as oracle
        from paper_2102_05297_b200 import ExactModelSet
        from paper_2102_05297_b200.space import replay_arrays, well_performing_mask
        ds = spec.dataset
        rt, th, req, hr = replay_arrays(ds)
        stop = well_performing_mask(ds, spec.slack)
        seeds = np.random.SeedSequence(spec.seed).spawn(spec.repetitions)
        self.first, self.n, self.rt = first, n, rt
        self.traj = []
        for r in range(first, first + n):
            if spec.searcher == "profile":
                ms = ExactModelSet(ds)
                matrix = ms.prediction_matrix(ds.space)
                column = {c: j for j, c in enumerate(ms.counters)}
                steps, status, _ = oracle.profile_search(
                    matrix, column, rt, th, req, hr, pre_volta=ds.arch.generation == "pre_volta",
                    cores=ds.arch.cores, i=spec.resolved_outer_iterations(), n=spec.inner_steps,
                    seed=seeds[r], stop=stop)
            else:
                idx, status = oracle.random_search(len(ds.space), seed=seeds[r], stop=stop)
                steps = [(k, False) for k in idx]
            self.traj.append((steps, status))

    def status(self):
        nst = np.array([len(s) for s, _ in self.traj], dtype=np.int32)
        code = {"budget": 0, "stopped": 1, "exhausted": 2}
        status = np.array([code[st] for _, st in self.traj], dtype=np.int32)
        return nst, status, 0, 0, None

    def _rows(self, overhead):
        out = []
        for steps, _ in self.traj:
            rts = np.array([self.rt[i] for i, _ in steps])
            costs = np.array([self.rt[i] * (overhead if p else 1.0) for i, p in steps])
            out.append((np.minimum.accumulate(rts), np.cumsum(costs)))
        return out

    def aggregate_steps(self, overhead, max_len, sum0, sq0):
        s = np.zeros(max_len) if sum0 is None else sum0.copy()
        q = np.zeros(max_len) if sq0 is None else sq0.copy()
        self.rows = self._rows(overhead)
        for bsf, _ in self.rows:
            padded = np.concatenate([bsf, np.full(max_len - len(bsf), bsf[-1])])
            s += padded
            q += padded * padded
        total = np.array([t[-1] for _, t in self.rows])
        first = np.array([t[0] for _, t in self.rows])
        return s, q, total, first

    def aggregate_time(self, count, grid, sum0, sq0):
        if count == 0:
            return sum0, sq0
        s = np.zeros(grid.size) if sum0 is None else sum0.copy()
        q = np.zeros(grid.size) if sq0 is None else sq0.copy()
        for bsf, times in self.rows[:count]:
            pos = np.searchsorted(times, grid, side="right") - 1
            sampled = bsf[np.clip(pos, 0, len(bsf) - 1)]
            s += sampled
            q += sampled * sampled
        return s, q


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_05297_b200 import ExactModelSet, ExperimentSpec
        from paper_2102_05297_b200.dist import simulate_distributed
        ds = dataset_from_golden("gradient")
        res = {}
        for searcher in ("profile", "random"):
            spec = ExperimentSpec(dataset=ds, searcher=searcher,
                                  model=ExactModelSet(ds) if searcher == "profile" else None,
                                  name=f"{searcher}-search", repetitions=50, seed=7,
                                  time_repetitions=20)
            rep = simulate_distributed(spec, shard_factory=HostShard)
            for f in ("steps", "step_curve_mean", "step_curve_std", "time_grid_seconds",
                      "time_curve_mean", "time_curve_std"):
                res[f"{searcher}_{f}"] = getattr(rep, f)
            res[f"{searcher}_censored"] = np.int64(rep.censored)
            res[f"{searcher}_mean_time_seconds"] = np.float64(rep.mean_time_seconds)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


class FailingShard(HostShard):
    """Rank 1's range holds a repetition whose replay lookup failed."""

    def status(self):
        nst, status, a, b, _ = super().status()
        if self.first > 0:
            return nst, status, a, b, (self.first + 1, -4, 123)
        return nst, status, a, b, None


def _error_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_05297_b200 import ExperimentSpec
        from paper_2102_05297_b200.dist import simulate_distributed
        ds = dataset_from_golden("gradient")
        spec = ExperimentSpec(dataset=ds, searcher="random", repetitions=10, seed=7)
        try:
            simulate_distributed(spec, shard_factory=FailingShard)
            msg = "no error"
        except Exception as e:     # noqa: BLE001 - the message is the result
            msg = f"{type(e).__name__}: {e}"
        with open(os.path.join(out_dir, f"err{rank}.txt"), "w") as f:
            f.write(msg)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_rep_range_partitions():
    from paper_2102_05297_b200.dist import rep_range
    for reps in (1, 7, 50, 1000):
        for world in (1, 2, 3, 8):
            spans = [rep_range(reps, world, k) for k in range(world)]
            want = np.array_split(np.arange(reps), world)
            for (first, n), w in zip(spans, want):
                assert n == w.size and (n == 0 or first == int(w[0]))


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_report_matches_reference(world, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    gold = np.load(os.path.join(GOLDEN, "sim_gradient.npz"))
    for rank in range(world):
        got = np.load(tmp_path / f"rank{rank}.npz")
        for key in got.files:
            np.testing.assert_array_equal(got[key], gold[key], err_msg=f"rank {rank}: {key}")


@pytest.mark.timeout(120)
def test_failed_repetition_raises_on_every_rank(tmp_path):
    """A failed repetition on one rank is raised by all ranks (no rank is
    left waiting in a collective)."""
    world = 2
    mp.spawn(_error_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    msgs = [open(tmp_path / f"err{r}.txt").read() for r in range(world)]
    assert msgs[0] == msgs[1]
    assert msgs[0] == "CounterTuneError: dataset holds no measurement for configuration 123"
