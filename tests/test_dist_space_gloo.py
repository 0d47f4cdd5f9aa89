"""Configuration-space sharding of one search (dist_space.py) with the gloo
backend, world sizes 2 and 3.

CPU: every rank scores only its contiguous shard -- the scorer sees every
other configuration masked as explored -- through a host stand-in for the
device scorer (the oracle's Eq. 16, pinned to the reference by
test_oracle_golden.py; test infrastructure only), and the all-gathered
raw-score vector must equal the unsharded one bit for bit on every rank.

GPU: the same with the device scorer (both ranks on cuda:0), and a whole
live-protocol search with the space sharded must follow the reference's
trajectory.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_bounds_partition_the_space():
    from paper_2102_05297_b200.dist_space import shard_bounds
    for n in (0, 1, 7, 210, 1784, 205216):
        for world in (1, 2, 3, 8):
            parts = [shard_bounds(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def _cases(ds):
    """A few (profile, deltas, explored) Eq. 16 inputs on the dataset."""
    import countertune_oracle as oracle
    from paper_2102_05297_b200 import counters as cc
    rng = np.random.default_rng(11)
    n = len(ds.space)
    out = []
    for k in range(4):
        prof = int(rng.integers(0, n))
        explored = rng.random(n) < 0.2 * k
        d = rng.uniform(-1, 1, len(cc.DELTA_KEYS))
        d[rng.random(len(d)) < 0.3] = 0.0
        out.append((prof, dict(zip(cc.DELTA_KEYS, map(float, d))), explored,
                    k % 2 == 1))
    return out


def _cpu_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import countertune_oracle as oracle
        from paper_2102_05297_b200 import ExactModelSet, spaces
        from paper_2102_05297_b200.dist_space import score_configurations_sharded
        ds = spaces.transpose()
        ms = ExactModelSet(ds)
        matrix = ms.prediction_matrix(ds.space)
        column = {c: j for j, c in enumerate(ms.counters)}
        seen = []

        def host_scorer(models, c_profile, delta, space, shard_explored, literal_sign):
            seen.append(int((~shard_explored).sum()))
            raw, _ = oracle.score(matrix, column, c_profile.index, list(delta.items()),
                                  shard_explored, literal_sign)
            return raw

        res = {}
        for k, (prof, delta, explored, lit) in enumerate(_cases(ds)):
            sv = score_configurations_sharded(ms, ds.space.configurations[prof], delta,
                                              ds.space, explored, literal_sign=lit,
                                              scorer=host_scorer)
            res[f"raw{k}"] = sv.raw
        res["seen"] = np.array(seen)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_scores_are_the_unsharded_scores(world, tmp_path):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import countertune_oracle as oracle
    from paper_2102_05297_b200 import ExactModelSet, spaces
    from paper_2102_05297_b200.dist_space import shard_bounds
    mp.spawn(_cpu_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ds = spaces.transpose()
    ms = ExactModelSet(ds)
    matrix = ms.prediction_matrix(ds.space)
    column = {c: j for j, c in enumerate(ms.counters)}
    n = len(ds.space)
    for rank in range(world):
        got = np.load(os.path.join(tmp_path, f"rank{rank}.npz"))
        lo, hi = shard_bounds(n, world, rank)
        for k, (prof, delta, explored, lit) in enumerate(_cases(ds)):
            want, _ = oracle.score(matrix, column, prof, list(delta.items()), explored, lit)
            assert np.array_equal(got[f"raw{k}"].view(np.uint64), want.view(np.uint64)), (rank, k)
            # this rank scored only its own shard's unexplored configurations
            assert got["seen"][k] == int((~explored[lo:hi]).sum())


def _gpu_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import dataset_from_golden, golden
        from paper_2102_05297_b200 import ExactModelSet
        from paper_2102_05297_b200.dist_live import run_profile_search_distributed
        from paper_2102_05297_b200.dist_space import score_configurations_sharded
        from paper_2102_05297_b200.search import DatasetReplaySource, score_configurations
        ds = dataset_from_golden("b200_transpose")
        ms = ExactModelSet(ds)
        res = {}
        for k, (prof, delta, explored, lit) in enumerate(_cases(ds)):
            a = score_configurations_sharded(ms, ds.space.configurations[prof], delta, ds.space,
                                             explored, literal_sign=lit).raw
            b = score_configurations(ms, ds.space.configurations[prof], delta, ds.space,
                                     explored, literal_sign=lit).raw
            res[f"same{k}"] = np.array(np.array_equal(a.view(np.uint64), b.view(np.uint64)))
        traj = golden("traj_b200_transpose.npz")
        seeds = np.random.SeedSequence(42).spawn(int(traj["reps"]))
        for r in range(3):
            tr = run_profile_search_distributed(DatasetReplaySource(ds), ms, i=int(traj["i"]),
                                                n=5, seed=seeds[r], shard_space=True)
            res[f"traj{r}"] = np.array([s.config_index for s in tr.steps])
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_space_search_on_the_gpu_is_the_reference_trajectory(tmp_path):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from conftest import golden, ragged
    world = 2
    mp.spawn(_gpu_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    traj = golden("traj_b200_transpose.npz")
    want = ragged(traj, "exact_nostop")
    for rank in range(world):
        got = np.load(os.path.join(tmp_path, f"rank{rank}.npz"))
        for k in range(4):
            assert bool(got[f"same{k}"]), (rank, k)
        for r in range(3):
            assert got[f"traj{r}"].tolist() == want[r], (rank, r)
