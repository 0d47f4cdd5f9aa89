"""One experiment's repetitions sharded over the ranks of a process group.

The reference fans repetitions out over worker processes with strided
chunks and merges the results on the parent (harness.py:175-187); reports do
not depend on the worker count.  Here every rank owns one GPU and a
contiguous range of repetitions (so the SeedSequence children of rank k are
spawn keys [first_k, first_k + n_k), ct_seed_spec.rep_offset), runs its
range as one batched launch and aggregates it on its device.  The only
exchange is the report itself:

  * all-gather of the per-repetition step counts, statuses and completion
    times (O(R) numbers);
  * the reference sums the padded best-so-far curves over repetitions in
    repetition order (harness.py:196-201, 218-223), so the partial column
    sums are passed down the rank chain 0 -> 1 -> ... -> W-1 (point-to-point,
    one hop per rank) and broadcast from the last rank: the float additions
    happen in exactly the reference's order and the report is byte-identical
    for any world size.

Collectives use the group's backend: NCCL over NVLink between GPUs, gloo on
CPU (the tests run world_size 2 with gloo and a host-side shard).
"""

from typing import Callable, Optional, Tuple

import numpy as np

from . import _native
from .harness import (SEARCHER_PROFILE, TIME_GRID_POINTS, ConvergenceReport, ExperimentSpec,
                      _as_table, launch, prepare_device)
from .search import rep_error


def rep_range(reps: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [first, first + n) of rank `rank` (np.array_split sizes)."""
    base, extra = divmod(reps, world)
    n = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, n


class DeviceShard:
    """The repetitions [first, first + n) of an experiment on one GPU."""

    def __init__(self, spec: ExperimentSpec, first: int, n: int, device: int = 0):
        self.first, self.n = first, n
        self.ctx = _native.context(device)
        table = None
        if spec.searcher == SEARCHER_PROFILE:
            table = _as_table(spec.model, spec.dataset.space)
        params, _ = prepare_device(self.ctx, spec, table)
        if n:
            launch(self.ctx, spec, params, first, n)

    def status(self):
        """(n_steps, status, configs scored, uncertified draws, error).

        error is None, or (global repetition, status code, failing index) of
        the range's first failed repetition.  It is returned, not raised: the
        caller exchanges it with the other ranks first, so that every rank
        raises the same exception instead of one rank leaving its peers
        blocked in a collective."""
        if self.n == 0:
            return (np.zeros(0, np.int32), np.zeros(0, np.int32), 0, 0, None)
        nst, status, err, stats = self.ctx.fetch_status(self.n)
        bad = np.flatnonzero(status == _native.CT_STATUS_ERROR)
        error = None
        if bad.size:
            r = int(bad[0])
            error = (self.first + r, int(err[r]), self.ctx.failing_index(r, self.n))
        return nst, status, int(stats.configs_scored), int(stats.uncertified), error

    def aggregate_steps(self, overhead, max_len, sum0, sq0):
        if self.n == 0:
            return sum0, sq0, np.zeros(0), np.zeros(0)
        return self.ctx.aggregate_steps(overhead, self.n, max_len, sum0, sq0)

    def aggregate_time(self, count, grid, sum0, sq0):
        if count == 0:
            return sum0, sq0
        return self.ctx.aggregate_time(count, grid, sum0, sq0)


def _tensor_device(dist):
    import torch
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _all_gather_1d(dist, arr: np.ndarray, counts, dev) -> np.ndarray:
    """Concatenation in rank order of each rank's 1-D float64/int64 array."""
    import torch
    width = max(counts) if counts else 0
    pad = np.zeros(width, dtype=arr.dtype)
    pad[:arr.size] = arr
    t = torch.from_numpy(pad).to(dev)
    outs = [torch.empty_like(t) for _ in counts]
    dist.all_gather(outs, t)
    return np.concatenate([o.cpu().numpy()[:c] for o, c in zip(outs, counts)])


def _chain_pairs(dist, rank: int, world: int, dev, length: int,
                 fn: Callable[[Optional[np.ndarray], Optional[np.ndarray]],
                              Tuple[Optional[np.ndarray], Optional[np.ndarray]]]):
    """Run fn(sum0, sq0) on every rank in rank order, each rank starting from
    its predecessor's (sum, sq) (None on rank 0, or if no predecessor has
    contributed yet); return the last rank's pair on every rank.

    The message is [has, sum(length), sq(length)] float64."""
    import torch
    sum0 = sq0 = None
    if rank > 0:
        buf = torch.empty(1 + 2 * length, dtype=torch.float64, device=dev)
        dist.recv(buf, src=rank - 1)
        host = buf.cpu().numpy()
        if host[0] != 0.0:
            sum0, sq0 = host[1:1 + length].copy(), host[1 + length:].copy()
    s, q = fn(sum0, sq0)
    msg = np.zeros(1 + 2 * length)
    if s is not None:
        msg[0] = 1.0
        msg[1:1 + length] = s
        msg[1 + length:] = q
    t = torch.from_numpy(msg).to(dev)
    if rank < world - 1:
        dist.send(t, dst=rank + 1)
    dist.broadcast(t, src=world - 1)
    host = t.cpu().numpy()
    if host[0] == 0.0:
        return None, None
    return host[1:1 + length].copy(), host[1 + length:].copy()


def simulate_distributed(spec: ExperimentSpec, device: int = 0,
                         shard_factory: Optional[Callable] = None) -> ConvergenceReport:
    """harness.simulate over the default process group (one rank per GPU).

    shard_factory(spec, first, n) -> shard (DeviceShard interface); the
    default runs the range on `device`.  Every rank returns the same report.
    """
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = _tensor_device(dist)
    reps = spec.repetitions
    first, n = rep_range(reps, world, rank)
    shard = (shard_factory or (lambda s, f, c: DeviceShard(s, f, c, device)))(spec, first, n)
    nst_local, status_local, scored, uncert, error = shard.status()
    counts = [rep_range(reps, world, k)[1] for k in range(world)]

    # every rank learns of any rank's failed repetition before the report's
    # collectives start, and all raise the error of the lowest failed
    # repetition (the one a sequential run meets first)
    mine = np.array(error if error is not None else (reps, 0, -1), dtype=np.int64)
    errs = _all_gather_1d(dist, mine, [3] * world, dev).reshape(world, 3)
    worst = errs[int(np.argmin(errs[:, 0]))]
    if int(worst[0]) < reps:
        raise rep_error(int(worst[1]), int(worst[2]))

    nst = _all_gather_1d(dist, nst_local.astype(np.int64), counts, dev)
    status = _all_gather_1d(dist, status_local.astype(np.int64), counts, dev)
    tot = torch.tensor([scored, uncert], dtype=torch.int64, device=dev)
    dist.all_reduce(tot)
    scored, uncert = (int(x) for x in tot.cpu().tolist())
    max_len = int(nst.max())

    local = {}

    def steps_fn(s0, q0):
        s, q, total, firsts = shard.aggregate_steps(spec.profiling_overhead, max_len, s0, q0)
        local["total"], local["first"] = total, firsts
        return s, q

    col_sum, col_sq = _chain_pairs(dist, rank, world, dev, max_len, steps_fn)
    total_times = _all_gather_1d(dist, np.asarray(local["total"], dtype=np.float64), counts, dev)
    first_times = _all_gather_1d(dist, np.asarray(local["first"], dtype=np.float64), counts, dev)
    mean = col_sum / reps
    var = np.maximum(0.0, col_sq / reps - mean * mean)
    step_std = np.sqrt(var)

    tr = reps if spec.time_repetitions is None else min(reps, spec.time_repetitions)
    t_start = float(np.max(first_times[:tr]))     # exact in any order
    t_end = float(np.max(total_times[:tr]))
    if t_end > t_start:
        grid = np.linspace(t_start, t_end, TIME_GRID_POINTS)
    else:
        grid = np.array([t_start])
    count = min(n, max(0, tr - first))
    tc_sum, tc_sq = _chain_pairs(dist, rank, world, dev, grid.size,
                                 lambda s0, q0: shard.aggregate_time(count, grid, s0, q0))
    tmean = tc_sum / tr
    tvar = np.maximum(0.0, tc_sq / tr - tmean * tmean)
    ds = spec.dataset
    return ConvergenceReport(
        name=spec.name, searcher=spec.searcher,
        dataset_label=f"{ds.arch.name}/{ds.input_label}", repetitions=reps,
        inner_steps=spec.inner_steps, outer_iterations=spec.resolved_outer_iterations(),
        seed=spec.seed, slack=spec.slack, profiling_overhead=spec.profiling_overhead,
        steps=nst.astype(float),
        censored=int(np.count_nonzero(status != _native.CT_STATUS_STOPPED)),
        mean_time_seconds=float(np.mean(total_times)) / 1e6,
        step_curve_mean=mean, step_curve_std=step_std, time_grid_seconds=grid / 1e6,
        time_curve_mean=tmean, time_curve_std=np.sqrt(tvar),
        configs_scored=scored, uncertified_draws=uncert)
