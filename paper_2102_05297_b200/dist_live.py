"""Live profile search with the empirical tests of an outer iteration spread
over the GPUs of one box (SURVEY section 8e, row "live tuning").

Alg. 1's n draws depend only on the iteration's weights and the Generator,
not on the runtimes measured between them (search.py:388-398), so every
rank runs the same searcher (same seed, same model, its own GPU for the
scoring kernels) and, per outer iteration:

  * the profiled configuration is measured once, on ``profile_rank``, and
    its Measurement (runtime, threads, the Table-1 counters) is broadcast --
    one message of 2 + 25 float64;
  * draw k is timed on rank k mod W, all ranks time their candidates
    concurrently, and an all-gather of the runtimes (n float64 per rank)
    gives every rank the iteration's runtimes in draw order; the "tiny
    cross-GPU argmax" -- later ties win, truncated at the first stop
    configuration -- is then evaluated identically on every rank.

The model itself is shared once: ``broadcast_table`` sends rank 0's
prediction table (N x C float64, e.g. 31 MB at N = 205,216) to every rank, so
only one rank needs the model (north_star: NCCL "for that and for the model
broadcast").  Nothing else crosses the interconnect, so every rank ends with
the same SearchTrace, and for a replayed source it is the reference's trajectory for
any world size.  Collectives use the default group's backend (NCCL over
NVLink with one rank per GPU; gloo on CPU for the tests).
"""

from typing import Callable, List, Optional, Set

import numpy as np

from . import counters as cc
from .search import (DEFAULT_INNER_STEPS, DEFAULT_INST_REACTION, Measurement, SearchTrace,
                     _as_table, _profile_search_batches)

_NAMES = cc.ABBREVIATIONS


def _device(dist):
    import torch
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _encode(m: Optional[Measurement]) -> np.ndarray:
    v = np.full(2 + len(_NAMES), np.nan)
    if m is not None:
        v[0] = m.runtime_us
        v[1] = -1.0 if m.global_threads is None else float(m.global_threads)
        for j, a in enumerate(_NAMES):
            if m.counters and a in m.counters:
                v[2 + j] = m.counters[a]
    return v


def _decode(v: np.ndarray) -> Measurement:
    counters = {a: float(v[2 + j]) for j, a in enumerate(_NAMES) if not np.isnan(v[2 + j])}
    threads = None if v[1] < 0 else int(v[1])
    return Measurement(runtime_us=float(v[0]), global_threads=threads, counters=counters)


def broadcast_table(table, space=None, src: int = 0):
    """Rank src's PredictionTable (or model: it is materialised there first)
    on every rank, by one broadcast of its N x C float64 matrix.  Other ranks
    pass None (or anything) plus the space."""
    import torch
    import torch.distributed as dist
    from .search import PredictionTable
    rank = dist.get_rank()
    dev = _device(dist)
    if rank == src:
        t = _as_table(table, space if space is not None else table.space)
        names = list(t.counter_names)
        shape = torch.tensor(list(t.matrix.shape), dtype=torch.int64, device=dev)
    else:
        names = None
        shape = torch.zeros(2, dtype=torch.int64, device=dev)
    dist.broadcast(shape, src=src)
    holder = [names]
    dist.broadcast_object_list(holder, src=src)
    n, c = (int(x) for x in shape.cpu().tolist())
    buf = (torch.from_numpy(np.ascontiguousarray(t.matrix, dtype=np.float64)).to(dev)
           if rank == src else torch.empty((n, c), dtype=torch.float64, device=dev))
    dist.broadcast(buf, src=src)
    if rank == src:
        return t
    return PredictionTable(space, holder[0], buf.cpu().numpy())


def run_profile_search_distributed(source, models, *, i: int, n: int = DEFAULT_INNER_STEPS,
                                   seed=0, inst_reaction: float = DEFAULT_INST_REACTION,
                                   literal_sign: bool = False,
                                   stop_indices: Optional[Set[int]] = None,
                                   score_top_k: Optional[int] = None, profile_rank: int = 0,
                                   core_factory: Optional[Callable] = None,
                                   shard_space: bool = False) -> SearchTrace:
    """run_profile_search over the default process group; every rank passes
    its own measurement source (its GPU) and gets the same trace back.

    ``seed`` must be regenerable (an int or SeedSequence), so that all ranks
    draw the same stream.  ``core_factory`` replaces the device searcher
    (tests drive the protocol with a host stand-in).  ``shard_space`` also
    splits every Eq. 16 pass over the ranks' GPUs (dist_space.py)."""
    import torch
    import torch.distributed as dist
    if i < 1:
        raise ValueError(f"need at least one outer iteration, got i={i}")
    if n < 0:
        raise ValueError(f"inner step count must be >= 0, got n={n}")
    if isinstance(seed, (np.random.Generator, np.random.BitGenerator)):
        raise ValueError("a distributed search needs a regenerable seed (int or SeedSequence)")
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = _device(dist)
    space = source.space
    if core_factory is None:
        table = _as_table(models, space)
        score_fn = None
        if shard_space:
            from .dist_space import score_configurations_sharded
            score_fn = score_configurations_sharded
        core = _profile_search_batches(space, source.arch, table, len(space), i=i, n=n,
                                       seed=seed, inst_reaction=inst_reaction,
                                       literal_sign=literal_sign, stop_indices=stop_indices,
                                       score_top_k=score_top_k, score_fn=score_fn)
    else:
        core = core_factory(space, source.arch, i=i, n=n, seed=seed,
                            inst_reaction=inst_reaction, literal_sign=literal_sign,
                            stop_indices=stop_indices, score_top_k=score_top_k)
    try:
        batch, profiled = next(core)
        while True:
            if profiled:
                got = _profile_step(dist, dev, source, batch[0], rank, profile_rank)
            else:
                got = _timed_batch(dist, dev, source, batch, rank, world)
            batch, profiled = core.send(got)
    except StopIteration as done:
        return done.value


def _profile_step(dist, dev, source, idx: int, rank: int, owner: int) -> List[Measurement]:
    import torch
    m = source.measure(idx, profiled=True) if rank == owner else None
    t = torch.from_numpy(_encode(m)).to(dev)
    dist.broadcast(t, src=owner)
    return [_decode(t.cpu().numpy())]


def _timed_batch(dist, dev, source, batch: List[int], rank: int,
                 world: int) -> List[Measurement]:
    import torch
    k = len(batch)
    per = -(-k // world)
    local = np.full(per, np.nan)
    for slot, pos in enumerate(range(rank, k, world)):
        local[slot] = source.measure(batch[pos], profiled=False).runtime_us
    t = torch.from_numpy(local).to(dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    gathered = [o.cpu().numpy() for o in outs]
    runtimes = [float(gathered[pos % world][pos // world]) for pos in range(k)]
    return [Measurement(runtime_us=r) for r in runtimes]
