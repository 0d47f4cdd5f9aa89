"""Configuration-space sharding of one search over the GPUs of one box
(north_star: "the configuration space is sharded across the 8 GPUs";
SURVEY section 8e).

Eq. 16 (``score_configurations``, reference ``search.py:89-141``) is
elementwise over configurations.  Each rank therefore scores a contiguous
shard ``[lo, hi)`` of the space on its own GPU: every configuration outside
the shard is masked as explored for the device scorer (``k_score_single``
reads no table entry and does no arithmetic for an explored configuration),
and one all-gather assembles the raw-score vector in index order.  The raw
scores are bit-identical to the unsharded ones, so the rest of an outer
iteration -- Eq. 17, the n certified draws, the expert system -- runs
replicated on every rank from the same Generator, and every rank follows the
reference's trajectory.

The only data-path exchange is that all-gather: N float64 per outer
iteration (1.6 MB at N = 205,216).  At the paper's sizes one GPU scores a
whole space in microseconds, so this is not the scaling axis (DESIGN.md
section 6); repetition sharding (``dist.py``) and the live-candidate split
(``dist_live.py``) are.  ``dist_live.run_profile_search_distributed(...,
shard_space=True)`` combines it with the live-candidate split.
"""

from typing import Callable, Dict, Iterable, Optional, Tuple

import numpy as np

from .search import ScoreVector, _explored_mask, score_configurations


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Rank ``rank``'s contiguous share of ``n`` configurations (the first
    ``n % world`` ranks take one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _device(dist, group):
    import torch
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def score_configurations_sharded(models, c_profile, delta: Dict[str, float], space,
                                 explored: Iterable[int], literal_sign: bool = False,
                                 score_top_k: Optional[int] = None, *, group=None,
                                 scorer: Optional[Callable] = None) -> ScoreVector:
    """``score_configurations`` with the configurations sharded over the
    process group (same arguments, same result on every rank).

    ``scorer(models, c_profile, delta, space, shard_explored, literal_sign)``
    replaces the device scorer (tests drive the protocol with a host
    stand-in); it returns the raw-score vector of the whole space, of which
    only the shard's entries are used."""
    import torch
    import torch.distributed as dist
    if score_top_k is not None:
        raise ValueError("score_top_k needs the whole space's distances on one rank; "
                         "it is not supported with a sharded space")
    n = len(space)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    lo, hi = shard_bounds(n, world, rank)
    full_mask = _explored_mask(explored, n)
    shard_mask = full_mask.copy()
    shard_mask[:lo] = True
    shard_mask[hi:] = True
    if scorer is None:
        raw = score_configurations(models, c_profile, delta, space, shard_mask,
                                   literal_sign=literal_sign).raw
    else:
        raw = np.asarray(scorer(models, c_profile, delta, space, shard_mask, literal_sign),
                         dtype=np.float64)
    per = -(-n // world)
    dev = _device(dist, group)
    local = torch.zeros(per, dtype=torch.float64, device=dev)
    local[:hi - lo] = torch.from_numpy(np.ascontiguousarray(raw[lo:hi])).to(dev)
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    out = np.empty(n, dtype=np.float64)
    for r, t in enumerate(parts):
        a, b = shard_bounds(n, world, r)
        out[a:b] = t[:b - a].cpu().numpy()
    return ScoreVector(raw=out, explored=full_mask)
