"""Multi-GPU plumbing: one process per GPU, torch.distributed for the few
host-side exchanges.  The data path never crosses ranks:

* block-range sharding (configs 3 and 5): rank g owns overlap-save blocks
  [P*g/G, P*(g+1)/G) of one long signal, reads its input range plus the N'+1-sample halo
  (`shard`), runs `conv_execute_blocks` and writes a disjoint output range;
* signal sharding (config 4): rank g owns database signals [n*g/G, n*(g+1)/G), computes
  per-signal (score, lag) with `conv_xcorr_max`, reduces them to its winner on the device
  (`conv_best_match`), and only the winners are gathered (`gather_best_match`, NCCL all_gather
  of 24 B per rank).
"""
from __future__ import annotations

from . import binding


def shard(L, N, W_block, mode, rank, world):
    """Blocks, input range (with halo) and output range of `rank` (host-only, C ABI)."""
    return binding.shard_range(L, N, W_block, mode, rank, world)


def signal_range(n_signals, rank, world):
    return n_signals * rank // world, n_signals * (rank + 1) // world


def _device_best_match(out, n, scores=None, lags=None, cand=None, first=0):
    binding.best_match(out, n, score_dev=scores, lag_dev=lags, cand_dev=cand, first_index=first)


def gather_best_match(scores, lags, first_signal, group=None, reduce=None):
    """All ranks learn the database winner: the largest score, ties to the smallest global
    signal index (reading C17).  `scores` (float64) / `lags` (int64) are this rank's per-signal
    results for signals first_signal .. first_signal+len-1.  Each rank reduces its own signals to
    one candidate {score, lag, index} on the device (conv_best_match), the world's candidates are
    all-gathered (NCCL: one 3-double tensor per rank) and reduced again by the same kernel:
    stream-ordered, no host round trip until the caller reads the result.  `reduce` replaces the
    device kernel (CPU / gloo tests of this host logic).  Returns the tensor {score, lag, index}."""
    import torch
    import torch.distributed as dist

    red = reduce or _device_best_match
    world = dist.get_world_size(group)
    dev = scores.device
    local = torch.empty(3, dtype=torch.float64, device=dev)
    red(local, scores.numel(), scores=scores, lags=lags, first=first_signal)
    if dist.get_backend(group) == "nccl":
        cand = torch.empty(3 * world, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(cand, local, group=group)
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local, group=group)
        cand = torch.cat(parts)
    best = torch.empty(3, dtype=torch.float64, device=dev)
    red(best, world, cand=cand)
    return best


def best_match_tuple(best):
    """(signal, score, lag) of a gather_best_match result (reads it back to the host)."""
    b = best.cpu().tolist()
    return int(b[2]), float(b[0]), int(b[1])
