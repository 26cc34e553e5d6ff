"""Multi-GPU plumbing: one process per GPU, torch.distributed for the few
host-side exchanges.  The data path never crosses ranks:

* block-range sharding (configs 3 and 5): rank g owns overlap-save blocks
  [P*g/G, P*(g+1)/G) of one long signal, reads its input range plus the N'+1-sample halo
  (`shard`), runs `conv_execute_blocks` and writes a disjoint output range;
* signal sharding (config 4): rank g owns database signals [n*g/G, n*(g+1)/G), computes
  per-signal (score, lag) with `conv_xcorr_max`, and only the scores are gathered
  (`gather_best_match`, NCCL all_gather of 16 B/signal).
"""
from __future__ import annotations

from . import binding


def shard(L, N, W_block, mode, rank, world):
    """Blocks, input range (with halo) and output range of `rank` (host-only, C ABI)."""
    return binding.shard_range(L, N, W_block, mode, rank, world)


def signal_range(n_signals, rank, world):
    return n_signals * rank // world, n_signals * (rank + 1) // world


def gather_best_match(scores, lags, first_signal, group=None):
    """All ranks learn the database winner: the largest score, ties to the smallest global
    signal index (reading C17).  `scores` (float64) / `lags` (int64) are this rank's
    per-signal results for signals first_signal .. first_signal+len-1 (any device the
    process group's backend supports).  Returns (signal, score, lag)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = scores.device
    n = torch.tensor([scores.numel()], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    m = int(max(int(x.item()) for x in ns))
    pad = m - scores.numel()
    packed = torch.stack([torch.cat([scores.double(), torch.full((pad,), float("-inf"), device=dev, dtype=torch.float64)]),
                          torch.cat([lags.double(), torch.zeros(pad, device=dev, dtype=torch.float64)]),
                          torch.cat([torch.arange(first_signal, first_signal + scores.numel(), device=dev,
                                                  dtype=torch.float64),
                                     torch.full((pad,), float("inf"), device=dev, dtype=torch.float64)])])
    parts = [torch.zeros_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    allp = torch.cat(parts, dim=1).cpu()
    best = float("-inf")
    win = None
    for j in range(allp.shape[1]):
        sc, lg, idx = float(allp[0, j]), int(allp[1, j]), allp[2, j]
        if idx == float("inf"):
            continue
        idx = int(idx)
        if sc > best or (sc == best and win is not None and idx < win[0]):
            best, win = sc, (idx, sc, lg)
    return win
