"""Multi-GPU plumbing of the hot path.

* P1 -- independent units: requests (and kv heads) are sharded across ranks with
  no collective on the data path (batch_shard).
* P2 -- long-video sequence split: rank r of G keeps chunk r of every width
  segment of the reordered slot list (``wq_shard_slots`` on the device; the same
  bounds as ``segment_chunk`` here), decodes it into (m, l, o) partials, and the
  partials are exchanged with ONE all-gather and merged by log-sum-exp
  (``wq_merge_partials``).

Only host-side orchestration lives here; every arithmetic step runs in libwq.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def segment_chunk(lo: int, hi: int, G: int, r: int) -> tuple[int, int]:
    """Slots [lo + n*r//G, lo + n*(r+1)//G) of a segment [lo, hi) for rank r (n = hi - lo)."""
    n = hi - lo
    return lo + (n * r) // G, lo + (n * (r + 1)) // G


def shard_plan(seg_off_b, G: int, r: int):
    """Host mirror of wq_shard_slots for one request: (slot ranges, rank-local seg_off)."""
    ranges, local = [], [0]
    for k in range(4):
        a, b = segment_chunk(int(seg_off_b[k]), int(seg_off_b[k + 1]), G, r)
        ranges.append((a, b))
        local.append(local[-1] + (b - a))
    return ranges, local


def batch_shard(B: int, G: int, r: int) -> tuple[int, int]:
    """Contiguous request range of rank r under P1 (requests are independent units)."""
    return (B * r) // G, (B * (r + 1)) // G


def all_gather_partials(part: torch.Tensor, group=None) -> torch.Tensor:
    """[B][Hq][d+2] fp32 partials of every rank -> [G][B][Hq][d+2] (one collective)."""
    G = dist.get_world_size(group)
    out = torch.empty((G, *part.shape), dtype=part.dtype, device=part.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, part.contiguous(), group=group)
    else:                                  # gloo (CPU tests): list form
        dist.all_gather(list(out.unbind(0)), part.contiguous(), group=group)
    return out
