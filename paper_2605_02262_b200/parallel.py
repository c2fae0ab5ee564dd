"""Multi-GPU plumbing of the hot path.

* P1 -- independent units: (request, kv-head) units are sharded across ranks with
  no collective on the data path (unit_shard: whole requests = batch_shard, or kv heads of
  one request when there are more ranks than requests).
* P2 -- long-video sequence split: rank r of G keeps chunk r of every width
  segment of the reordered slot list (``wq_shard_slots`` on the device; the same
  bounds as ``segment_chunk`` here), decodes it into (m, l, o) partials, and the
  partials are exchanged with ONE all-gather and merged by log-sum-exp
  (``wq_merge_partials``).

* P2 fused: ``PeerMerge`` sets up one symmetric buffer per rank
  (cudaMalloc, CUDA IPC handles exchanged over the process group, peers mapped with
  peer access over NVLink) for ``wq_decode_attention_peer``, whose kernel exchanges the
  partials through peer memory and merges them itself -- no NCCL call, no merge kernel.

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


def unit_shard(B: int, H: int, G: int, r: int) -> tuple[int, int, int, int]:
    """P1 over (request, kv-head) units (north star: "partitioned ... by KV head and batch"):
    rank r takes the b-major unit range [U r/G, U (r+1)/G), U = B*H, returned as
    (b0, b1, h0, h1) = requests [b0, b1) x kv heads [h0, h1).  Supported when every rank's
    range is whole requests (then h0, h1 = 0, H: batch sharding) or kv heads of ONE request
    (head sharding, e.g. B = 4, H = 4 on 8 GPUs: two heads each) -- the ranges a [B][H]
    geometry slice can express.  Units are independent: no collective on the data path."""
    U = B * H
    u0, u1 = (U * r) // G, (U * (r + 1)) // G
    if u1 <= u0:
        raise ValueError(f"rank {r} of {G} gets no (request, head) unit (B*H = {U})")
    if u0 % H == 0 and u1 % H == 0:
        return u0 // H, u1 // H, 0, H
    if u0 // H == (u1 - 1) // H:
        b = u0 // H
        return b, b + 1, u0 - b * H, u1 - b * H
    raise ValueError(f"units [{u0}, {u1}) of rank {r} span partial requests (B={B}, H={H}, G={G})")


def all_gather_partials(part: torch.Tensor, group=None) -> torch.Tensor:
    """[B][Hq][d+2] fp32 partials of every rank -> [G][B][Hq][d+2] (one collective)."""
    G = dist.get_world_size(group)
    out = torch.empty((G, *part.shape), dtype=part.dtype, device=part.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, part.contiguous(), group=group)
    else:                                  # gloo (CPU tests): list form
        dist.all_gather(list(out.unbind(0)), part.contiguous(), group=group)
    return out


def _cudart():
    from cuda.bindings import runtime as cudart
    return cudart


def _ck(res):
    err = res[0] if isinstance(res, tuple) else res
    if int(err) != 0:
        raise RuntimeError(f"CUDA runtime error {err}")
    return res[1] if isinstance(res, tuple) and len(res) > 1 else None


class PeerMerge:
    """Symmetric buffers of the fused cross-GPU LSE merge (include/wq.h wq_peer_buffer_bytes).

    Every rank cudaMallocs one zero-filled buffer, publishes its IPC handle with
    all_gather_object, and maps the peers' buffers (cudaIpcOpenMemHandle, lazy peer
    access).  ``ptrs`` is the int64 device tensor of the G buffer addresses (entry rank =
    own buffer); ``next_epoch()`` numbers the calls 1, 2, ... identically on all ranks."""

    def __init__(self, g, group=None, device=None):
        from paper_2605_02262_b200 import wq
        self.G = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.bytes = wq.wq_peer_buffer_bytes(g, self.G)
        self.err_off = wq.wq_peer_error_offset(g, self.G)
        rt = _cudart()
        self.local = int(_ck(rt.cudaMalloc(self.bytes)))
        _ck(rt.cudaMemset(self.local, 0, self.bytes))
        self.opened = []
        addrs = [0] * self.G
        addrs[self.rank] = self.local
        if self.G > 1:
            h = _ck(rt.cudaIpcGetMemHandle(self.local))
            handles = [None] * self.G
            dist.all_gather_object(handles, bytes(h.reserved), group=group)
            for p in range(self.G):
                if p == self.rank:
                    continue
                hp = rt.cudaIpcMemHandle_t()
                hp.reserved = handles[p]
                ptr = int(_ck(rt.cudaIpcOpenMemHandle(hp, rt.cudaIpcMemLazyEnablePeerAccess)))
                self.opened.append(ptr)
                addrs[p] = ptr
        _ck(rt.cudaDeviceSynchronize())
        self.ptrs = torch.tensor(addrs, dtype=torch.int64, device=dev)
        self.epoch = 0
        if self.G > 1:
            dist.barrier(group=group)

    def timed_out(self) -> bool:
        """True if a wait of this rank's decode kernels for its peers timed out (the
        outputs of that call are invalid)."""
        import numpy as np
        rt = _cudart()
        v = np.zeros(1, np.uint32)
        _ck(rt.cudaDeviceSynchronize())
        _ck(rt.cudaMemcpy(v.ctypes.data, self.local + self.err_off, 4, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost))
        return bool(v[0])

    def next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch

    def close(self):
        rt = _cudart()
        for p in self.opened:
            rt.cudaIpcCloseMemHandle(p)
        self.opened = []
        if self.local:
            rt.cudaFree(self.local)
            self.local = 0
