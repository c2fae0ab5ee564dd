"""World-size-2 gloo tests (CPU) of the multi-GPU host logic:
the sequence split of every width segment, the one all-gather of (m, l, o)
partials and the LSE merge give the unsplit attention; P1 batch shards cover
every request exactly once."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_02262_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(orc):
    rng = np.random.default_rng(3)
    B, H, Hq, d, S, W = 2, 2, 14, 64, 16, 11
    M = W * S
    K = (rng.standard_normal((B, H, M, d)) * 1.5 + rng.standard_normal((1, H, 1, d)) * 3).astype(np.float16)
    V = rng.standard_normal((B, H, M, d)).astype(np.float16)
    q = rng.standard_normal((B, Hq, d)).astype(np.float16)
    kr = rng.standard_normal((B, H, 9, d)).astype(np.float16)
    vr = rng.standard_normal((B, H, 9, d)).astype(np.float16)
    rest_len = np.array([9, 4], np.int32)
    g = orc.geom(B, H, Hq, d, M, S, [2, 4, 8, 16])
    sims = rng.uniform(0, 1, (B, W))
    thr = orc.thresholds([0.5], 2.0, 4)
    bits, rank, perm, seg = orc.assign_bits(sims, thr, g)
    return g, K, V, q, kr, vr, rest_len, perm[0], seg[0]


def _worker(rank, world, port, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    g, K, V, q, kr, vr, rest_len, perm, seg = _case(oracle)
    sm = 1 / math.sqrt(64)
    B, W = perm.shape
    perm_r = np.zeros_like(perm)
    seg_r = np.zeros_like(seg)
    for b in range(B):
        ranges, local = parallel.shard_plan(seg[b], world, rank)
        slots = [s for a, e in ranges for s in range(a, e)]
        perm_r[b, :len(slots)] = perm[b, slots]
        seg_r[b] = local
    pk, of = oracle.reorder_quantize_pack(K, V, 0, g, perm_r, seg_r)
    rl = rest_len if rank == 0 else np.zeros_like(rest_len)
    _, part = oracle.decode_attention(q, pk, of, seg_r, perm_r, g, kr, vr, rl, sm, want_partial=True)
    gathered = parallel.all_gather_partials(torch.from_numpy(part))
    if rank == 0:
        merged = oracle.merge(gathered.numpy())
        pk0, of0 = oracle.reorder_quantize_pack(K, V, 0, g, perm, seg)
        full = oracle.decode_attention(q, pk0, of0, seg, perm, g, kr, vr, rest_len, sm)
        np.save(result_path, np.array([np.max(np.abs(merged - full))]))
    dist.barrier()
    dist.destroy_process_group()


def test_sequence_split_allgather_merge_gloo(orc, tmp_path):
    out = str(tmp_path / "err.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert np.load(out)[0] < 1e-12


def test_shard_plan_partitions_every_segment():
    rng = np.random.default_rng(0)
    for _ in range(50):
        counts = rng.integers(0, 40, 4)
        seg = np.concatenate([[0], np.cumsum(counts)])
        for G in (1, 2, 3, 8):
            seen = []
            for r in range(G):
                ranges, local = parallel.shard_plan(seg, G, r)
                for k, (a, e) in enumerate(ranges):
                    assert seg[k] <= a <= e <= seg[k + 1]
                    assert abs((e - a) - counts[k] / G) < 1 + 1e-9       # balanced to one slot
                    seen += list(range(a, e))
                assert local[-1] == sum(e - a for a, e in ranges)
            assert sorted(seen) == list(range(seg[-1]))


def test_batch_shard_covers_requests():
    for B in (1, 4, 16, 64):
        for G in (1, 2, 4, 8):
            got = []
            for r in range(G):
                a, e = parallel.batch_shard(B, G, r)
                got += list(range(a, e))
            assert got == list(range(B))


def test_unit_shard_partitions_request_head_units():
    """P1 over (request, kv-head) units: the ranks' (b, h) ranges partition the B*H units
    (C3 at 2/4/8 GPUs = whole requests; C5 (B=4, H=4) at 8 GPUs = two heads of one request)."""
    for B, H, G in [(16, 4, 2), (16, 4, 4), (16, 4, 8), (4, 4, 8), (4, 4, 16), (8, 2, 16), (64, 4, 8), (1, 4, 2),
                    (2, 4, 8)]:
        seen = []
        for r in range(G):
            b0, b1, h0, h1 = parallel.unit_shard(B, H, G, r)
            assert 0 <= b0 < b1 <= B and 0 <= h0 < h1 <= H
            if b1 - b0 > 1:
                assert (h0, h1) == (0, H)
            seen += [(b, h) for b in range(b0, b1) for h in range(h0, h1)]
        assert sorted(seen) == [(b, h) for b in range(B) for h in range(H)], (B, H, G)
        assert len(seen) == len(set(seen))
    with pytest.raises(ValueError):
        parallel.unit_shard(3, 4, 5, 3)          # units [7, 9) straddle requests 1 and 2
