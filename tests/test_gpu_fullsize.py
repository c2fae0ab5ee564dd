"""Full-size GPU parity on every BASELINE config (north star: "bit-exact quantization/
reorder and <= 2e-3 attention error against the oracle on all 5 configs").

* C1-C3: every layer -- assign for all layers, the packed bytes of one request and the
  attention of one request per layer (the request rotates over the layers).
* C4 (B = 64) and its window-size sweep S = 16/32/64/128: bytes of
  two requests and attention of two requests on 4 layers per S.
* C5: the packed bytes of all 4 requests on 4 layers, attention of one request on every
  layer.
* bench.py's exact launch path (bench.Workload + bench.build_step: CUDA-graph replay of
  the step with PDL-chained decodes, WQ_DECODE_EARLY) at the full C5 size, its outputs
  against the oracle on sampled (token, layer, request) triples.
* wq_shard_slots against the host plan (parallel.shard_plan) for G in {1, 2, 3, 8}.
The oracle runs on the sampled requests only (it needs ~0.4 s per C5 request-layer)."""
import math

import numpy as np
import pytest
import torch

from paper_2605_02262_b200 import configs, parallel, synth, wq

pytestmark = pytest.mark.gpu
ATTN_TOL = 2e-3


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    wq.load()


def rel_err(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return float((np.abs(got - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)).max())


def search(orc, cfg):
    """Scores + assign of every layer on the GPU; assign checked bit-exact against the
    oracle (on the GPU scores); sampled scores against the literal Eq.8 oracle."""
    m = cfg.model
    vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, "cuda")
    sc = wq.wq_window_scores(vis, txt, cfg.S)
    torch.cuda.synchronize()
    rng = np.random.default_rng(cfg.idx * 100 + cfg.S)
    vh, th = vis.cpu().numpy(), txt.cpu().numpy()
    for _ in range(4):
        b, w = int(rng.integers(cfg.B)), int(rng.integers(cfg.W))
        assert abs(sc[b, w].item() - orc.window_score(vh[b], th[b], cfg.S, w)) <= 1e-12
    del vis, txt, vh, th
    thr = orc.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
    g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, cfg.layers, g, wq.AssignOpts(cfg.budget, 1, 0))
    torch.cuda.synchronize()
    og = orc.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, list(cfg.widths))
    ob, orank, operm, oseg = orc.assign_bits(sc.cpu().numpy(), thr, og, cfg.budget, 1, 0)
    assert np.array_equal(bits.cpu().numpy(), ob)
    assert np.array_equal(rank.cpu().numpy(), orank)
    assert np.array_equal(perm.cpu().numpy(), operm)
    assert np.array_equal(seg.cpu().numpy(), oseg)
    return g, perm, seg


def layer_check(orc, cfg, g, perm_l, seg_l, layer, byte_reqs, attn_reqs, gran=0):
    """gran: WQ_GRAN_* of the packed image (1: the paper-literal groups, WQ_DECODE_GROUP)."""
    m = cfg.model
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, layer, "cuda")
    q = synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, layer, device="cuda")
    sm = 1 / math.sqrt(m.d)
    offs = wq.wq_layer_layout(g, seg_l, gran=gran)
    packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device="cuda")
    wq.wq_reorder_quantize_pack(K, V, 0, g, perm_l, seg_l, offs, packed, gran=gran)
    out = torch.empty((cfg.B, m.Hq, m.d), dtype=torch.float16, device="cuda")
    wq.wq_decode_attention(q, packed, offs, seg_l, g, kr, vr, rest_len, sm, out=out,
                           flags=wq.WQ_DECODE_GROUP if gran else 0)
    torch.cuda.synchronize()
    g1 = orc.geom(1, m.H, m.Hq, m.d, cfg.M, cfg.S, list(cfg.widths))
    pm, sg = perm_l.cpu().numpy(), seg_l.cpu().numpy()
    of = offs.cpu().numpy()
    for b in byte_reqs:
        opk, ooffs = orc.reorder_quantize_pack(K[b:b + 1].cpu().numpy(), V[b:b + 1].cpu().numpy(), 0, g1,
                                               pm[b:b + 1], sg[b:b + 1], gran=gran)
        n = int(ooffs[-1])
        got = packed[int(of[b * m.H]):int(of[b * m.H]) + n].cpu().numpy()
        assert np.array_equal(got, opk[:n]), (cfg.name, layer, b)
    for b in attn_reqs:
        lo, hi = int(of[b * m.H]), int(of[(b + 1) * m.H])
        ob = of[b * m.H:(b + 1) * m.H + 1] - of[b * m.H]
        ref = orc.decode_attention(q[b:b + 1].cpu().numpy(), packed[lo:hi].cpu().numpy(), ob, sg[b:b + 1],
                                   pm[b:b + 1], g1, kr[b:b + 1].cpu().numpy(), vr[b:b + 1].cpu().numpy(),
                                   rest_len[b:b + 1].cpu().numpy(), sm, gran=gran)
        e = rel_err(out[b:b + 1].float().cpu().numpy(), ref)
        assert e <= ATTN_TOL, (cfg.name, layer, b, e)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_every_layer(orc, name):
    cfg = configs.CONFIGS[name]
    g, perm, seg = search(orc, cfg)
    for l in range(cfg.layers):
        b = l % cfg.B
        layer_check(orc, cfg, g, perm[l], seg[l], l, [b], [(b + 1) % cfg.B])


@pytest.mark.parametrize("S", [16, 32, 64, 128])
def test_c4_window_sweep(orc, S):
    cfg = configs.c4(S)
    g, perm, seg = search(orc, cfg)
    for l in (0, 9, 18, cfg.layers - 1):
        layer_check(orc, cfg, g, perm[l], seg[l], l, [l % cfg.B, cfg.B - 1], [(3 * l + 1) % cfg.B, 0])


def test_c5_all_requests_bytes(orc):
    cfg = configs.CONFIGS["C5"]
    g, perm, seg = search(orc, cfg)
    for l in range(cfg.layers):
        byte_reqs = list(range(cfg.B)) if l in (0, 9, 18, cfg.layers - 1) else []
        layer_check(orc, cfg, g, perm[l], seg[l], l, byte_reqs, [l % cfg.B])


@pytest.mark.parametrize("name,S", [("C5", None), ("C4", 16), ("C4", 128), ("C2", None)])
def test_group_granularity_full_size(orc, name, S):
    """The paper-literal group quantizer (WQ_GRAN_GROUP, reading Q37) at full config size:
    bytes of every request and attention of one request on 3 layers."""
    cfg = configs.c4(S) if name == "C4" else configs.CONFIGS[name]
    g, perm, seg = search(orc, cfg)
    for l in (0, cfg.layers // 2, cfg.layers - 1):
        layer_check(orc, cfg, g, perm[l], seg[l], l, list(range(min(cfg.B, 4))), [l % cfg.B], gran=1)


def test_bench_launch_path_c5(orc):
    """bench.py's timed step itself (Workload + build_step: graph replay, PDL-chained
    decodes) at the full C5 size, 2 generated tokens; the outputs of sampled (token,
    layer, request) triples against the oracle over the step's own packed images, whose
    bytes are checked against the oracle for one request per sampled layer."""
    import bench
    cfg = configs.CONFIGS["C5"]
    m = cfg.model
    w = bench.Workload(cfg, torch.device("cuda", 0), n_gen=2)
    step = bench.build_step(w, None, torch.cuda.current_stream(), True, 1)
    w.out.zero_()
    step()
    torch.cuda.synchronize()
    g1 = orc.geom(1, m.H, m.Hq, m.d, cfg.M, cfg.S, list(cfg.widths))
    sm = 1 / math.sqrt(m.d)
    for (t, l, b) in [(0, 0, 0), (1, 0, 3), (0, 13, 1), (1, 27, 2), (1, 14, 0)]:
        pm, sg = w.perm[l].cpu().numpy(), w.seg[l].cpu().numpy()
        of = w.offs[l].cpu().numpy()
        lo, hi = int(of[b * m.H]), int(of[(b + 1) * m.H])
        pk = w.packed[l][lo:hi].cpu().numpy()
        if t == 0:
            opk, _ = orc.reorder_quantize_pack(w.K[l][b:b + 1].cpu().numpy(), w.V[l][b:b + 1].cpu().numpy(), 0, g1,
                                               pm[b:b + 1], sg[b:b + 1])
            assert np.array_equal(pk, opk[:hi - lo]), (l, b)
        ob = of[b * m.H:(b + 1) * m.H + 1] - of[b * m.H]
        ref = orc.decode_attention(w.q[t, l][b:b + 1].cpu().numpy(), pk, ob, sg[b:b + 1], pm[b:b + 1], g1,
                                   w.kr[l][b:b + 1].cpu().numpy(), w.vr[l][b:b + 1].cpu().numpy(),
                                   w.rest_len[t][b:b + 1].cpu().numpy(), sm)
        e = rel_err(w.out[t, l][b:b + 1].float().cpu().numpy(), ref)
        assert e <= ATTN_TOL, (t, l, b, e)
    # a second replay reproduces the step bit for bit (no state leaks between steps)
    first = w.out.clone()
    step()
    torch.cuda.synchronize()
    assert torch.equal(first, w.out)


def test_shard_slots_vs_host_plan(orc):
    """wq_shard_slots (device) = parallel.shard_plan (host) for G in {1, 2, 3, 8}: rank r
    keeps chunk r of every width segment; the G chunks partition the slot list."""
    cfg = configs.CONFIGS["C5"]
    m = cfg.model
    rng = np.random.default_rng(3)
    B, W = 5, 1568
    scores = torch.tensor(rng.uniform(0, 1, (B, W)), dtype=torch.float64, device="cuda")
    thr = orc.thresholds([0.5, 0.2], 2.0, 4)
    g = wq.geom(B, m.H, m.Hq, m.d, W * 32, 32, (2, 4, 8, 16))
    bits, rank, perm, seg = wq.wq_assign_bits(scores, thr, 2, g)
    for l in range(2):
        pm, sg = perm[l].cpu().numpy(), seg[l].cpu().numpy()
        for G in (1, 2, 3, 8):
            seen = [[] for _ in range(B)]
            for r in range(G):
                pr, sr = wq.wq_shard_slots(perm[l], seg[l], G, r)
                torch.cuda.synchronize()
                pr, sr = pr.cpu().numpy(), sr.cpu().numpy()
                for b in range(B):
                    ranges, local = parallel.shard_plan(sg[b], G, r)
                    assert list(sr[b]) == local, (G, r, b)
                    want = np.concatenate([pm[b, a:c] for a, c in ranges])
                    assert np.array_equal(pr[b, :local[-1]], want), (G, r, b)
                    seen[b].extend(want.tolist())
            for b in range(B):
                assert sorted(seen[b]) == sorted(pm[b].tolist())
