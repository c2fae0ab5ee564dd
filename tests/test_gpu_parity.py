"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Integer outputs (ranks, bits, perms, segment offsets, packed
bytes) must be bit-exact; scores within 1e-12 absolute (Q6); attention within
2e-3 max row-wise relative error (north star, Q30)."""
import math

import numpy as np
import pytest
import torch

from paper_2605_02262_b200 import configs, synth
from paper_2605_02262_b200 import wq

pytestmark = pytest.mark.gpu

ATTN_TOL = 2e-3


def rel_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    num = np.abs(got - ref).max(axis=-1)
    den = np.maximum(np.abs(ref).max(axis=-1), 1e-6)
    return float((num / den).max())


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    wq.load()


def ogeom(orc, g):
    return orc.geom(g.B, g.H, g.Hq, g.d, g.M, g.S, list(g.widths)[:g.n_widths])


def run_layer(g, K, V, kr, vr, rest_len, perm, seg, q, sm, partial=False):
    """GPU path for one layer: layout -> quantize -> decode."""
    dev = K.device
    offs = wq.wq_layer_layout(g, seg)
    total = int(offs[-1].item())
    packed = torch.zeros(max(total, 16), dtype=torch.uint8, device=dev)
    wq.wq_reorder_quantize_pack(K, V, 0, g, perm, seg, offs, packed)
    out = torch.empty((g.B, g.Hq, g.d), dtype=torch.float16, device=dev)
    part = torch.empty((g.B, g.Hq, g.d + 2), dtype=torch.float32, device=dev) if partial else None
    wq.wq_decode_attention(q, packed, offs, seg, g, kr, vr, rest_len, sm, out=out, partial=part)
    torch.cuda.synchronize()
    return offs, packed, out, part


def small_case(seed, B=2, H=2, Hq=14, d=64, S=16, W=9, tail=5, R=21, widths=(2, 4, 8, 16), s=0.5):
    torch.manual_seed(seed)
    M = W * S + tail
    K, V = synth.kv_layer(B, H, M, d, S, seed, 0, "cuda")
    kr, vr = synth.rest_layer(B, H, R, d, seed, 0, "cuda")
    rest_len = torch.tensor([R - 3 * b for b in range(B)], dtype=torch.int32, device="cuda")
    q = synth.queries(B, Hq, H, d, seed, 0, device="cuda")
    vis, txt = synth.embeddings(B, M, 8, 64, S, seed, "cuda")
    g = wq.geom(B, H, Hq, d, M, S, widths)
    return dict(g=g, K=K, V=V, kr=kr, vr=vr, rest_len=rest_len, q=q, vis=vis, txt=txt, s=s)


# ---------------------------------------------------------------------------------------
def test_scores_parity(orc):
    for (B, M, N, D, S) in [(2, 16 * 9 + 5, 8, 64, 16), (1, 1568, 32, 896, 64), (3, 700, 5, 3584, 32)]:
        vis, txt = synth.embeddings(B, M, N, D, S, 123 + D, "cuda")
        sc = wq.wq_window_scores(vis, txt, S)
        torch.cuda.synchronize()
        ref = orc.window_scores(vis.cpu().numpy(), txt.cpu().numpy(), S)
        assert np.max(np.abs(sc.cpu().numpy() - ref)) <= 1e-12


def _assign_both(orc, scores_gpu, thr, g, budget=0.0, pin=1, vote=0):
    L = thr.shape[0]
    opts = wq.AssignOpts(budget, pin, vote)
    bits, rank, perm, seg = wq.wq_assign_bits(scores_gpu, thr, L, g, opts)
    torch.cuda.synchronize()
    ob, orank, operm, oseg = orc.assign_bits(scores_gpu.cpu().numpy(), thr, ogeom(orc, g), budget, pin, vote)
    return (bits.cpu().numpy(), rank.cpu().numpy(), perm.cpu().numpy(), seg.cpu().numpy()), (ob, orank, operm, oseg)


@pytest.mark.parametrize("widths,budget,pin,vote", [
    ((2, 4, 16), 0.0, 1, 0), ((2, 4, 8, 16), 0.0, 1, 0), ((2, 4, 8), 0.0, 1, 0),
    ((2, 4, 8, 16), 4.0, 1, 0), ((2, 4, 8, 16), 3.0, 0, 0), ((2, 4, 16), 0.0, 1, 1),
    ((2, 4, 8, 16), 4.5, 1, 1), ((4, 8), 0.0, 1, 0), ((16,), 0.0, 1, 0)])
def test_assign_parity(orc, widths, budget, pin, vote):
    B, W, S = 5, 197, 16
    rng = np.random.default_rng(len(widths) * 7 + int(budget))
    scores = rng.uniform(0.0, 0.95, (B, W))
    scores[1, 10:20] = scores[1, 30]                       # exact ties -> index order (Q7)
    scores[2, :] = np.round(scores[2, :], 1)               # many ties and threshold hits
    sc = torch.tensor(scores, dtype=torch.float64, device="cuda")
    s_prof = [0.5, 0.3, 0.9, 0.05, 0.5]
    thr = orc.thresholds(s_prof, 2.0, len(widths))
    g = wq.geom(B, 2, 14, 64, W * S + 3, S, widths)
    gpu, ref = _assign_both(orc, sc, thr, g, budget, pin, vote)
    for a, b, name in zip(gpu, ref, ("bits", "rank", "perm", "seg_off")):
        assert np.array_equal(a, b), name


def test_assign_parity_large_W(orc):
    """C5 geometry: W = 1568 windows, 28 layers, budget on."""
    cfg = configs.CONFIGS["C5"]
    vis, txt = synth.embeddings(2, cfg.M, 32, 256, cfg.S, cfg.seed, "cuda")
    sc = wq.wq_window_scores(vis, txt, cfg.S)
    thr = orc.thresholds([0.5] * 27 + [0.1], 2.0, 4)
    g = wq.geom(2, 4, 28, 128, cfg.M, cfg.S, cfg.widths)
    for budget in (0.0, 3.5):
        gpu, ref = _assign_both(orc, sc, thr, g, budget)
        for a, b in zip(gpu, ref):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("d,S,W,tail", [(64, 16, 9, 5), (64, 32, 5, 0), (128, 32, 6, 7), (128, 64, 3, 0),
                                        (128, 128, 2, 3), (64, 128, 2, 0), (128, 16, 11, 0)])
def test_quantize_pack_bit_exact(orc, d, S, W, tail):
    c = small_case(10 + d + S, d=d, S=S, W=W, tail=tail, Hq=4 if d == 64 else 28, H=2 if d == 64 else 4)
    g = c["g"]
    sc = wq.wq_window_scores(c["vis"], c["txt"], S)
    thr = orc.thresholds([0.4], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
    offs, packed, _, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0], c["q"],
                                   1 / math.sqrt(d))
    opk, ooffs = orc.reorder_quantize_pack(c["K"].cpu().numpy(), c["V"].cpu().numpy(), 0, ogeom(orc, g),
                                           perm[0].cpu().numpy(), seg[0].cpu().numpy())
    assert np.array_equal(offs.cpu().numpy(), ooffs)
    n = int(ooffs[-1])
    assert np.array_equal(packed.cpu().numpy()[:n], opk[:n])


def test_quantize_all_classes_present(orc):
    """Force every width class (and a permuted, non-identity slot order)."""
    c = small_case(77, d=128, S=32, W=8, tail=0, Hq=28, H=4, B=1)
    g = c["g"]
    bits = [16, 2, 8, 4, 2, 16, 8, 4]
    order = [i for k in (2, 4, 8, 16) for i, b in enumerate(bits) if b == k]
    perm = torch.tensor([order], dtype=torch.int32, device="cuda")
    seg = torch.tensor([[0, 2, 4, 6, 8]], dtype=torch.int32, device="cuda")
    offs, packed, out, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm, seg, c["q"],
                                     1 / math.sqrt(128))
    opk, ooffs = orc.reorder_quantize_pack(c["K"].cpu().numpy(), c["V"].cpu().numpy(), 0, ogeom(orc, g),
                                           perm.cpu().numpy(), seg.cpu().numpy())
    assert np.array_equal(packed.cpu().numpy()[:int(ooffs[-1])], opk[:int(ooffs[-1])])


# ---------------------------------------------------------------------------------------
def _decode_ref(orc, c, g, offs, packed, perm, seg, sm):
    return orc.decode_attention(c["q"].cpu().numpy(), packed.cpu().numpy(), offs.cpu().numpy(),
                                seg.cpu().numpy(), perm.cpu().numpy(), ogeom(orc, g), c["kr"].cpu().numpy(),
                                c["vr"].cpu().numpy(), c["rest_len"].cpu().numpy(), sm, want_partial=True)


@pytest.mark.parametrize("d,S,W,tail,B,H,Hq", [(64, 16, 9, 5, 2, 2, 14), (64, 32, 17, 0, 3, 2, 14),
                                               (128, 32, 12, 7, 2, 4, 28), (128, 64, 5, 0, 1, 4, 28),
                                               (128, 128, 3, 9, 2, 2, 8), (64, 64, 6, 1, 2, 1, 5),
                                               (128, 16, 30, 0, 4, 4, 28)])
def test_decode_parity(orc, d, S, W, tail, B, H, Hq):
    c = small_case(200 + d + S + W, d=d, S=S, W=W, tail=tail, B=B, H=H, Hq=Hq)
    g = c["g"]
    sc = wq.wq_window_scores(c["vis"], c["txt"], S)
    thr = orc.thresholds([0.45], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
    sm = 1 / math.sqrt(d)
    offs, packed, out, part = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0],
                                        c["q"], sm, partial=True)
    ref, rpart = _decode_ref(orc, c, g, offs, packed, perm[0], seg[0], sm)
    assert rel_err(out.float().cpu().numpy(), ref) <= ATTN_TOL
    # partial (m, l, o): compare normalized output and the log-sum-exp
    p = part.double().cpu().numpy()
    assert rel_err(p[..., 2:] / p[..., 1:2], ref) <= ATTN_TOL
    lse = p[..., 0] + np.log(p[..., 1])
    rlse = rpart[..., 0] + np.log(rpart[..., 1])
    assert np.max(np.abs(lse - rlse)) < 1e-3


def test_decode_all16_equals_bruteforce(orc):
    """North star: all windows at 16 bits -> fp64 brute-force attention."""
    c = small_case(31, d=128, S=32, W=10, tail=3, B=2, H=4, Hq=28, widths=(16,))
    g = c["g"]
    W = 10
    perm = torch.arange(W, dtype=torch.int32, device="cuda").repeat(2, 1)
    seg = torch.tensor([[0, 0, 0, 0, W]] * 2, dtype=torch.int32, device="cuda")
    sm = 1 / math.sqrt(128)
    _, _, out, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm, seg, c["q"], sm)
    win = np.tile(np.arange(W, dtype=np.int32), (2, 1))
    ref = orc.bruteforce_attention(c["q"].cpu().numpy(), c["K"].cpu().numpy(), c["V"].cpu().numpy(), 0,
                                   ogeom(orc, g), win, np.array([W, W], np.int32), c["kr"].cpu().numpy(),
                                   c["vr"].cpu().numpy(), c["rest_len"].cpu().numpy(), sm)
    assert rel_err(out.float().cpu().numpy(), ref) <= ATTN_TOL


def test_decode_edge_cases(orc):
    """Empty rest, rest-only (no windows), one token, ragged rest tiles."""
    c = small_case(41, d=64, S=16, W=4, tail=0, B=3, H=2, Hq=14)
    g = c["g"]
    sm = 0.125
    sc = wq.wq_window_scores(c["vis"], c["txt"], 16)
    thr = orc.thresholds([0.5], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
    for rl in ([0, 0, 0], [1, 17, 20], [16, 15, 21]):        # each <= R_max = 21
        c["rest_len"] = torch.tensor(rl, dtype=torch.int32, device="cuda")
        offs, packed, out, part = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0],
                                            c["q"], sm, partial=True)
        ref, _ = _decode_ref(orc, c, g, offs, packed, perm[0], seg[0], sm)
        assert rel_err(out.float().cpu().numpy(), ref) <= ATTN_TOL
    # no windows at all: only rest tokens (request 1 has a single token)
    seg0 = torch.zeros((3, 5), dtype=torch.int32, device="cuda")
    c["rest_len"] = torch.tensor([5, 1, 21], dtype=torch.int32, device="cuda")
    offs, packed, out, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg0, c["q"], sm)
    ref, _ = _decode_ref(orc, c, g, offs, packed, perm[0], seg0, sm)
    assert rel_err(out.float().cpu().numpy(), ref) <= ATTN_TOL
    # single rest token -> output equals v_0 exactly up to fp16 rounding
    assert np.allclose(out[1].float().cpu().numpy(), c["vr"][1, :, 0].float().cpu().numpy().repeat(7, 0),
                       atol=2e-3, rtol=2e-3)


def test_merge_partials_parity(orc):
    """Sequence split (§8(e)): two shards' partials merged on the GPU = unsplit."""
    c = small_case(55, d=128, S=32, W=14, tail=0, B=2, H=4, Hq=28)
    g = c["g"]
    sm = 1 / math.sqrt(128)
    sc = wq.wq_window_scores(c["vis"], c["txt"], 32)
    thr = orc.thresholds([0.45], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
    _, _, full, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0], c["q"], sm)
    parts = []
    for r in range(2):
        pl, sl = [], []
        for b in range(2):
            so = seg[0, b].cpu().numpy()
            pb = perm[0, b].cpu().numpy()
            slots, s5 = [], []
            for k in range(4):
                lo, hi = so[k], so[k + 1]
                mid = lo + (hi - lo) // 2
                s5.append(len(slots))
                slots += list(pb[lo:mid] if r == 0 else pb[mid:hi])
            s5.append(len(slots))
            pl.append(slots + [0] * (14 - len(slots)))
            sl.append(s5)
        pr = torch.tensor(pl, dtype=torch.int32, device="cuda")
        sr = torch.tensor(sl, dtype=torch.int32, device="cuda")
        rl = c["rest_len"] if r == 0 else torch.zeros_like(c["rest_len"])
        _, _, _, part = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], rl, pr, sr, c["q"], sm, partial=True)
        parts.append(part)
    merged = wq.wq_merge_partials(torch.stack(parts), g)
    torch.cuda.synchronize()
    ref = orc.merge(torch.stack(parts).double().cpu().numpy())
    assert rel_err(merged.float().cpu().numpy(), ref) <= 1e-3
    assert rel_err(merged.float().cpu().numpy(), full.float().cpu().numpy()) <= ATTN_TOL


def test_abi_errors():
    g = wq.geom(1, 2, 14, 96, 64, 16, (2, 4))
    with pytest.raises(wq.WQError) as e:
        wq.wq_decode_workspace(g)
    assert e.value.status == wq.WQ_EUNSUPPORTED
    g = wq.geom(1, 2, 14, 64, 64, 16, (4, 2))
    sc = torch.zeros((1, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(wq.WQError):
        wq.wq_assign_bits(sc, np.zeros((1, 1)), 1, g)
    g = wq.geom(1, 2, 14, 64, 64, 16, (2, 4, 8, 16))
    with pytest.raises(wq.WQError) as e:
        wq.wq_assign_bits(sc, np.zeros((1, 3)), 1, g, wq.AssignOpts(2.0, 1, 0))
    assert e.value.status == wq.WQ_EBUDGET


# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_config_layer_parity(orc, name):
    """One layer of each config at FULL size, in the launch configuration bench.py
    times: scores (sampled windows), assign (all), packed bytes (one request, all
    heads) and attention (sampled (b, h) units through the oracle)."""
    cfg = configs.CONFIGS[name]
    m = cfg.model
    B = cfg.B
    layer = cfg.layers - 1
    vis, txt = synth.embeddings(B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, "cuda")
    sc = wq.wq_window_scores(vis, txt, cfg.S)
    torch.cuda.synchronize()
    rng = np.random.default_rng(cfg.idx)
    vh, th = vis.cpu().numpy(), txt.cpu().numpy()
    for _ in range(6):
        b, w = int(rng.integers(B)), int(rng.integers(cfg.W))
        assert abs(sc[b, w].item() - orc.window_score(vh[b], th[b], cfg.S, w)) <= 1e-12
    thr = orc.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
    g = wq.geom(B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    gpu, ref = _assign_both(orc, sc, thr, g, cfg.budget)
    for a, b_ in zip(gpu, ref):
        assert np.array_equal(a, b_)
    perm = torch.tensor(ref[2][layer], device="cuda")
    seg = torch.tensor(ref[3][layer], device="cuda")
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, layer, "cuda")
    q = synth.queries(B, m.Hq, m.H, m.d, cfg.seed, layer, device="cuda")
    sm = 1 / math.sqrt(m.d)
    offs, packed, out, _ = run_layer(g, K, V, kr, vr, rest_len, perm, seg, q, sm)
    # packed bytes of request 0 (all heads) bit-exact
    g1 = orc.geom(1, m.H, m.Hq, m.d, cfg.M, cfg.S, list(cfg.widths))
    opk, ooffs = orc.reorder_quantize_pack(K[:1].cpu().numpy(), V[:1].cpu().numpy(), 0, g1,
                                           ref[2][layer][:1], ref[3][layer][:1])
    n0 = int(ooffs[-1])
    assert np.array_equal(packed[:n0].cpu().numpy(), opk[:n0])
    # attention of sampled requests through the oracle (full cache of those requests)
    bs = sorted(set([0, B - 1]))
    for b in bs:
        sub = dict(q=q[b:b + 1], kr=kr[b:b + 1], vr=vr[b:b + 1], rest_len=rest_len[b:b + 1])
        gb = wq.geom(1, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
        ob = offs[b * m.H:(b + 1) * m.H + 1] - offs[b * m.H]
        pk = packed[int(offs[b * m.H].item()):int(offs[(b + 1) * m.H].item())]
        r = _decode_ref(orc, sub, gb, ob, pk, perm[b:b + 1], seg[b:b + 1], sm)[0]
        assert rel_err(out[b:b + 1].float().cpu().numpy(), r) <= ATTN_TOL


def test_decode_early_flag_matches(orc):
    """WQ_DECODE_EARLY (programmatic dependent launch after a previous decode on the
    stream) gives the same bytes as flags = 0, with both launches writing one output."""
    outs = []
    for flags in (0, wq.WQ_DECODE_EARLY):
        res = []
        for seed in (301, 302, 303):
            c = small_case(seed, d=128, S=32, W=12, tail=7, B=2, H=4, Hq=28)
            g = c["g"]
            sc = wq.wq_window_scores(c["vis"], c["txt"], 32)
            thr = orc.thresholds([0.45], 2.0, 4)
            _, _, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
            offs = wq.wq_layer_layout(g, seg[0])
            packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device="cuda")
            wq.wq_reorder_quantize_pack(c["K"], c["V"], 0, g, perm[0], seg[0], offs, packed)
            res.append((c, g, offs, packed, seg[0].contiguous()))
        torch.cuda.synchronize()
        out = torch.empty((2, 28, 128), dtype=torch.float16, device="cuda")
        ws = torch.zeros(wq.wq_decode_workspace(res[0][1]), dtype=torch.uint8, device="cuda")
        got = []
        for i, (c, g, offs, packed, seg) in enumerate(res):
            wq.wq_decode_attention(c["q"], packed, offs, seg, g, c["kr"], c["vr"], c["rest_len"], 0.088,
                                   out=out, workspace=ws, flags=flags if i > 0 else 0)
            got.append(out.clone())
        torch.cuda.synchronize()
        outs.append(torch.stack(got))
    assert torch.equal(outs[0], outs[1])


def test_decode_tcgen05_variant_parity():
    """The opt-in tcgen05/TMEM decode kernel (WQ_DECODE_TC=1, head dim 128) passes the same
    decode parity cases against the oracle (run in a child process: the switch is read once)."""
    import os, subprocess, sys
    env = dict(os.environ, WQ_DECODE_TC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", os.path.abspath(__file__),
                        "-k", "(decode_parity or decode_all16 or decode_edge or config_layer) and not tcgen05"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("d,S,W,tail,B,H,Hq", [(128, 32, 12, 7, 2, 4, 28), (64, 16, 9, 5, 2, 2, 14),
                                               (128, 128, 3, 9, 2, 2, 8)])
def test_unfused_baseline_parity(orc, d, S, W, tail, B, H, Hq):
    """T9 unfused path: the FP16 image is bit-exact with the oracle's and its decode
    matches the oracle's attention over that image."""
    c = small_case(300 + d + S, d=d, S=S, W=W, tail=tail, B=B, H=H, Hq=Hq)
    g = c["g"]
    sc = wq.wq_window_scores(c["vis"], c["txt"], S)
    thr = orc.thresholds([0.45], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
    sm = 1 / math.sqrt(d)
    offs, packed, _, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0], c["q"], sm)
    seg16, offs16 = wq.wq_dequant_layout(g, seg[0])
    img16 = torch.zeros(int(offs16[-1].item()) + 16, dtype=torch.uint8, device="cuda")
    wq.wq_dequantize_image(packed, offs, seg[0], g, offs16, img16)
    out = torch.empty((g.B, g.Hq, g.d), dtype=torch.float16, device="cuda")
    wq.wq_decode_attention(c["q"], img16, offs16, seg16, g, c["kr"], c["vr"], c["rest_len"], sm, out=out)
    torch.cuda.synchronize()
    rimg, roffs16, rseg16 = orc.dequantize_image(packed.cpu().numpy(), offs.cpu().numpy(), seg[0].cpu().numpy(),
                                                 ogeom(orc, g))
    assert np.array_equal(seg16.cpu().numpy(), rseg16)
    assert np.array_equal(offs16.cpu().numpy(), roffs16)
    n = int(roffs16[-1])
    assert np.array_equal(img16.cpu().numpy()[:n], rimg[:n])
    ref = orc.decode_attention(c["q"].cpu().numpy(), rimg, roffs16, rseg16, perm[0].cpu().numpy(), ogeom(orc, g),
                               c["kr"].cpu().numpy(), c["vr"].cpu().numpy(), c["rest_len"].cpu().numpy(), sm)
    assert rel_err(out.float().cpu().numpy(), ref) <= ATTN_TOL


@pytest.mark.parametrize("d,S,W,tail,B,H,Hq", [(128, 32, 40, 7, 2, 4, 28), (64, 16, 30, 5, 2, 2, 14),
                                               (128, 128, 5, 9, 2, 2, 8), (128, 16, 90, 0, 1, 4, 28)])
def test_unreordered_baseline_parity(orc, d, S, W, tail, B, H, Hq):
    """T8 "Module III off" path: the unreordered image holds the packed records in original
    window order at the prefix offsets, and its decode (windows in original order, per-window
    width) matches the oracle's attention over the same codes (Eq.12-13: order-invariant)."""
    c = small_case(400 + d + S + W, d=d, S=S, W=W, tail=tail, B=B, H=H, Hq=Hq)
    g = c["g"]
    sc = wq.wq_window_scores(c["vis"], c["txt"], S)
    thr = orc.thresholds([0.45], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
    sm = 1 / math.sqrt(d)
    offs, packed, _, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0], c["q"], sm)
    woff = wq.wq_unreordered_layout(g, bits[0].contiguous())
    uimg = torch.zeros_like(packed)
    wq.wq_unreorder_image(packed, offs, seg[0], perm[0], g, woff, uimg)
    out = torch.empty((g.B, g.Hq, g.d), dtype=torch.float16, device="cuda")
    part = torch.empty((g.B, g.Hq, g.d + 2), dtype=torch.float32, device="cuda")
    wq.wq_decode_attention_unreordered(c["q"], uimg, offs, seg[0], woff, g, c["kr"], c["vr"], c["rest_len"], sm,
                                       out=out, partial=part)
    torch.cuda.synchronize()
    bl, pm, sg, of = bits[0].cpu().numpy(), perm[0].cpu().numpy(), seg[0].cpu().numpy(), offs.cpu().numpy()
    wo, ui, pk = woff.cpu().numpy(), uimg.cpu().numpy(), packed.cpu().numpy()
    rb = {b_: orc.record_bytes(b_, d, S) for b_ in (2, 4, 8, 16)}
    for b in range(g.B):
        assert np.array_equal(wo[b], np.concatenate([[0], np.cumsum([rb[int(x)] for x in bl[b]])]))
        for h in range(g.H):
            u = b * g.H + h
            so = 0
            for slot in range(sg[b, 4]):
                k = int(np.searchsorted(sg[b, 1:], slot, side="right"))
                n = rb[(2, 4, 8, 16)[k]]
                w = pm[b, slot]
                assert bl[b, w] == (2, 4, 8, 16)[k]
                assert np.array_equal(ui[of[u] + wo[b, w]:of[u] + wo[b, w] + n], pk[of[u] + so:of[u] + so + n])
                so += n
    ref = _decode_ref(orc, c, g, offs, packed, perm[0], seg[0], sm)[0]
    assert rel_err(out.float().cpu().numpy(), ref) <= ATTN_TOL
    p = part.double().cpu().numpy()
    assert rel_err(p[..., 2:] / p[..., 1:2], ref) <= ATTN_TOL


def test_pearson_scores_parity(orc):
    """T11 similarity variant: GPU Pearson window scores vs the literal oracle (1e-12 abs)."""
    rng = np.random.default_rng(5)
    B, M, N, D, S = 2, 6 * 32 + 7, 9, 136, 32
    vis = torch.from_numpy(rng.standard_normal((B, M, D)).astype(np.float16) + 0.3).cuda()
    txt = torch.from_numpy(rng.standard_normal((B, N, D)).astype(np.float16) - 0.2).cuda()
    vis[0, 5] = 0.75                                   # constant row: contributes 0
    got = wq.wq_window_scores(vis, txt, S, metric=wq.WQ_SIM_PEARSON).cpu().numpy()
    ref = orc.window_scores_pearson(vis.cpu().numpy(), txt.cpu().numpy(), S)
    assert np.max(np.abs(got - ref)) < 1e-12
    cos = wq.wq_window_scores(vis, txt, S).cpu().numpy()
    assert np.max(np.abs(cos - orc.window_scores(vis.cpu().numpy(), txt.cpu().numpy(), S))) < 1e-12


def test_peer_merge_single_rank(orc):
    """The fused cross-GPU merge path (wq_decode_attention_peer) with G = 1: the kernel writes
    its partials to its slot of the symmetric buffer, bumps the arrival counter, waits for it
    and merges -- over several epochs (both parities) it must equal the plain decode."""
    from paper_2605_02262_b200.parallel import PeerMerge
    for d, S, W, tail, B, H, Hq in [(128, 32, 40, 7, 2, 4, 28), (64, 16, 30, 5, 2, 2, 14)]:
        c = small_case(500 + d + S, d=d, S=S, W=W, tail=tail, B=B, H=H, Hq=Hq)
        g = c["g"]
        sc = wq.wq_window_scores(c["vis"], c["txt"], S)
        thr = orc.thresholds([0.45], 2.0, 4)
        bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
        sm = 1 / math.sqrt(d)
        offs, packed, out, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0],
                                         c["q"], sm)
        pm = PeerMerge(g)
        ref = _decode_ref(orc, c, g, offs, packed, perm[0], seg[0], sm)[0]
        for _ in range(3):
            o2 = torch.zeros_like(out)
            wq.wq_decode_attention_peer(c["q"], packed, offs, seg[0], g, c["kr"], c["vr"], c["rest_len"], sm, o2,
                                        pm.ptrs, pm.local, 1, 0, pm.next_epoch())
            torch.cuda.synchronize()
            assert rel_err(o2.float().cpu().numpy(), ref) <= ATTN_TOL
            assert torch.equal(o2, out)
        assert not pm.timed_out()
        pm.close()


@pytest.mark.parametrize("d,S,W,tail,B,H,Hq", [(128, 32, 40, 7, 2, 4, 28), (64, 16, 30, 5, 3, 2, 14)])
def test_peer_merge_two_rank_emulation(orc, d, S, W, tail, B, H, Hq):
    """The G = 2 exchange of the fused cross-GPU merge, executed: two virtual ranks share
    one launch (half of the SMs each), each decodes its wq_shard_slots shard of the
    sequence split and exchanges its (m, l, o) rows with the other through the two
    symmetric buffers (peer stores, red.release.sys counters, ld.acquire.sys wait, LSE
    merge).  Over several epochs (both buffer parities) both ranks' merged outputs equal
    each other, stay within 2e-3 of the oracle's unsplit attention, and no wait times out."""
    c = small_case(600 + d + S, d=d, S=S, W=W, tail=tail, B=B, H=H, Hq=Hq)
    g = c["g"]
    sc = wq.wq_window_scores(c["vis"], c["txt"], S)
    thr = orc.thresholds([0.45], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
    sm = 1 / math.sqrt(d)
    offs, packed, full, _ = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0], c["q"], sm)
    ref = _decode_ref(orc, c, g, offs, packed, perm[0], seg[0], sm)[0]
    ranks = []
    for r in range(2):
        pr, sr = wq.wq_shard_slots(perm[0], seg[0], 2, r)
        rl = c["rest_len"] if r == 0 else torch.zeros_like(c["rest_len"])
        o_r = wq.wq_layer_layout(g, sr)
        pk = torch.zeros(int(o_r[-1].item()) + 16, dtype=torch.uint8, device="cuda")
        wq.wq_reorder_quantize_pack(c["K"], c["V"], 0, g, pr, sr, o_r, pk)
        ranks.append(dict(q=c["q"], packed=pk, offs=o_r, seg_off=sr.contiguous(), k_rest=c["kr"], v_rest=c["vr"],
                          rest_len=rl, out=torch.zeros_like(full),
                          workspace=torch.zeros(wq.wq_decode_workspace(g), dtype=torch.uint8, device="cuda")))
    nb = wq.wq_peer_buffer_bytes(g, 2)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    err_off = wq.wq_peer_error_offset(g, 2)
    for epoch in (1, 2, 3, 4):
        for rk in ranks:
            rk["out"].zero_()
        wq.wq_decode_attention_peer_emulated(ranks, g, sm, ptrs, [b.data_ptr() for b in bufs], epoch)
        torch.cuda.synchronize()
        for r in range(2):
            assert int(bufs[r][err_off:err_off + 4].view(torch.int32).item()) == 0, "peer wait timed out"
        assert torch.equal(ranks[0]["out"], ranks[1]["out"])
        assert rel_err(ranks[0]["out"].float().cpu().numpy(), ref) <= ATTN_TOL
        assert rel_err(ranks[0]["out"].float().cpu().numpy(), full.float().cpu().numpy()) <= ATTN_TOL


def _peer_ipc_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2605_02262_b200.parallel import PeerMerge, _cudart, _ck
        g = wq.geom(2, 2, 14, 64, 160, 16, (2, 4, 8, 16))
        pm = PeerMerge(g, device=torch.device("cuda", 0))
        ptrs = pm.ptrs.cpu().tolist()
        assert ptrs[rank] == pm.local and len(set(ptrs)) == world
        rt = _cudart()
        # every rank writes its signature into slot `rank` of every peer's buffer
        sig = np.full(16, 1000 + rank, np.int32)
        for p in range(world):
            _ck(rt.cudaMemcpy(ptrs[p] + 64 * rank, sig.ctypes.data, 64, rt.cudaMemcpyKind.cudaMemcpyHostToDevice))
        torch.cuda.synchronize()
        dist.barrier()
        got = np.zeros(16 * world, np.int32)
        _ck(rt.cudaMemcpy(got.ctypes.data, pm.local, 64 * world, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost))
        ok = all((got[16 * p:16 * (p + 1)] == 1000 + p).all() for p in range(world))
        dist.barrier()
        pm.close()
        dist.destroy_process_group()
        q.put((rank, bool(ok), ""))
    except Exception as e:  # pragma: no cover
        q.put((rank, False, repr(e)))


def test_peer_merge_ipc_setup_two_processes():
    """PeerMerge's CUDA IPC exchange (the setup of the fused cross-GPU merge) between two
    processes on one GPU: every rank writes into every peer's mapped buffer and reads back
    its own.  (No kernel waits on another process: only the mappings are exercised.)"""
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + random.randint(0, 999)
    procs = [ctx.Process(target=_peer_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def test_ablation_paths_full_size_c5(orc):
    """The T8 (unreordered) and T9 (unfused) baselines and the fused peer-merge path at the
    full C5 size bench.py times, with the oracle on a sampled request: unreordered and peer
    decodes within 2e-3 of the oracle over the same codes; the unfused path within 2e-3 of the
    oracle's attention over its FP16 image."""
    from paper_2605_02262_b200.parallel import PeerMerge
    cfg = configs.CONFIGS["C5"]
    m = cfg.model
    B, layer = cfg.B, cfg.layers - 1
    vis, txt = synth.embeddings(B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, "cuda")
    sc = wq.wq_window_scores(vis, txt, cfg.S)
    del vis, txt
    thr = orc.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
    g = wq.geom(B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, cfg.layers, g)
    bl, perm, seg = bits[layer].contiguous(), perm[layer].contiguous(), seg[layer].contiguous()
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, layer, "cuda")
    q = synth.queries(B, m.Hq, m.H, m.d, cfg.seed, layer, device="cuda")
    sm = 1 / math.sqrt(m.d)
    offs, packed, out, _ = run_layer(g, K, V, kr, vr, rest_len, perm, seg, q, sm)
    del K, V
    woff = wq.wq_unreordered_layout(g, bl)
    uimg = torch.zeros_like(packed)
    wq.wq_unreorder_image(packed, offs, seg, perm, g, woff, uimg)
    out_u = torch.empty_like(out)
    wq.wq_decode_attention_unreordered(q, uimg, offs, seg, woff, g, kr, vr, rest_len, sm, out=out_u)
    seg16, offs16 = wq.wq_dequant_layout(g, seg)
    img16 = torch.zeros(int(offs16[-1].item()) + 16, dtype=torch.uint8, device="cuda")
    wq.wq_dequantize_image(packed, offs, seg, g, offs16, img16)
    out_16 = torch.empty_like(out)
    wq.wq_decode_attention(q, img16, offs16, seg16, g, kr, vr, rest_len, sm, out=out_16)
    pm = PeerMerge(g)
    out_p = torch.empty_like(out)
    wq.wq_decode_attention_peer(q, packed, offs, seg, g, kr, vr, rest_len, sm, out_p, pm.ptrs, pm.local, 1, 0,
                                pm.next_epoch())
    torch.cuda.synchronize()
    pm.close()
    assert torch.equal(out_p, out)
    b = B - 1
    sub = dict(q=q[b:b + 1], kr=kr[b:b + 1], vr=vr[b:b + 1], rest_len=rest_len[b:b + 1])
    gb = wq.geom(1, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    ob = offs[b * m.H:(b + 1) * m.H + 1] - offs[b * m.H]
    pk = packed[int(offs[b * m.H].item()):int(offs[(b + 1) * m.H].item())]
    r = _decode_ref(orc, sub, gb, ob, pk, perm[b:b + 1], seg[b:b + 1], sm)[0]
    assert rel_err(out_u[b:b + 1].float().cpu().numpy(), r) <= ATTN_TOL
    # the FP16 image of request b, bit-exact, and its attention
    ob16 = offs16[b * m.H:(b + 1) * m.H + 1] - offs16[b * m.H]
    pk16 = img16[int(offs16[b * m.H].item()):int(offs16[(b + 1) * m.H].item())]
    rimg, roffs16, rseg16 = orc.dequantize_image(pk.cpu().numpy(), ob.cpu().numpy(), seg[b:b + 1].cpu().numpy(),
                                                 ogeom(orc, gb))
    assert np.array_equal(pk16.cpu().numpy(), rimg[:int(roffs16[-1])])
    r16 = _decode_ref(orc, sub, gb, ob16, pk16, perm[b:b + 1], seg16[b:b + 1], sm)[0]
    assert rel_err(out_16[b:b + 1].float().cpu().numpy(), r16) <= ATTN_TOL


@pytest.mark.parametrize("B,H,Hq,d,S,W,tail,N,vis_off", [(2, 2, 14, 64, 16, 9, 5, 8, 3), (1, 4, 28, 128, 32, 12, 7, 32, 0),
                                                      (3, 4, 8, 128, 64, 4, 0, 5, 16)])
def test_layer_scores_parity(orc, B, H, Hq, d, S, W, tail, N, vis_off):
    """Per-layer scorer (§8(f) row 4, reading Q36): post-RoPE visual keys (kv heads
    concatenated, read in place through the head stride) against the GQA-averaged text
    queries, 1e-12 absolute against the literal oracle."""
    M = W * S + tail
    K, _ = synth.kv_layer(B, H, vis_off + M, d, S, 70 + d, 1, "cuda")
    qt = synth.text_queries(B, Hq, N, d, 70 + d, 1, "cuda")
    got = wq.wq_window_scores_layer(K, vis_off, qt, M, S)
    torch.cuda.synchronize()
    ref = orc.window_scores_layer(K.cpu().numpy(), vis_off, qt.cpu().numpy(), M, S)
    assert np.max(np.abs(got.cpu().numpy() - ref)) <= 1e-12


def test_layer_scores_c5_geometry(orc):
    """The layer scorer at the full C5 layer shape (B = 4, H = 4, d = 128, 50,176 visual
    tokens, N = 32): request 1 against the oracle (every window), bit-exact assignment
    from those scores."""
    cfg = configs.CONFIGS["C5"]
    m = cfg.model
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, 3, "cuda")
    del V, kr, vr
    qt = synth.text_queries(cfg.B, m.Hq, cfg.n_text, m.d, cfg.seed, 3, "cuda")
    got = wq.wq_window_scores_layer(K, 0, qt, cfg.M, cfg.S)
    torch.cuda.synchronize()
    ref = orc.window_scores_layer(K[1:2].cpu().numpy(), 0, qt[1:2].cpu().numpy(), cfg.M, cfg.S)
    assert np.max(np.abs(got[1:2].cpu().numpy() - ref)) <= 1e-12
    thr = orc.thresholds([0.5], cfg.alpha, 4)
    g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    gpu, oref = _assign_both(orc, got, thr, g)
    for a_, b_ in zip(gpu, oref):
        assert np.array_equal(a_, b_)


@pytest.mark.parametrize("B,M,N,D,S,widths,budget,vote,metric,L", [
    (2, 16 * 9 + 5, 8, 64, 16, (2, 4, 8, 16), 0.0, 0, 0, 3), (3, 32 * 40, 5, 896, 32, (2, 4, 8, 16), 4.0, 0, 0, 5),
    (4, 32 * 50, 7, 3584, 32, (2, 4, 16), 3.5, 1, 0, 2), (2, 64 * 20 + 7, 6, 256, 64, (2, 4, 8), 0.0, 1, 1, 4),
    (2, 16 * 300, 32, 512, 16, (4, 8), 5.0, 0, 1, 2)])
def test_fused_search_equals_chain(orc, B, M, N, D, S, widths, budget, vote, metric, L):
    """wq_search (scores + rank + assign of L layers in one cooperative launch, one rank
    sort per request) gives bit-identical scores, ranks, bits, perms and seg_off to the
    unfused chain, and matches the oracle's assignment."""
    vis, txt = synth.embeddings(B, M, N, D, S, 900 + D, "cuda")
    g = wq.geom(B, 2, 14, 64, M, S, widths)
    s_prof = [0.5, 0.3, 0.9, 0.05, 0.6][:L]
    thr = orc.thresholds(s_prof, 2.0, len(widths))
    opts = wq.AssignOpts(budget, 1, vote)
    sc0 = wq.wq_window_scores(vis, txt, S, metric=metric)
    bits0, rank0, perm0, seg0 = wq.wq_assign_bits(sc0, thr, L, g, opts)
    sc1, bits1, rank1, perm1, seg1 = wq.wq_search(vis, txt, thr, L, g, opts, metric=metric)
    torch.cuda.synchronize()
    assert torch.equal(sc0, sc1)
    for x, y in ((bits0, bits1), (rank0, rank1), (perm0, perm1), (seg0, seg1)):
        assert torch.equal(x, y)
    ob, orank, operm, oseg = orc.assign_bits(sc1.cpu().numpy(), thr, ogeom(orc, g), budget, 1, vote)
    assert np.array_equal(bits1.cpu().numpy(), ob) and np.array_equal(perm1.cpu().numpy(), operm)


def test_fused_search_c5(orc):
    """The fused search at the full C5 size (B = 4, 50,176 visual tokens, D = 3584, 28
    layers, budget 3.5): bit-identical to the chain."""
    cfg = configs.CONFIGS["C5"]
    m = cfg.model
    vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, "cuda")
    thr = orc.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
    g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    opts = wq.AssignOpts(3.5, 1, 0)
    sc0 = wq.wq_window_scores(vis, txt, cfg.S)
    chain = wq.wq_assign_bits(sc0, thr, cfg.layers, g, opts)
    fused = wq.wq_search(vis, txt, thr, cfg.layers, g, opts)
    torch.cuda.synchronize()
    assert torch.equal(sc0, fused[0])
    for x, y in zip(chain, fused[1:]):
        assert torch.equal(x, y)
