"""C1-sized run of every libwq device call, for the checked build (tests/test_gpu_checked.py):
scores (cosine, Pearson), rank + assign (budget and vote), layout, quantize, decode
(flags 0, then a PDL-chained WQ_DECODE_EARLY decode, and partials), merge, shard,
the unfused (T9) and unreordered (T8) baselines, the group granularity (quantize +
WQ_DECODE_GROUP decode), the per-layer scorer, the fused search and the two-rank
fused-merge emulation.
Exits 0 when every call returned WQ_OK; under WQ_VARIANT=checked (-DWQ_CHECKS=1) every
device-side bounds check of the path ran."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_02262_b200 import configs, synth, wq  # noqa: E402


def main():
    wq.load(build_if_missing=False)
    cfg = configs.CONFIGS["C1"]
    m = cfg.model
    dev = "cuda"
    vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, dev)
    sc = wq.wq_window_scores(vis, txt, cfg.S)
    wq.wq_window_scores(vis, txt, cfg.S, metric=wq.WQ_SIM_PEARSON)
    g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, (2, 4, 8, 16))
    thr = wq.wq_thresholds([0.5, 0.3], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 2, g, wq.AssignOpts(4.5, 1, 1))
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 2, g, wq.AssignOpts(0.0, 1, 0))
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, 0, dev)
    q = synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, 0, device=dev)
    sm = 1 / math.sqrt(m.d)
    offs = wq.wq_layer_layout(g, seg[0])
    packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
    wq.wq_reorder_quantize_pack(K, V, 0, g, perm[0], seg[0], offs, packed)
    out = torch.empty((cfg.B, m.Hq, m.d), dtype=torch.float16, device=dev)
    part = torch.empty((cfg.B, m.Hq, m.d + 2), dtype=torch.float32, device=dev)
    ws = torch.zeros(wq.wq_decode_workspace(g), dtype=torch.uint8, device=dev)
    wq.wq_decode_attention(q, packed, offs, seg[0], g, kr, vr, rest_len, sm, out=out, partial=part, workspace=ws)
    wq.wq_decode_attention(q, packed, offs, seg[0], g, kr, vr, rest_len, sm, out=out, workspace=ws,
                           flags=wq.WQ_DECODE_EARLY)
    wq.wq_merge_partials(torch.stack([part, part]), g)
    # paper-literal group granularity: layout, quantize, decode (plain and PDL-chained)
    offs_g = wq.wq_layer_layout(g, seg[0], gran=wq.WQ_GRAN_GROUP)
    packed_g = torch.zeros(int(offs_g[-1].item()) + 16, dtype=torch.uint8, device=dev)
    wq.wq_reorder_quantize_pack(K, V, 0, g, perm[0], seg[0], offs_g, packed_g, gran=wq.WQ_GRAN_GROUP)
    for fl in (wq.WQ_DECODE_GROUP, wq.WQ_DECODE_GROUP | wq.WQ_DECODE_EARLY):
        wq.wq_decode_attention(q, packed_g, offs_g, seg[0], g, kr, vr, rest_len, sm, out=out, partial=part,
                               workspace=ws, flags=fl)
    # more (request, head) units than SMs (the cost-stream split of whole units) and S = 128
    # windows consumed as 32-token parts, FP16 windows as two 64-token items
    for S_ in (64, 128):
        Bn, Hn, Mn = 40, 4, 5 * S_ + 7
        gb = wq.geom(Bn, Hn, 7 * Hn, 128, Mn, S_, (2, 4, 8, 16))
        Kb = torch.randn((Bn, Hn, Mn, 128), device=dev).half()
        Vb = torch.randn((Bn, Hn, Mn, 128), device=dev).half()
        wb = Mn // S_
        bits_b = torch.tensor([[2, 4, 8, 16, 2][:wb] for _ in range(Bn)], dtype=torch.int32)
        perm_b = torch.argsort(bits_b * 8 + torch.arange(wb), dim=1).to(torch.int32).to(dev)
        seg_b = torch.tensor([[0, 2, 3, 4, 5] for _ in range(Bn)], dtype=torch.int32, device=dev)
        ob = wq.wq_layer_layout(gb, seg_b)
        pb = torch.zeros(int(ob[-1].item()) + 16, dtype=torch.uint8, device=dev)
        wq.wq_reorder_quantize_pack(Kb, Vb, 0, gb, perm_b, seg_b, ob, pb)
        krb = torch.randn((Bn, Hn, 21, 128), device=dev).half()
        rlb = torch.full((Bn,), 19, dtype=torch.int32, device=dev)
        qb = torch.randn((Bn, 7 * Hn, 128), device=dev).half()
        wq.wq_decode_attention(qb, pb, ob, seg_b, gb, krb, krb, rlb, 0.088, out=torch.empty_like(qb))
    # per-layer K/Q scorer and the fused search
    qt = synth.text_queries(cfg.B, m.Hq, cfg.n_text, m.d, cfg.seed, 0, dev)
    wq.wq_window_scores_layer(K, 0, qt, cfg.M, cfg.S)
    wq.wq_search(vis, txt, thr, 2, g, wq.AssignOpts(4.5, 1, 1))
    wq.wq_search(vis, txt, thr, 2, g, wq.AssignOpts(0.0, 1, 0), metric=wq.WQ_SIM_PEARSON)
    pr, sr = wq.wq_shard_slots(perm[0], seg[0], 2, 1)
    seg16, offs16 = wq.wq_dequant_layout(g, seg[0])
    img16 = torch.zeros(int(offs16[-1].item()) + 16, dtype=torch.uint8, device=dev)
    wq.wq_dequantize_image(packed, offs, seg[0], g, offs16, img16)
    woff = wq.wq_unreordered_layout(g, bits[0].contiguous())
    uimg = torch.zeros_like(packed)
    wq.wq_unreorder_image(packed, offs, seg[0], perm[0], g, woff, uimg)
    wq.wq_decode_attention_unreordered(q, uimg, offs, seg[0], woff, g, kr, vr, rest_len, sm, out=out)
    # fused merge, two virtual ranks in one launch (d = 64 needs S = 16 here)
    g16 = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, 16, (2, 4, 8, 16))
    sc16 = wq.wq_window_scores(vis, txt, 16)
    _, _, perm16, seg16b = wq.wq_assign_bits(sc16, thr[:1], 1, g16)
    ranks = []
    for r in range(2):
        p_r, s_r = wq.wq_shard_slots(perm16[0], seg16b[0], 2, r)
        o_r = wq.wq_layer_layout(g16, s_r)
        pk = torch.zeros(int(o_r[-1].item()) + 16, dtype=torch.uint8, device=dev)
        wq.wq_reorder_quantize_pack(K, V, 0, g16, p_r, s_r, o_r, pk)
        ranks.append(dict(q=q, packed=pk, offs=o_r, seg_off=s_r.contiguous(), k_rest=kr, v_rest=vr,
                          rest_len=rest_len if r == 0 else torch.zeros_like(rest_len), out=torch.zeros_like(out),
                          workspace=torch.zeros(wq.wq_decode_workspace(g16), dtype=torch.uint8, device=dev)))
    nb = wq.wq_peer_buffer_bytes(g16, 2)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device=dev) for _ in range(2)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=dev)
    for epoch in (1, 2):
        wq.wq_decode_attention_peer_emulated(ranks, g16, sm, ptrs, [b.data_ptr() for b in bufs], epoch)
    torch.cuda.synchronize()
    print("checked_run: ok")


if __name__ == "__main__":
    main()
