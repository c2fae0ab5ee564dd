"""Error margins of wq_decode_attention against the oracle (GPU): max row relative
error of the fp16 output and of the fp32 partial O/L, per config (full-size layer,
two sampled requests) and per small case.  Diagnostic companion of
tests/test_gpu_parity.py (same helpers, same inputs)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle as orc
from paper_2605_02262_b200 import configs, synth, wq
from test_gpu_parity import _decode_ref, rel_err, run_layer, small_case


def report(tag, out, part, ref):
    o = rel_err(out.float().cpu().numpy(), ref)
    p = part.double().cpu().numpy()
    pe = rel_err(p[..., 2:] / p[..., 1:2], ref)
    print(f"{tag:28s} out {o:.3e}  partial {pe:.3e}", flush=True)
    return o, pe


def main():
    worst = [0.0, 0.0]
    for i, (d, S, W, tail, B, H, Hq) in enumerate([(64, 16, 9, 5, 2, 2, 14), (128, 32, 12, 7, 2, 4, 28),
                                                    (128, 64, 5, 0, 1, 4, 28), (128, 128, 3, 9, 2, 2, 8),
                                                    (128, 16, 30, 0, 4, 4, 28)]):
        c = small_case(200 + d + S + W, d=d, S=S, W=W, tail=tail, B=B, H=H, Hq=Hq)
        g = c["g"]
        sc = wq.wq_window_scores(c["vis"], c["txt"], S)
        thr = orc.thresholds([0.45], 2.0, 4)
        _, _, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
        offs, packed, out, part = run_layer(g, c["K"], c["V"], c["kr"], c["vr"], c["rest_len"], perm[0], seg[0],
                                            c["q"], 1 / math.sqrt(d), partial=True)
        ref, _ = _decode_ref(orc, c, g, offs, packed, perm[0], seg[0], 1 / math.sqrt(d))
        r = report(f"small d{d} S{S} W{W}", out, part, ref)
        worst = [max(worst[0], r[0]), max(worst[1], r[1])]
    names = sys.argv[1:] or ["C1", "C2", "C3", "C5"]
    for name in names:
        cfg = configs.CONFIGS[name]
        m = cfg.model
        layer = cfg.layers - 1
        vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, "cuda")
        sc = wq.wq_window_scores(vis, txt, cfg.S)
        thr = orc.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
        g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
        _, _, perm, seg = wq.wq_assign_bits(sc, thr, cfg.layers, g, wq.AssignOpts(cfg.budget, 1, 0))
        perm, seg = perm[layer].contiguous(), seg[layer].contiguous()
        K, V, kr, vr, rest_len = synth.layer_tensors(cfg, layer, "cuda")
        q = synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, layer, device="cuda")
        sm = 1 / math.sqrt(m.d)
        offs, packed, out, part = run_layer(g, K, V, kr, vr, rest_len, perm, seg, q, sm, partial=True)
        for b in sorted({0, cfg.B - 1}):
            sub = dict(q=q[b:b + 1], kr=kr[b:b + 1], vr=vr[b:b + 1], rest_len=rest_len[b:b + 1])
            gb = wq.geom(1, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
            ob = offs[b * m.H:(b + 1) * m.H + 1] - offs[b * m.H]
            pk = packed[int(offs[b * m.H].item()):int(offs[(b + 1) * m.H].item())]
            ref = _decode_ref(orc, sub, gb, ob, pk, perm[b:b + 1], seg[b:b + 1], sm)[0]
            r = report(f"{name} layer {layer} b{b}", out[b:b + 1], part[b:b + 1], ref)
            worst = [max(worst[0], r[0]), max(worst[1], r[1])]
    print(f"WORST out {worst[0]:.3e} partial {worst[1]:.3e}")


if __name__ == "__main__":
    main()
