"""wq_reorder_quantize_pack time on a config (default C5): layers rotate so K/V come from
HBM; reports us per call and algorithmic GB/s (K+V read + packed image written)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import oracle
from paper_2605_02262_b200 import configs, synth, wq

cfg = configs.CONFIGS[os.environ.get("CFG", "C5")]
if os.environ.get("S"):
    cfg = cfg.with_(S=int(os.environ["S"]), name=f"{cfg.name}-S{os.environ['S']}")
m = cfg.model
L = int(os.environ.get("NL", "4"))
dev = "cuda"
vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, dev)
g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
thr = oracle.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
sc = wq.wq_window_scores(vis, txt, cfg.S)
bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, cfg.layers, g, wq.AssignOpts(cfg.budget, 1, 0))
layers = []
nbytes = 0
for l in range(L):
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, dev)
    offs = wq.wq_layer_layout(g, seg[l])
    packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
    nw = int(seg[l][:, 4].sum().item()) * m.H
    nbytes += nw * 4 * cfg.S * m.d + int(offs[-1].item())
    layers.append((K, V, perm[l].contiguous(), seg[l].contiguous(), offs, packed))
nbytes /= L


def run(n):
    for i in range(n):
        K, V, p, s, offs, packed = layers[i % L]
        wq.wq_reorder_quantize_pack(K, V, 0, g, p, s, offs, packed)


run(2 * L)
torch.cuda.synchronize()
n = 10 * L
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
run(n)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / n
print(f"quantize {cfg.name}: {us:8.2f} us/call  {nbytes / us / 1e3:7.1f} GB/s  ({nbytes / 1e6:.1f} MB/call)")
