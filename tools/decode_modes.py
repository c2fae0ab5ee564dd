"""Decode launch time on C5 under the kernel's debug modes (WQ_DECODE_DEBUG):
0 normal, 1 no compute (TMA stream only), 2 no copy (compute on stale smem), 3 neither.
Layers rotate so the packed images (~104 MB each) come from HBM, as in bench.py."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2605_02262_b200 import configs, synth, wq

cfg = configs.CONFIGS[os.environ.get("CFG", "C5")]
m = cfg.model
L = int(os.environ.get("NL", "6"))
dev = "cuda"
vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, dev)
g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
import oracle
thr = oracle.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
sc = wq.wq_window_scores(vis, txt, cfg.S)
bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, cfg.layers, g, wq.AssignOpts(cfg.budget, 1, 0))
layers = []
for l in range(L):
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, dev)
    offs = wq.wq_layer_layout(g, seg[l])
    packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
    wq.wq_reorder_quantize_pack(K, V, 0, g, perm[l], seg[l], offs, packed)
    q = synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, l, device=dev)
    del K, V
    layers.append((q, packed, offs, seg[l].contiguous(), kr, vr, rest_len))
ws = torch.zeros(wq.wq_decode_workspace(g), dtype=torch.uint8, device=dev)
out = torch.empty((cfg.B, m.Hq, m.d), dtype=torch.float16, device=dev)
nbytes = sum(int(x[2][-1].item()) for x in layers) / L
sm = 1 / math.sqrt(m.d)


EARLY = int(os.environ.get("EARLY", "0"))


def run(n):
    for i in range(n):
        q, packed, offs, s, kr, vr, rl = layers[i % L]
        wq.wq_decode_attention(q, packed, offs, s, g, kr, vr, rl, sm, out=out, workspace=ws,
                               flags=wq.WQ_DECODE_EARLY if (EARLY and i > 0) else 0)


import time
for mode in [int(x) for x in os.environ.get("MODES", "0,1,2,3").split(",")]:
    os.environ["WQ_DECODE_DEBUG"] = str(mode)
    run(3 * L)
    torch.cuda.synchronize()
    n = 20 * L
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter()
    e0.record()
    run(n)
    e1.record()
    host = (time.perf_counter() - t0) * 1e6 / n
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    # the same launches captured once in a CUDA graph (no host work between kernels)
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        run(2)
    torch.cuda.current_stream().wait_stream(s_)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        run(n)
    gr.replay()
    torch.cuda.synchronize()
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    ug = e0.elapsed_time(e1) * 1e3 / n
    print(f"mode {mode}: eager {us:7.2f} us/launch (host issue {host:6.2f} us)  graph {ug:7.2f} us/launch  "
          f"{nbytes / ug / 1e3:7.1f} GB/s (packed image bytes)", flush=True)
os.environ["WQ_DECODE_DEBUG"] = "0"
