"""Device time of the per-layer scorer (wq_window_scores_layer) on one full layer of a
config (default C5): text pool of the GQA-averaged queries + window scores of the keys."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_02262_b200 import configs, synth, wq  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
m = cfg.model
K, V, kr, vr, rl = synth.layer_tensors(cfg, 0, "cuda")
qt = synth.text_queries(cfg.B, m.Hq, cfg.n_text, m.d, cfg.seed, 0, "cuda")
sc = torch.empty((cfg.B, cfg.W), dtype=torch.float64, device="cuda")
ws = torch.empty(wq.wq_window_scores_workspace(cfg.B, m.H * m.d), dtype=torch.uint8, device="cuda")
ts = []
for i in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    wq.wq_window_scores_layer(K, 0, qt, cfg.M, cfg.S, scores=sc, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1) * 1e3)
mb = cfg.B * m.H * cfg.M * m.d * 2 / 1e6
us = statistics.median(ts)
print(f"{cfg.name}: per-layer scorer {us:.1f} us for {mb:.0f} MB of keys = {mb / us:.2f} TB/s")
