"""wq_window_scores device time on a config's embeddings (default C5): cosine and Pearson."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_02262_b200 import configs, synth, wq  # noqa: E402

cfg = configs.CONFIGS[os.environ.get("CFG", "C5")]
m = cfg.model
vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, "cuda")
for name, metric in (("cosine", wq.WQ_SIM_COSINE), ("pearson", wq.WQ_SIM_PEARSON)):
    sc = wq.wq_window_scores(vis, txt, cfg.S, metric=metric)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        wq.wq_window_scores(vis, txt, cfg.S, scores=sc, metric=metric)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 5
    print(f"{cfg.name} {name}: {us:8.1f} us  {vis.numel() * 2 / us / 1e3:7.1f} GB/s")
