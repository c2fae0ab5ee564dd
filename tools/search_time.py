"""Fused search (wq_search: one cooperative launch) vs the unfused chain (wq_window_scores:
text pool + window scores; wq_assign_bits: rank + assign) on a config's full size, budget
on and off; device time per call (CUDA events, median of reps)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_02262_b200 import configs, synth, wq  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


for name in sys.argv[1:] or ["C5", "C3", "C2"]:
    cfg = configs.CONFIGS[name]
    m = cfg.model
    vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, "cuda")
    thr = wq.wq_thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
    g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    for budget in (cfg.budget, 3.5):
        opts = wq.AssignOpts(budget, 1, 0)
        W, L = cfg.W, cfg.layers
        sc = torch.empty((cfg.B, W), dtype=torch.float64, device="cuda")
        sws = torch.empty(wq.wq_window_scores_workspace(cfg.B, m.D), dtype=torch.uint8, device="cuda")
        outs = (torch.empty((L, cfg.B, W), dtype=torch.uint8, device="cuda"),
                torch.empty((cfg.B, W), dtype=torch.int32, device="cuda"),
                torch.empty((L, cfg.B, W), dtype=torch.int32, device="cuda"),
                torch.empty((L, cfg.B, 5), dtype=torch.int32, device="cuda"))

        def chain():
            wq.wq_window_scores(vis, txt, cfg.S, scores=sc, workspace=sws)
            wq.wq_assign_bits(sc, thr, L, g, opts, *outs)

        fo = (sc,) + outs

        def fused():
            wq.wq_search(vis, txt, thr, L, g, opts, outs=fo)

        def assign_only():
            wq.wq_assign_bits(sc, thr, L, g, opts, *outs)

        print(f"{name} budget={budget}: chain {timed(chain):8.1f} us (assign alone {timed(assign_only):7.1f})  "
              f"fused {timed(fused):8.1f} us", flush=True)
