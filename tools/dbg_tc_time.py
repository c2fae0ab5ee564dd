"""Per-group clock64 stamps of one C5-shaped tcgen05 decode launch (build variant
WQ_VARIANT=tcprof WQ_NVCC_DEFS=-DWQ_TC_PROFILE=1): for a few CTAs, per group j the
cycles of (dequant start, dequant published, K MMAs issued, softmax has S, P' published)
relative to the kernel start, and the per-group deltas."""
import math, sys, os
os.environ.setdefault("WQ_VARIANT", "tcprof")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02262_b200 import configs, synth, wq
import oracle
cfg = configs.CONFIGS[os.environ.get("CFG", "C5")]; m = cfg.model
dev = "cuda"
vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, dev)
g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
thr = oracle.thresholds(cfg.sensitivities(), cfg.alpha, len(cfg.widths))
sc = wq.wq_window_scores(vis, txt, cfg.S)
bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, cfg.layers, g, wq.AssignOpts(cfg.budget, 1, 0))
l = cfg.layers - 1
K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, dev)
q = synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, l, device=dev)
offs = wq.wq_layer_layout(g, seg[l])
packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
wq.wq_reorder_quantize_pack(K, V, 0, g, perm[l], seg[l], offs, packed)
ws = torch.zeros(wq.wq_decode_workspace(g), dtype=torch.uint8, device=dev)
out = torch.empty((cfg.B, m.Hq, m.d), dtype=torch.float16, device=dev)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
TS = 200
os.environ["WQ_DECODE_DEBUG"] = "8"
for it in range(4):
    ws[-nsm * TS * 8:].zero_()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); wq.wq_decode_attention(q, packed, offs, seg[l].contiguous(), g, kr, vr, rest_len, 1 / math.sqrt(128), out=out, workspace=ws); e1.record()
    torch.cuda.synchronize()
print(f"event us {e0.elapsed_time(e1) * 1e3:.1f}")
tsb = ws[-nsm * TS * 8:].view(torch.int64).view(nsm, TS).cpu().numpy().astype(np.float64)
for cta in [0, 1, 70, 147]:
    t0 = tsb[cta, 0]
    print(f"CTA {cta}: total {tsb[cta, 1] - t0:.0f} cycles")
    ev = tsb[cta, 10:10 + 5 * 38].reshape(38, 5) - t0
    ev[tsb[cta, 10:10 + 5 * 38].reshape(38, 5) == 0] = np.nan
    print("   j   dq_start  dq_pub  K_iss  S_ready  P_pub   | dq  K-dq  S-K  P-S  dqstart_delta")
    for j in range(38):
        e = ev[j]
        if np.all(np.isnan(e)): continue
        d = [e[1] - e[0], e[2] - e[1], e[3] - e[2], e[4] - e[3], (e[0] - ev[j - 1][0]) if j else np.nan]
        print(f"  {j:2d} " + " ".join(f"{x:8.0f}" for x in e) + "  | " + " ".join(f"{x:5.0f}" for x in d))

if os.environ.get("WQ_VARIANT") == "tcprof99":
    print("per-warp publish cycles (rel. to warp 0) per group:")
    for cta in [0, 70]:
        t0 = tsb[cta, 0]
        pw = tsb[cta, 10:10 + 8 * 23].reshape(23, 8) - t0
        for j in range(23):
            print(f"  cta {cta} j {j:2d}  w0 {pw[j, 0]:8.0f}  " + " ".join(f"{x - pw[j, 0]:6.0f}" for x in pw[j]))
