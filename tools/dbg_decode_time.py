"""Per-CTA globaltimer stamps of one C5-shaped decode layer (WQ_DECODE_DEBUG has bit 8)."""
import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02262_b200 import configs, synth, wq
cfg = configs.CONFIGS["C5"]; m = cfg.model
dev = "cuda"
vis, txt = synth.embeddings(cfg.B, cfg.M, 32, m.D, cfg.S, cfg.seed, dev)
g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
thr = wq.wq_thresholds([0.5], 2.0, 4)
sc = wq.wq_window_scores(vis, txt, cfg.S)
bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
K, V, kr, vr, rest_len = synth.layer_tensors(cfg, 0, dev)
q = synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, 0, device=dev)
offs = wq.wq_layer_layout(g, seg[0])
packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
wq.wq_reorder_quantize_pack(K, V, 0, g, perm[0], seg[0], offs, packed)
ws = torch.zeros(wq.wq_decode_workspace(g), dtype=torch.uint8, device=dev)
out = torch.empty((cfg.B, m.Hq, m.d), dtype=torch.float16, device=dev)
for it in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); wq.wq_decode_attention(q, packed, offs, seg[0], g, kr, vr, rest_len, 1 / math.sqrt(128), out=out, workspace=ws); e1.record()
    torch.cuda.synchronize()
    print("event us", e0.elapsed_time(e1) * 1e3)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
tsb = ws[-nsm * 576:].view(torch.int64).view(nsm, 72).cpu().numpy()
NW = 11
wt = tsb[:, 8:8 + 4 * NW].reshape(nsm, NW, 4) / 1e3
kt = tsb[:, 56:61].sum(0) / 1e3; kc = tsb[:, 61:66].sum(0)
print("per-kind compute us per item (2,4,8,16,rest):", np.round(kt / np.maximum(kc, 1), 3), "counts", kc)
epi = tsb[:, 68:72] / 1e3
slow = np.argsort(-(tsb[:, 4] - tsb[:, 0]))[:4]
for cidx in list(slow) + [int(np.argsort(tsb[:, 4] - tsb[:, 0])[0])]:
    print("CTA", cidx, "dur us", (tsb[cidx, 4] - tsb[cidx, 0]) / 1e3, "items", tsb[cidx, 5], "per-warp (tag, full, comp, ep):", np.round(wt[cidx, :, :], 1).tolist()[:2], "epi (barrier, tree, ticket, merge):", np.round(epi[cidx], 1))
print("mean over warps/CTAs:", np.round(wt.mean((0, 1)), 2), "max:", np.round(wt.max((0, 1)), 2))
t0 = tsb[:, 0].min()
r = (tsb[:, :5] - t0) / 1e3
tsb = tsb[:, :8]
print("per-CTA us: start, prologue, producer_done, consumers_done(last unit), epilogue_done; items")
for i in list(range(0, nsm, 16)) + [nsm - 1]:
    print(i, np.round(r[i], 2), tsb[i, 5])
print("max:", np.round(r.max(0), 2), "median:", np.round(np.median(r, 0), 2))
