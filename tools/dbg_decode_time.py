"""Per-CTA globaltimer stamps of C5-shaped decode launches (WQ_DECODE_DEBUG bit 8 plus
optional mode bits from DBG, e.g. DBG=19 for the no-copy/no-math/no-epilogue skeleton)."""
import math, sys, os
os.environ.setdefault("WQ_VARIANT", "prof")   # timestamps need a WQ_DEC_PROFILE=1 build
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_02262_b200 import configs, synth, wq
import oracle
_c = os.environ.get("CFG", "C5")
cfg = configs.CONFIGS[_c] if _c in configs.CONFIGS else configs.c4(int(_c[3:])); m = cfg.model
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
NW = int(os.environ.get("NW", "11"))
TS = 200
TSB = TS * 8
for mode in [int(x) for x in os.environ.get("DBG", "0").split(",")]:
    os.environ["WQ_DECODE_DEBUG"] = str(8 | mode)
    for it in range(4):
        ws[-nsm * TSB:].zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); wq.wq_decode_attention(q, packed, offs, seg[l].contiguous(), g, kr, vr, rest_len, 1 / math.sqrt(m.d), out=out, workspace=ws); e1.record()
        torch.cuda.synchronize()
    print(f"=== mode {mode}: event us {e0.elapsed_time(e1) * 1e3:.1f}")
    tsb = ws[-nsm * TSB:].view(torch.int64).view(nsm, TS).cpu().numpy().astype(np.float64)
    t0 = tsb[:, 0].min()
    st = (tsb[:, :5] - t0) / 1e3
    st[tsb[:, :5] == 0] = np.nan
    wt = tsb[:, 8:8 + 4 * NW].reshape(nsm, NW, 4) / 1965.0   # SM cycles -> us
    print("per-CTA us (start, prologue done, producer done, consumers done, end) min/median/max:")
    for k, nm in enumerate(["start", "prologue", "producer", "loop_end", "end"]):
        print(f"  {nm:9s} {np.nanmin(st[:, k]):7.2f} {np.nanmedian(st[:, k]):7.2f} {np.nanmax(st[:, k]):7.2f}")
    print("per-warp us (full-wait, compute, epilogue, loop total) mean/max:", np.round(wt[:, :, :4].mean((0, 1)), 2), np.round(wt[:, :, :4].max((0, 1)), 2))
    print("epilogue CTA merge / ticket+merge us mean/max:", np.round(tsb[:, 68:70].mean(0) / 1965.0, 2), np.round(tsb[:, 68:70].max(0) / 1965.0, 2))
    print("items per CTA min/max:", tsb[:, 5].min(), tsb[:, 5].max())
    for k, nm in ((62, "producer start"), (60, "first publish"), (61, "warp0 loop start")):
        v = (tsb[:, k] - t0) / 1e3
        print(f"  {nm:18s} min/median/max us: {v.min():.2f} {np.median(v):.2f} {v.max():.2f}")
    dur = (tsb[:, 4] - tsb[:, 0]) / 1e3
    order = np.argsort(-dur)
    print("CTAs by loop end: (cta, end us, loop_end us, producer us, last?, k, items, class counts 2/4/8/16/rest)")
    lo = np.argsort(-st[:, 3])
    for cta in list(lo[:8]) + list(lo[-4:]):
        print("   ", cta, round(st[cta, 4], 2), round(st[cta, 3], 2), round(st[cta, 2], 2), int(tsb[cta, 6]), int(tsb[cta, 7]), int(tsb[cta, 5]), tsb[cta, 63:68].astype(int).tolist())
    # least-squares per-class item time (CTA-level us per item): loop duration ~ sum n_k t_k + c
    n = tsb[:, 63:68]
    dur_loop = st[:, 3] - (tsb[:, 61] - t0) / 1e3
    A = np.concatenate([n, np.ones((nsm, 1))], 1)
    ok = np.isfinite(dur_loop)
    sol, *_ = np.linalg.lstsq(A[ok], dur_loop[ok], rcond=None)
    print("fit us/item (2,4,8,16,rest) + const:", np.round(sol, 4), " resid rms", round(float(np.sqrt(np.mean((A[ok] @ sol - dur_loop[ok]) ** 2))), 3))
    ref70 = tsb[:, 70]
    print("producer setup cycles after prologue (median, max): entry / geo / items / planned")
    for k in (55, 57, 58, 56):
        print("   ", k, np.median(tsb[:, k] - ref70), np.max(tsb[:, k] - ref70))
    slow = int(np.nanargmax(st[:, 3]))
    print("slowest CTA", slow)
    for cta in (0, slow):
        ref = tsb[cta, 70]
        pi = tsb[cta, 72:136]; fd = tsb[cta, 136:200]
        n = int((pi > 0).sum())
        print(f"CTA {cta} stage trace (cycles after prologue): producer issue / warp0 full-done")
        print("   ", [int(x - ref) if x > 0 else -1 for x in pi[:n]])
        print("   ", [int(x - ref) if x > 0 else -1 for x in fd[:n]])
