"""Per-CTA globaltimer stamps of decode launches in the bench's launch pattern: a chain of
PDL-dependent decodes (WQ_DECODE_EARLY after the first) over rotated layer images, the
last TWO launches each with their own workspace, so both timelines share one clock.
Shows where a launch's time goes between the previous launch's last CTA and its own.
Needs the profiling build: WQ_VARIANT=prof WQ_NVCC_DEFS=-DWQ_DEC_PROFILE=1."""
import math
import os
import sys

os.environ.setdefault("WQ_VARIANT", "prof")
os.environ["WQ_DECODE_DEBUG"] = "8"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_02262_b200 import configs, synth, wq  # noqa: E402

_c = os.environ.get("CFG", "C5")
cfg = configs.CONFIGS[_c] if _c in configs.CONFIGS else configs.c4(int(_c[3:]))
m = cfg.model
dev = "cuda"
L = int(os.environ.get("LAYERS", "4"))
vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, dev)
g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
sc = wq.wq_window_scores(vis, txt, cfg.S)
del vis, txt
thr = wq.wq_thresholds(cfg.sensitivities()[:L], cfg.alpha, len(cfg.widths))
bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, L, g, wq.AssignOpts(cfg.budget, 1, 0))
layers = []
for l in range(L):
    K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, dev)
    offs = wq.wq_layer_layout(g, seg[l])
    packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
    wq.wq_reorder_quantize_pack(K, V, 0, g, perm[l], seg[l], offs, packed)
    del K, V
    q = synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, l, 0, dev)
    layers.append((packed, offs, seg[l].contiguous(), kr, vr, rest_len, q))
nsm = torch.cuda.get_device_properties(0).multi_processor_count
nb = wq.wq_decode_workspace(g)
wss = [torch.zeros(nb, dtype=torch.uint8, device=dev) for _ in range(3)]
out = torch.empty((cfg.B, m.Hq, m.d), dtype=torch.float16, device=dev)
sm = 1.0 / math.sqrt(m.d)
TS = 200
N = 4 * L


def launch(i, ws):
    packed, offs, segl, kr, vr, rest_len, q = layers[i % L]
    wq.wq_decode_attention(q, packed, offs, segl, g, kr, vr, rest_len, sm, out=out, workspace=ws,
                           flags=(wq.WQ_DECODE_EARLY if i else 0))


for rep in range(3):
    for w in wss[1:]:
        w[-nsm * TS * 8:].zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(N):
        launch(i, wss[0] if i < N - 2 else wss[1 + (i - (N - 2))])
    e1.record()
    torch.cuda.synchronize()
print(f"{_c}: {N} PDL-chained launches, {e0.elapsed_time(e1) * 1e3 / N:.2f} us/launch (event, incl. profiling)")
st = []
for w in wss[1:]:
    st.append(w[-nsm * TS * 8:].view(torch.int64).view(nsm, TS).cpu().numpy().astype(np.float64))
A, B = st
t0 = A[:, 0].min()
names = [(0, "CTA start"), (1, "prologue done"), (61, "warp0 loop start"), (3, "loop end"), (4, "CTA end")]
for tag, X in (("launch N-1", A), ("launch N", B)):
    print(tag)
    for k, nm in names:
        v = (X[:, k] - t0) / 1e3
        v = v[X[:, k] > 0]
        if v.size:
            print(f"   {nm:17s} min {v.min():7.2f}  median {np.median(v):7.2f}  max {v.max():7.2f} us  (n={v.size})")
endA = (A[:, 4].max() - t0) / 1e3
ls = (B[:, 61][B[:, 61] > 0] - t0) / 1e3
le = (B[:, 3][B[:, 3] > 0] - t0) / 1e3
en = (B[:, 4][B[:, 4] > 0] - t0) / 1e3
print(f"N-1 last CTA end -> N first loop start {ls.min() - endA:.2f} us, median loop start {np.median(ls) - endA:.2f}")
print(f"N loop: median {np.median(le - np.median(ls)):.2f} us after median start; loop end spread "
      f"{le.min() - endA:.2f} .. {le.max() - endA:.2f} us after N-1's end; N end max {en.max() - endA:.2f}")
cw = (B[:, 4] - B[:, 3]) / 1e3
print(f"N epilogue (loop end -> CTA end): median {np.median(cw):.2f}  max {cw.max():.2f} us; "
      f"last-CTA flags {int(B[:, 6].sum())}")
for k, nm in ((53, "N griddep_wait returned"), (54, "N q staged")):
    v = (B[:, k][B[:, k] > 0] - t0) / 1e3
    if v.size:
        print(f"   {nm:24s} min {v.min() - endA:6.2f} median {np.median(v) - endA:6.2f} max {v.max() - endA:6.2f} us after N-1's end")
lo = np.argsort(-B[:, 3])
print("N CTAs by loop end (cta, loop_end, end after N-1's end us, last?, k-th CTA of unit, items, counts 2/4/8/16/rest):")
for cta in list(lo[:10]) + list(lo[-6:]):
    print("   ", cta, round((B[cta, 3] - t0) / 1e3 - endA, 2), round((B[cta, 4] - t0) / 1e3 - endA, 2), int(B[cta, 6]),
          int(B[cta, 7]), int(B[cta, 5]), B[cta, 63:68].astype(int).tolist())
n = B[:, 63:68]
ls0 = B[:, 61]
dur = (B[:, 3] - ls0) / 1e3
Am = np.concatenate([n, np.ones((nsm, 1))], 1)
ok = (B[:, 3] > 0) & (ls0 > 0)
sol, *_ = np.linalg.lstsq(Am[ok], dur[ok], rcond=None)
print("fit us/item (2,4,8,16,rest) + const:", np.round(sol, 4), " resid rms",
      round(float(np.sqrt(np.mean((Am[ok] @ sol - dur[ok]) ** 2))), 3))
