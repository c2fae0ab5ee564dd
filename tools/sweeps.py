"""Parameter sweeps of the paper reproduced on B200 with the GPU path.

* alpha sweep (Fig. thre_para, P:919-932 / P:960-962; Eq.10-11): C5 shape, for alpha in
  {0.5, 1, 2, 4, 8}: tokens per width (the paper: as alpha grows INT2 and FP16 shrink and
  INT4 grows) and the decode time per layer call (Fig. thre_para (a) is generation latency).
* window-size sweep (Fig. window_size; BASELINE config C4, B = 64): for S in
  {16, 32, 64, 128}: tokens per width, quantize and decode time per layer call.

Times are CUDA-event device times over NL rotated layers (every image >> L2 for C4;
C5 images are ~104 MB each, 4 layers rotated).  Writes a table to stdout and, with --out,
a JSON file.  usage: python tools/sweeps.py [--out profiles/r01_sweeps.json]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_02262_b200 import configs, synth, wq  # noqa: E402


def timed(fn, n, reps=5):
    for i in range(n):
        fn(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for i in range(n):
            fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * n)


def run_cfg(cfg, alpha, NL, dev):
    m = cfg.model
    g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, dev)
    sc = wq.wq_window_scores(vis, txt, cfg.S)
    del vis, txt
    thr = wq.wq_thresholds([0.5] * NL, alpha, len(cfg.widths))
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, NL, g, wq.AssignOpts(0.0, 1, 0))
    layers = []
    for l in range(NL):
        K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, dev)
        q = synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, l, device=dev)
        offs = wq.wq_layer_layout(g, seg[l])
        packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
        layers.append(dict(K=K, V=V, kr=kr, vr=vr, rl=rest_len, q=q, offs=offs, packed=packed))
    ws = torch.zeros(wq.wq_decode_workspace(g), dtype=torch.uint8, device=dev)
    out = torch.empty((cfg.B, m.Hq, m.d), dtype=torch.float16, device=dev)
    sm = 1.0 / math.sqrt(m.d)

    def quant(i):
        L = layers[i]
        wq.wq_reorder_quantize_pack(L["K"], L["V"], 0, g, perm[i], seg[i], L["offs"], L["packed"])

    def dec(i):
        L = layers[i]
        wq.wq_decode_attention(L["q"], L["packed"], L["offs"], seg[i], g, L["kr"], L["vr"], L["rl"], sm, out=out,
                               workspace=ws)

    t_q = timed(quant, NL)
    t_d = timed(dec, NL)
    s = seg[:NL].cpu()
    per_class = (s[:, :, 1:] - s[:, :, :-1]).sum(dim=(0, 1)).tolist()          # windows of width 2/4/8/16
    tokens = {str(b): int(n) * cfg.S // NL for b, n in zip((2, 4, 8, 16), per_class)}   # per layer, all requests
    img_mb = sum(int(L["offs"][-1].item()) for L in layers) / NL / 1e6
    return {"tokens_per_width": tokens, "quantize_us": round(t_q, 1), "decode_us": round(t_d, 2),
            "packed_MB_per_layer": round(img_mb, 1),
            "decode_GBps": round(img_mb * 1e6 / (t_d * 1e-6) / 1e9, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda")
    wq.load()
    res = {"alpha_sweep_C5": {}, "window_sweep_C4": {}}
    c5 = configs.CONFIGS["C5"]
    print("alpha sweep, C5 shape (B=4, 50,176 visual tokens, widths 2/4/8/16), per layer call:")
    print(f"{'alpha':>6s} {'INT2':>8s} {'INT4':>8s} {'INT8':>8s} {'FP16':>6s} {'image MB':>9s} {'decode us':>10s}")
    for a in (0.5, 1.0, 2.0, 4.0, 8.0):
        r = run_cfg(c5, a, 4, dev)
        res["alpha_sweep_C5"][str(a)] = r
        t = r["tokens_per_width"]
        print(f"{a:6.1f} {t['2']:8d} {t['4']:8d} {t['8']:8d} {t['16']:6d} {r['packed_MB_per_layer']:9.1f} "
              f"{r['decode_us']:10.2f}")
        torch.cuda.empty_cache()
    print("\nwindow-size sweep, C4 shape (B=64, 11,760 visual tokens, alpha 2), per layer call:")
    print(f"{'S':>4s} {'INT2':>8s} {'INT4':>8s} {'INT8':>8s} {'FP16':>7s} {'image MB':>9s} {'quant us':>9s} "
          f"{'decode us':>10s} {'dec GB/s':>9s}")
    for S in (16, 32, 64, 128):
        r = run_cfg(configs.c4(S), 2.0, 2, dev)
        res["window_sweep_C4"][str(S)] = r
        t = r["tokens_per_width"]
        print(f"{S:4d} {t['2']:8d} {t['4']:8d} {t['8']:8d} {t['16']:7d} {r['packed_MB_per_layer']:9.1f} "
              f"{r['quantize_us']:9.1f} {r['decode_us']:10.2f} {r['decode_GBps']:9.1f}")
        torch.cuda.empty_cache()
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
