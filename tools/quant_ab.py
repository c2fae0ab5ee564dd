"""A/B timing of wq_reorder_quantize_pack build variants on the SAME inputs in ONE process
(as tools/decode_ab.py): L layers' quantize launches back to back (each layer's K/V and
image > L2), interleaved rounds, median microseconds per launch and GB/s of algorithmic
bytes (read 4*S*d per window-head + write the record).
usage: python tools/quant_ab.py [--cfg C5] [--layers 8] [--rounds 6] VARIANT ..."""
import argparse
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_02262_b200 import configs, synth, wq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C5")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("variants", nargs="*", default=["prod"])
    a = ap.parse_args()
    cfg = configs.CONFIGS[a.cfg] if a.cfg in configs.CONFIGS else configs.c4(int(a.cfg[3:]))
    m = cfg.model
    wq.load()
    dev = "cuda"
    L = min(a.layers, cfg.layers)
    vis, txt = synth.embeddings(cfg.B, cfg.M, cfg.n_text, m.D, cfg.S, cfg.seed, dev)
    g = wq.geom(cfg.B, m.H, m.Hq, m.d, cfg.M, cfg.S, cfg.widths)
    sc = wq.wq_window_scores(vis, txt, cfg.S)
    del vis, txt
    thr = wq.wq_thresholds(cfg.sensitivities()[:L], cfg.alpha, len(cfg.widths))
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, L, g, wq.AssignOpts(cfg.budget, 1, 0))
    layers, nbytes = [], 0
    for l in range(L):
        K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, dev)
        offs = wq.wq_layer_layout(g, seg[l])
        tot = int(offs[-1].item())
        packed = torch.zeros(tot + 16, dtype=torch.uint8, device=dev)
        layers.append((K, V, perm[l].contiguous(), seg[l].contiguous(), offs, packed))
        nbytes += int(seg[l][:, 4].sum().item()) * m.H * cfg.S * m.d * 4 + tot
    torch.cuda.synchronize()
    libs = {}
    for v in a.variants:
        path = wq.lib_path() if v in ("", "prod") else os.path.join(ROOT, "paper_2605_02262_b200", "lib", v, "libwq.so")
        lib = C.CDLL(path)
        P = C.c_void_p
        lib.wq_reorder_quantize_pack.argtypes = [P, P, P, C.c_int32, C.POINTER(wq.Geom), P, C.c_int32, P, P, P, P]
        lib.wq_reorder_quantize_pack.restype = C.c_int
        libs[v] = lib
    stream = torch.cuda.current_stream()
    ref = None

    def run(v):
        lib = libs[v]
        for (K, V, pm, sg, offs, packed) in layers:
            st = (C.c_int64 * 3)(K.stride(0), K.stride(1), K.stride(2))
            rc = lib.wq_reorder_quantize_pack(C.c_void_p(K.data_ptr()), C.c_void_p(V.data_ptr()), st, 0, C.byref(g),
                                              C.c_void_p(pm.data_ptr()), pm.shape[1], C.c_void_p(sg.data_ptr()),
                                              C.c_void_p(offs.data_ptr()), C.c_void_p(packed.data_ptr()),
                                              C.c_void_p(stream.cuda_stream))
            assert rc == 0, v

    times = {v: [] for v in a.variants}
    for v in a.variants:
        run(v)
        torch.cuda.synchronize()
        img = layers[-1][5].clone()
        if ref is None:
            ref = img
        assert torch.equal(ref, img), f"variant {v} writes different bytes"
    for r in range(a.rounds):
        for v in a.variants:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(v)
            e1.record()
            torch.cuda.synchronize()
            times[v].append(e0.elapsed_time(e1) * 1e3 / L)
    for v in a.variants:
        t = statistics.median(times[v])
        print(f"{v or 'prod':10s} median {t:8.2f} us/launch  {nbytes / L / (t * 1e-6) / 1e9:7.1f} GB/s  "
              f"(min {min(times[v]):.2f} max {max(times[v]):.2f})", flush=True)


if __name__ == "__main__":
    main()
