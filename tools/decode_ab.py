"""A/B timing of decode-kernel build variants on the SAME inputs in ONE process.

usage: python tools/decode_ab.py [--cfg C5] [--layers 8] [--tokens 10] [--rounds 6] VARIANT ...
VARIANT "" (or "prod") is the product library lib/libwq.so, any other name lib/<name>/libwq.so
(built with WQ_VARIANT=<name> WQ_NVCC_DEFS="..." python -m paper_2605_02262_b200.build).
Each variant's wq_decode_attention_ex is loaded side by side (ctypes, RTLD_LOCAL) and timed
in the bench's launch pattern -- layers x tokens PDL-chained decodes (WQ_DECODE_EARLY after
the first) over rotated layer images (> L2) -- in interleaved rounds; prints the median
per-launch microseconds of each variant, so box-to-box noise cancels."""
import argparse
import ctypes as C
import math
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
    ap.add_argument("--tokens", type=int, default=10)
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
    layers = []
    for l in range(L):
        K, V, kr, vr, rest_len = synth.layer_tensors(cfg, l, dev)
        offs = wq.wq_layer_layout(g, seg[l])
        packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
        wq.wq_reorder_quantize_pack(K, V, 0, g, perm[l], seg[l], offs, packed)
        del K, V
        qs = [synth.queries(cfg.B, m.Hq, m.H, m.d, cfg.seed, l, t, dev) for t in range(a.tokens)]
        layers.append((packed, offs, seg[l].contiguous(), kr, vr, rest_len, qs))
    torch.cuda.synchronize()
    sm = 1.0 / math.sqrt(m.d)
    libs = {}
    for v in a.variants:
        path = wq.lib_path() if v in ("", "prod") else os.path.join(ROOT, "paper_2605_02262_b200", "lib", v, "libwq.so")
        lib = C.CDLL(path)
        P = C.c_void_p
        lib.wq_decode_attention_ex.argtypes = [P, P, P, P, C.POINTER(wq.Geom), P, P, P, P, C.c_int32, C.c_float, P, P,
                                               P, C.c_size_t, C.c_uint32, P]
        lib.wq_decode_attention_ex.restype = C.c_int
        lib.wq_decode_workspace.argtypes = [C.POINTER(wq.Geom), P]
        n = C.c_size_t(0)
        assert lib.wq_decode_workspace(C.byref(g), C.byref(n)) == 0
        ws = torch.zeros(n.value, dtype=torch.uint8, device=dev)
        libs[v] = (lib, ws)
    out = torch.empty((cfg.B, m.Hq, m.d), dtype=torch.float16, device=dev)
    stream = torch.cuda.current_stream()

    def run(v):
        lib, ws = libs[v]
        first = True
        for t in range(a.tokens):
            for (packed, offs, segl, kr, vr, rest_len, qs) in layers:
                rs = (C.c_int64 * 2)(kr.stride(0), kr.stride(1))
                rc = lib.wq_decode_attention_ex(C.c_void_p(qs[t].data_ptr()), C.c_void_p(packed.data_ptr()),
                                                C.c_void_p(offs.data_ptr()), C.c_void_p(segl.data_ptr()), C.byref(g),
                                                C.c_void_p(kr.data_ptr()), C.c_void_p(vr.data_ptr()), rs,
                                                C.c_void_p(rest_len.data_ptr()), kr.shape[2], sm,
                                                C.c_void_p(out.data_ptr()), None, C.c_void_p(ws.data_ptr()),
                                                ws.numel(), 0 if first else 1, C.c_void_p(stream.cuda_stream))
                assert rc == 0, v
                first = False

    times = {v: [] for v in a.variants}
    for v in a.variants:
        run(v)
    torch.cuda.synchronize()
    for r in range(a.rounds):
        for v in a.variants:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(v)
            e1.record()
            torch.cuda.synchronize()
            times[v].append(e0.elapsed_time(e1) * 1e3 / (a.tokens * L))
    for v in a.variants:
        t = times[v]
        print(f"{v or 'prod':14s} median {statistics.median(t):7.2f} us/launch  min {min(t):7.2f}  max {max(t):7.2f}",
              flush=True)


if __name__ == "__main__":
    main()
