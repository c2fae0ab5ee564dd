"""Repeat the decode edge-case flow and check quantize bytes + decode vs oracle each time."""
import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2605_02262_b200 import synth, wq
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import small_case, ogeom, rel_err
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    c = small_case(41, d=64, S=16, W=4, tail=0, B=3, H=2, Hq=14)
    g = c["g"]; sm = 0.125
    sc = wq.wq_window_scores(c["vis"], c["txt"], 16)
    thr = oracle.thresholds([0.5], 2.0, 4)
    bits, rank, perm, seg = wq.wq_assign_bits(sc, thr, 1, g)
    for rl in ([0, 0, 0], [1, 17, 33], [16, 15, 21]):
        rest_len = torch.tensor(rl, dtype=torch.int32, device="cuda")
        offs = wq.wq_layer_layout(g, seg[0])
        packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device="cuda")
        wq.wq_reorder_quantize_pack(c["K"], c["V"], 0, g, perm[0], seg[0], offs, packed)
        out = torch.empty((3, 14, 64), dtype=torch.float16, device="cuda")
        wq.wq_decode_attention(c["q"], packed, offs, seg[0], g, c["kr"], c["vr"], rest_len, sm, out=out)
        torch.cuda.synchronize()
        opk, ooffs = oracle.reorder_quantize_pack(c["K"].cpu().numpy(), c["V"].cpu().numpy(), 0, ogeom(oracle, g),
                                                  perm[0].cpu().numpy(), seg[0].cpu().numpy())
        n = int(ooffs[-1])
        pb = packed.cpu().numpy()[:n]
        qok = np.array_equal(pb, opk[:n])
        ref = oracle.decode_attention(c["q"].cpu().numpy(), opk, ooffs, seg[0].cpu().numpy(), perm[0].cpu().numpy(),
                                      ogeom(oracle, g), c["kr"].cpu().numpy(), c["vr"].cpu().numpy(), np.array(rl, np.int32), sm)
        e = rel_err(out.float().cpu().numpy(), ref)
        if not qok or not (e <= 2e-3):
            bad += 1
            diff = np.nonzero(pb != opk[:n])[0]
            print(f"it {it} rl {rl}: quant ok {qok} (first diff bytes {diff[:8]} of {len(diff)}), decode err {e}")
            o = out.float().cpu().numpy()
            rows = np.nonzero(np.abs(o - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6) > 2e-3)
            print("   bad rows (b, hq):", list(zip(rows[0].tolist(), rows[1].tolist()))[:20])
            for rep in range(4):
                out2 = torch.empty((3, 14, 64), dtype=torch.float16, device="cuda")
                part = torch.empty((3, 14, 66), dtype=torch.float32, device="cuda")
                wq.wq_decode_attention(c["q"], packed, offs, seg[0], g, c["kr"], c["vr"], rest_len, sm, out=out2, partial=part)
                torch.cuda.synchronize()
                e2 = rel_err(out2.float().cpu().numpy(), ref)
                print("   rerun", rep, "err", e2, "m,l of b2 hq7:", part[2, 7, :2].tolist(), "out b2h7[:4]", out2[2, 7, :4].tolist(), "ref", ref[2, 7, :4])
print("bad", bad)
