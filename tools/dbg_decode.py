"""Debug harness: small decode cases vs the oracle, per-row error report."""
import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2605_02262_b200 import synth, wq

def case(seed, B, H, Hq, d, S, W, tail, R, widths=(2, 4, 8, 16), force=None):
    M = W * S + tail
    K, V = synth.kv_layer(B, H, M, d, S, seed, 0, "cuda")
    kr, vr = synth.rest_layer(B, H, R, d, seed, 0, "cuda")
    rest_len = torch.tensor([max(R - 3 * b, 0) for b in range(B)], dtype=torch.int32, device="cuda")
    q = synth.queries(B, Hq, H, d, seed, 0, device="cuda")
    g = wq.geom(B, H, Hq, d, M, S, widths)
    og = oracle.geom(B, H, Hq, d, M, S, list(widths))
    rng = np.random.default_rng(seed)
    if force is None:
        sims = rng.uniform(0, 1, (B, W))
        thr = oracle.thresholds([0.45], 2.0, len(widths))
        _, _, perm, seg = oracle.assign_bits(sims, thr, og)
        perm, seg = perm[0], seg[0]
    else:
        k = {2: 0, 4: 1, 8: 2, 16: 3}[force]
        perm = np.tile(np.arange(W, dtype=np.int32), (B, 1))
        seg = np.zeros((B, 5), np.int32); seg[:, k + 1:] = W
    perm_t = torch.tensor(perm, device="cuda"); seg_t = torch.tensor(seg, device="cuda")
    offs = wq.wq_layer_layout(g, seg_t)
    packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device="cuda")
    wq.wq_reorder_quantize_pack(K, V, 0, g, perm_t, seg_t, offs, packed)
    out = torch.zeros((B, Hq, d), dtype=torch.float16, device="cuda")
    part = torch.zeros((B, Hq, d + 2), dtype=torch.float32, device="cuda")
    sm = 1 / math.sqrt(d)
    wq.wq_decode_attention(q, packed, offs, seg_t, g, kr, vr, rest_len, sm, out=out, partial=part)
    torch.cuda.synchronize()
    ref, rp = oracle.decode_attention(q.cpu().numpy(), packed.cpu().numpy(), offs.cpu().numpy(), seg, perm, og,
                                      kr.cpu().numpy(), vr.cpu().numpy(), rest_len.cpu().numpy(), sm, want_partial=True)
    got = out.float().cpu().numpy()
    err = np.abs(got - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
    p = part.double().cpu().numpy()
    print(f"B{B} H{H} Hq{Hq} d{d} S{S} W{W} tail{tail} R{R} force={force}: max rel err {err.max():.3e}", flush=True)
    if err.max() > 2e-3:
        for b in range(B):
            print("  b", b, "err per hq", np.array2string(err[b], precision=2), "m gpu", np.round(p[b, :, 0], 3), "m ref", np.round(rp[b, :, 0], 3))
            print("     l gpu", np.round(p[b, :, 1], 3), "l ref", np.round(rp[b, :, 1], 3))

for f in (16, 2, 4, 8, None):
    case(1, 1, 1, 7, 64, 16, 3, 0, 0, force=f)
case(2, 1, 1, 7, 64, 16, 3, 0, 5)
case(3, 1, 1, 7, 128, 32, 4, 0, 0, force=2)
case(4, 2, 2, 14, 64, 16, 9, 5, 21)
case(5, 2, 4, 28, 128, 32, 12, 7, 21)
