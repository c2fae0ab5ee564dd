"""GPU parity of the paper-literal group quantizer (WQ_GRAN_GROUP, §8(f) row 3; reading
Q37 of DESIGN.md): one (s, mn) per (window, KV head, K|V) group over its S*d values
("grouped by sliding windows", Eq.14-16 per group), record = codes + a 16-byte
{mn_K, s_K, mn_V, s_V} block.  Packed images are byte-exact with the oracle's gran = 1,
decode attention under WQ_DECODE_GROUP within 2e-3 of the oracle's gran = 1 decode.
Edge windows are whole degenerate groups (constant, signed zeros, subnormal range, fp16
extremes, all codes at q_max but one)."""
import ctypes as C
import math

import numpy as np
import pytest
import torch

from paper_2605_02262_b200 import synth, wq

pytestmark = pytest.mark.gpu
ATTN_TOL = 2e-3
CLASS = (2, 4, 8, 16)
GRP = wq.WQ_GRAN_GROUP


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    wq.load()


def rel_err(got, ref):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return float((np.abs(got - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)).max())


def plan(bits):
    """perm / seg_off of per-request width lists (class-major, window order inside)."""
    B, W = len(bits), len(bits[0])
    perm = np.zeros((B, W), np.int32)
    seg = np.zeros((B, 5), np.int32)
    for b in range(B):
        perm[b] = [w for k in CLASS for w in range(W) if bits[b][w] == k]
        n = 0
        for i, k in enumerate(CLASS):
            seg[b, i] = n
            n += sum(1 for x in bits[b] if x == k)
        seg[b, 4] = n
    return perm, seg


def run(c, gran=GRP, flags=0):
    dev = "cuda"
    g = wq.geom(c["B"], c["H"], c["Hq"], c["d"], c["M"], c["S"], CLASS)
    K, V = torch.as_tensor(c["K"]).to(dev), torch.as_tensor(c["V"]).to(dev)
    perm, seg = torch.from_numpy(c["perm"]).to(dev), torch.from_numpy(c["seg"]).to(dev)
    offs = wq.wq_layer_layout(g, seg, gran=gran)
    packed = torch.zeros(int(offs[-1].item()) + 16, dtype=torch.uint8, device=dev)
    wq.wq_reorder_quantize_pack(K, V, 0, g, perm, seg, offs, packed, gran=gran)
    out = torch.empty((c["B"], c["Hq"], c["d"]), dtype=torch.float16, device=dev)
    part = torch.empty((c["B"], c["Hq"], c["d"] + 2), dtype=torch.float32, device=dev)
    wq.wq_decode_attention(torch.as_tensor(c["q"]).to(dev), packed, offs, seg, g, torch.as_tensor(c["kr"]).to(dev),
                           torch.as_tensor(c["vr"]).to(dev), torch.from_numpy(c["rest_len"]).to(dev),
                           1 / math.sqrt(c["d"]), out=out, partial=part,
                           flags=flags | (wq.WQ_DECODE_GROUP if gran else 0))
    torch.cuda.synchronize()
    return offs.cpu().numpy(), packed.cpu().numpy(), out.float().cpu().numpy(), part.double().cpu().numpy()


def oracle(orc, c):
    og = orc.geom(c["B"], c["H"], c["Hq"], c["d"], c["M"], c["S"], list(CLASS))
    K, V = np.asarray(c["K"].cpu() if torch.is_tensor(c["K"]) else c["K"]), \
        np.asarray(c["V"].cpu() if torch.is_tensor(c["V"]) else c["V"])
    opk, ooffs = orc.reorder_quantize_pack(K, V, 0, og, c["perm"], c["seg"], gran=1)
    q = np.asarray(c["q"].cpu() if torch.is_tensor(c["q"]) else c["q"])
    kr = np.asarray(c["kr"].cpu() if torch.is_tensor(c["kr"]) else c["kr"])
    vr = np.asarray(c["vr"].cpu() if torch.is_tensor(c["vr"]) else c["vr"])
    ref, rpart = orc.decode_attention(q, opk, ooffs, c["seg"], c["perm"], og, kr, vr, c["rest_len"],
                                      1 / math.sqrt(c["d"]), want_partial=True, gran=1)
    return opk, ooffs, ref, rpart


def synth_case(seed, B, H, Hq, d, S, W, tail, R=21):
    M = W * S + tail
    K, V = synth.kv_layer(B, H, M, d, S, seed, 0, "cuda")
    kr, vr = synth.rest_layer(B, H, R, d, seed, 0, "cuda")
    q = synth.queries(B, Hq, H, d, seed, 0, device="cuda")
    rng = np.random.default_rng(seed)
    bits = [list(rng.choice(CLASS, W, p=[0.4, 0.3, 0.2, 0.1])) for _ in range(B)]
    perm, seg = plan(bits)
    rest_len = np.array([max(R - 4 * b, 0) for b in range(B)], np.int32)
    return dict(B=B, H=H, Hq=Hq, d=d, S=S, M=M, K=K, V=V, kr=kr, vr=vr, q=q, perm=perm, seg=seg, rest_len=rest_len)


def edge_ok(got, ref):
    """Degenerate groups: |err| <= 2e-3 * (row max |ref|) + 2^-16.  The absolute term is the
    fp16 P' = p * s_V operand underflowing when s_V is subnormal (a zero / constant /
    subnormal V group: s_V = 2^-24..2^-14), worth at most 2^(b-1) * 2^-24 of a row whose
    exact output is ~0 (include/wq.h, decode numerical domain)."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return bool((np.abs(got - ref) <= 2e-3 * np.abs(ref).max(-1, keepdims=True) + 2.0 ** -16).all())


def check(orc, c, attn=True, edge=False):
    offs, packed, out, part = run(c)
    opk, ooffs, ref, rpart = oracle(orc, c)
    assert np.array_equal(offs, ooffs)
    n = int(ooffs[-1])
    bad = np.nonzero(packed[:n] != opk[:n])[0]
    assert bad.size == 0, f"{bad.size} bytes differ, first at {bad[:8]}"
    if attn and edge:
        assert edge_ok(out, ref)
        assert edge_ok(part[..., 2:] / part[..., 1:2], ref)
    elif attn:
        assert rel_err(out, ref) <= ATTN_TOL
        assert rel_err(part[..., 2:] / part[..., 1:2], ref) <= ATTN_TOL
        lse, rlse = part[..., 0] + np.log(part[..., 1]), rpart[..., 0] + np.log(rpart[..., 1])
        assert np.max(np.abs(lse - rlse)) < 1e-3


@pytest.mark.parametrize("d,S,W,tail,B,H,Hq", [(64, 16, 9, 5, 2, 2, 14), (64, 32, 17, 0, 3, 2, 14),
                                               (128, 32, 12, 7, 2, 4, 28), (128, 64, 5, 0, 1, 4, 28),
                                               (128, 128, 3, 9, 2, 2, 8), (64, 64, 6, 1, 2, 1, 5),
                                               (128, 16, 30, 0, 4, 4, 28), (64, 128, 2, 0, 1, 2, 4)])
def test_group_bytes_and_decode(orc, d, S, W, tail, B, H, Hq):
    check(orc, synth_case(900 + d + S + W, B, H, Hq, d, S, W, tail))


def test_group_early_flag(orc):
    """WQ_DECODE_EARLY | WQ_DECODE_GROUP: same outputs as WQ_DECODE_GROUP alone."""
    c = synth_case(5, 2, 4, 28, 128, 32, 12, 7)
    _, _, o1, p1 = run(c)
    _, _, o2, p2 = run(c, flags=wq.WQ_DECODE_EARLY)
    assert np.array_equal(o1, o2) and np.array_equal(p1, p2)


def test_group_empty_and_all16(orc):
    """An all-FP16 request next to a quantized one; then a request with no slots at all
    (seg_off all zero: an empty image) and no rest tokens next to a quantized one."""
    c = synth_case(6, 2, 2, 14, 64, 16, 6, 0)
    bits = [[16] * 6, [2, 4, 8, 2, 4, 8]]
    c["perm"], c["seg"] = plan(bits)
    check(orc, c)
    c["seg"][0] = 0
    c["rest_len"] = np.array([3, 0], np.int32)
    check(orc, c)


def edge_window(rng, kind, S, d, ext):
    """One (window, head) group [S][d] of a degenerate kind."""
    x = rng.standard_normal((S, d)).astype(np.float16)
    if kind == "const":
        x[:] = 1.5
    elif kind == "zero_pos_first":
        x = rng.choice([0.25, 0.5, 1.0], (S, d)).astype(np.float16)
        x[0, 0], x[S - 1, d - 1] = np.float16(0.0), np.float16(-0.0)
    elif kind == "zero_neg_first":
        x = rng.choice([0.25, 0.5, 1.0], (S, d)).astype(np.float16)
        x[0, 0], x[S - 1, d - 1] = np.float16(-0.0), np.float16(0.0)
    elif kind == "only_neg_zero":
        x = np.where(rng.random((S, d)) < 0.5, np.float16(-0.0), np.float16(2.0)).astype(np.float16)
    elif kind == "subnormal":
        x = rng.choice(np.array([0, 2 ** -24, 2 ** -23, 3 * 2 ** -24], np.float16), (S, d))
    elif kind == "qmax_but_one":
        x[:] = 1.0
        x[S // 2, d // 3] = 0.0
    elif kind == "extreme":
        x = (rng.choice([-1.0, 1.0], (S, d)) * ext).astype(np.float16)
        x[0, 0], x[0, 1] = ext, -ext
    elif kind == "zeros":
        x[:] = 0.0
    return x


KINDS = ["const", "zero_pos_first", "zero_neg_first", "only_neg_zero", "subnormal", "qmax_but_one", "extreme",
         "zeros"]


def edge_case(d, S, ext, seed):
    rng = np.random.default_rng(seed)
    B, H, W, R = 2, 2 if d == 64 else 4, len(KINDS), 13
    Hq = 7 * H
    M = W * S
    K = np.zeros((B, H, M, d), np.float16)
    V = np.zeros((B, H, M, d), np.float16)
    for b in range(B):
        for h in range(H):
            for w in range(W):
                kk = KINDS[(w + h + b) % W]
                K[b, h, w * S:(w + 1) * S] = edge_window(rng, kk, S, d, ext)
                V[b, h, w * S:(w + 1) * S] = edge_window(rng, KINDS[(w + 3 * h + b + 1) % W], S, d, ext)
    bits = [[2, 4, 8, 2, 4, 8, 16, 2], [8, 4, 2, 2, 16, 4, 8, 2]]
    perm, seg = plan(bits)
    q = (0.3 * rng.standard_normal((B, Hq, d))).astype(np.float16)
    kr = rng.standard_normal((B, H, R, d)).astype(np.float16)
    vr = rng.standard_normal((B, H, R, d)).astype(np.float16)
    return dict(B=B, H=H, Hq=Hq, d=d, S=S, M=M, K=K, V=V, perm=perm, seg=seg, q=q, kr=kr, vr=vr,
                rest_len=np.array([5, 13], np.int32))


@pytest.mark.parametrize("d,S", [(128, 32), (64, 16), (128, 128), (64, 64)])
def test_group_edges_bytes_at_fp16_extremes(orc, d, S):
    check(orc, edge_case(d, S, 65504.0, d + S), attn=False)


@pytest.mark.parametrize("d,S", [(128, 32), (64, 16), (128, 128), (64, 64)])
def test_group_edges_in_domain(orc, d, S):
    """Extremes +-250 keep s_V < 255 for every width (the WQ_DECODE_GROUP domain)."""
    check(orc, edge_case(d, S, 250.0, 3 * d + S), edge=True)


def test_group_signed_zero_param_block(orc):
    """A group whose minimum is a zero stores mn = 0x8000 when a -0 is present (Q17
    IEEE minimum), in either element order; read back from the 16-byte block."""
    for kind in ("zero_pos_first", "zero_neg_first"):
        c = edge_case(64, 16, 4.0, 41)
        rng = np.random.default_rng(3)
        for w in range(len(KINDS)):
            c["K"][0, 0, w * 16:(w + 1) * 16] = edge_window(rng, kind, 16, 64, 4.0)
        offs, packed, _, _ = run(c)
        opk, ooffs, _, _ = oracle(orc, c)
        assert np.array_equal(packed[:int(ooffs[-1])], opk[:int(ooffs[-1])])
        rec = packed[int(offs[0]):]
        kbytes = 16 * 64 * 2 // 8                  # first record of (0, 0) is 2-bit
        mn_k = int(rec[2 * kbytes]) | (int(rec[2 * kbytes + 1]) << 8)
        assert mn_k == 0x8000
        assert not rec[2 * kbytes + 8:2 * kbytes + 16].any()


def test_group_packed_bytes_and_errors():
    g = wq.geom(2, 4, 28, 128, 12 * 32, 32, CLASS)
    n = [3, 2, 1, 4]
    assert wq.wq_packed_bytes(g, n, gran=GRP) == sum(k * (32 * 128 * b // 4 + (16 if b < 16 else 0))
                                                     for k, b in zip(n, CLASS))
    assert wq.wq_packed_bytes(g, n, True, gran=GRP) == wq.wq_packed_bytes(g, n, True)
    L = wq.load()
    out = C.c_int64(0)
    narr = (C.c_int32 * 4)(*n)
    assert L.wq_packed_bytes_ex(C.byref(g), narr, 0, 2, C.byref(out)) == wq.WQ_EINVAL
    seg = torch.zeros((2, 5), dtype=torch.int32, device="cuda")
    offs = torch.zeros(9, dtype=torch.int64, device="cuda")
    assert L.wq_layer_layout_ex(C.byref(g), C.c_void_p(seg.data_ptr()), 7, C.c_void_p(offs.data_ptr()),
                                None) == wq.WQ_EINVAL
    with pytest.raises(wq.WQError):
        wq.wq_reorder_quantize_pack(torch.zeros((2, 4, 384, 128), dtype=torch.float16, device="cuda"),
                                    torch.zeros((2, 4, 384, 128), dtype=torch.float16, device="cuda"), 0, g,
                                    torch.zeros((2, 12), dtype=torch.int32, device="cuda"), seg, offs,
                                    torch.zeros(64, dtype=torch.uint8, device="cuda"), gran=-1)
