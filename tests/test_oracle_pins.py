"""Pins of the CPU oracle against what the paper and mathematics fix (not gpu).

Each test names the passage it follows.  Sources of expected values:
  * tests/golden/paper_pins.json  -- paper numbers / SPEC worked examples (cited)
  * closed forms derived by hand in the comments
  * independent library routines (numpy float16, numpy matmul) on tiny inputs
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


# --------------------------------------------------------------------------------------
# fp16 conversions (IEEE 754 binary16) vs numpy -- independent implementation
# --------------------------------------------------------------------------------------
def test_f16_to_f64_all_values(orc):
    allh = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = allh.view(np.float16).astype(np.float64)
    got = np.array([orc.f16_to_f64(int(h)) for h in allh])
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin], ref[fin])
    assert np.array_equal(np.isnan(got), np.isnan(ref))


def _ru_reference(x32: np.ndarray) -> np.ndarray:
    """RU(x) from numpy's RN: if RN(x) < x step one fp16 ulp toward +inf."""
    rn = x32.astype(np.float16)
    below = rn.astype(np.float64) < x32.astype(np.float64)
    with np.errstate(over="ignore"):
        up = np.nextafter(rn, np.float16(np.inf))
    return np.where(below, up, rn).view(np.uint16)


def _boundary_floats():
    h = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float32)   # finite >= 0
    xs = [h, np.nextafter(h, np.float32(np.inf)), np.nextafter(h, np.float32(0))]
    mid = ((h[:-1].astype(np.float64) + h[1:].astype(np.float64)) / 2).astype(np.float32)
    xs += [mid, np.nextafter(mid, np.float32(np.inf)), np.nextafter(mid, np.float32(0))]
    rng = np.random.default_rng(1)
    xs.append(rng.uniform(0, 70000, 20000).astype(np.float32))
    xs.append((2.0 ** rng.uniform(-30, 16, 20000)).astype(np.float32))
    x = np.concatenate(xs)
    return np.concatenate([x, -x])


def test_f32_to_f16_rn_matches_numpy(orc):
    x = _boundary_floats()
    x = x[np.abs(x) < 65520]
    got = np.array([orc.f32_to_f16_rn(float(v)) for v in x], np.uint16)
    assert np.array_equal(got, x.astype(np.float16).view(np.uint16))


def test_f32_to_f16_ru_matches_numpy_derived(orc):
    """Q17 rounds the scale UP; RU checked on every fp16 boundary neighbourhood."""
    x = _boundary_floats()
    x = x[np.abs(x) <= 65504]
    got = np.array([orc.f32_to_f16_ru(float(v)) for v in x], np.uint16)
    ref = _ru_reference(x)
    ok = got == ref
    # -0.0 vs +0.0 for tiny negatives: both encode zero; compare values
    zero = (got.view(np.float16) == 0) & (ref.view(np.float16) == 0)
    assert np.all(ok | zero), x[~(ok | zero)][:10]
    assert orc.f32_to_f16_ru(1e-30) == 0x0001                   # tiny positive -> 2^-24
    assert orc.f32_to_f16_ru(65504.5) == 0x7C00                 # above max -> +inf


# --------------------------------------------------------------------------------------
# Eq.10-11 thresholds
# --------------------------------------------------------------------------------------
def test_thresholds_paper_values(orc):
    p = GOLD["thresholds"]
    assert abs(orc.f1(p["s"], p["alpha"]) - p["f1"]) < p["tol"]
    assert abs(orc.f2(p["s"], p["alpha"]) - p["f2"]) < p["tol"]
    # closed forms (e-1)/(e^2-1) = 1/(e+1) and (e^-1-1)/(e^-2-1) = e/(e+1)
    assert abs(orc.f1(0.5, 2.0) - 1 / (math.e + 1)) < 1e-15
    assert abs(orc.f2(0.5, 2.0) - math.e / (math.e + 1)) < 1e-15


@pytest.mark.parametrize("alpha", [0.5, 1.0, 2.0, 4.0])
def test_threshold_properties(orc, alpha):
    """f1(0)=f2(0)=0, f1(1)=f2(1)=1, f1 <= f2 on [0,1]; f2(1-s) = 1-f1(s)."""
    assert orc.f1(0.0, alpha) == 0.0 and orc.f2(0.0, alpha) == 0.0
    assert orc.f1(1.0, alpha) == 1.0 and orc.f2(1.0, alpha) == 1.0
    grid = np.linspace(0, 1, 101)
    f1 = np.array([orc.f1(s, alpha) for s in grid])
    f2 = np.array([orc.f2(s, alpha) for s in grid])
    assert np.all(f1 <= f2 + 1e-15)
    assert np.all(np.diff(f1) > 0) and np.all(np.diff(f2) > 0)
    f2r = np.array([orc.f2(1 - s, alpha) for s in grid])
    assert np.max(np.abs(f2r - (1 - f1))) < 1e-12


def test_thresholds_n_widths_and_errors(orc):
    s = [0.5, -0.3, 1.7]                                       # clamp to [0,1] (Q10)
    t3 = orc.thresholds(s, 2.0, 3)
    assert np.allclose(t3[0], [1 / (math.e + 1), math.e / (math.e + 1)], atol=1e-15)
    assert np.array_equal(t3[1], [0.0, 0.0]) and np.array_equal(t3[2], [1.0, 1.0])
    t4 = orc.thresholds(s, 2.0, 4)
    assert abs(t4[0, 1] - 0.5) < 1e-15                          # (f1+f2)/2 = 1/2 at s = 1/2
    t2 = orc.thresholds([0.5], 2.0, 2)
    assert abs(t2[0, 0] - 0.5) < 1e-15
    with pytest.raises(ValueError):
        orc.thresholds(s, 0.0, 3)                               # alpha <= 0


# --------------------------------------------------------------------------------------
# Eq.8 window similarity
# --------------------------------------------------------------------------------------
def test_similarity_spec_examples(orc):
    """SPEC S:276-278 via a D=16 zero-padded embedding."""
    for case in GOLD["similarity_examples"]["cases"]:
        txt = np.zeros((len(case["text"]), 16), np.float16)
        txt[:, :2] = case["text"]
        win = np.zeros((len(case["window"]), 16), np.float16)
        win[:, :2] = case["window"]
        got = orc.window_score(win, txt, S=len(case["window"]), w=0)
        assert abs(got - case["sim"]) < GOLD["similarity_examples"]["tol"]


def _cos_mean_numpy(win, txt):
    w = win.astype(np.float64)
    t = txt.astype(np.float64)
    wn = np.linalg.norm(w, axis=1, keepdims=True)
    tn = np.linalg.norm(t, axis=1, keepdims=True)
    cos = (t / tn) @ (w / wn).T
    return cos.mean()


def test_similarity_vs_numpy_and_invariants(orc):
    rng = np.random.default_rng(7)
    D, S, N = 64, 16, 5
    vis = rng.standard_normal((3 * S, D)).astype(np.float16)
    txt = rng.standard_normal((N, D)).astype(np.float16)
    for w in range(3):
        got = orc.window_score(vis, txt, S, w)
        assert abs(got - _cos_mean_numpy(vis[w * S:(w + 1) * S], txt)) < 1e-12
    # scaling a row by a power of two (exact in fp16) and permuting tokens: unchanged
    base = orc.window_score(vis, txt, S, 1)
    vis2 = vis.copy()
    vis2[S + 3] *= np.float16(4.0)
    vis2[S:2 * S] = vis2[S:2 * S][::-1]
    txt2 = txt[::-1].copy()
    assert abs(orc.window_score(vis2, txt2, S, 1) - base) < 1e-13


def test_similarity_zero_rows_contribute_zero(orc):
    """Q5: a zero-norm row contributes 0, denominator stays S*N."""
    D, S = 16, 16
    win = np.zeros((S, D), np.float16)
    win[:, 0] = 1.0
    win[5] = 0.0                                               # one zero row
    txt = np.zeros((2, D), np.float16)
    txt[:, 0] = 1.0
    assert abs(orc.window_score(win, txt, S, 0) - (S - 1) / S) < 1e-15


def test_window_scores_batch_shape(orc):
    rng = np.random.default_rng(3)
    vis = rng.standard_normal((2, 40, 32)).astype(np.float16)   # M=40, S=16 -> W=2, tail 8
    txt = rng.standard_normal((2, 3, 32)).astype(np.float16)
    sc = orc.window_scores(vis, txt, 16)
    assert sc.shape == (2, 2)
    assert abs(sc[1, 1] - _cos_mean_numpy(vis[1, 16:32], txt[1])) < 1e-12


# --------------------------------------------------------------------------------------
# Assignment (Alg.2 partition P:420-444)
# --------------------------------------------------------------------------------------
def _g(orc, W, widths=(2, 4, 16), B=1, S=16):
    return orc.geom(B, 1, 1, 64, W * S, S, widths)


def test_band_examples(orc):
    p = GOLD["band_examples"]
    g = _g(orc, 3)
    bits, rank, perm, seg = orc.assign_bits(np.array([p["sims"]]), np.array([p["thr"]]), g, pin=0)
    assert list(bits[0, 0]) == p["bits"]
    # boundaries fall in the middle band (strict inequalities of Alg.1, Q8)
    bits, *_ = orc.assign_bits(np.array([[0.2, 0.8, 0.19999]]), np.array([[0.2, 0.8]]), g, pin=0)
    assert list(bits[0, 0]) == [4, 4, 2]


def test_band_limits_s0_s1(orc):
    """s=1 -> thresholds 1 -> all INT2 but the pin; s=0 -> every sim>0 FP16."""
    sims = np.array([[0.3, 0.99, 0.5, 0.01]])
    g = _g(orc, 4)
    thr1 = orc.thresholds([1.0], 2.0, 3)
    bits, *_ = orc.assign_bits(sims, thr1, g, pin=1)
    assert list(bits[0, 0]) == [16, 2, 2, 2]
    thr0 = orc.thresholds([0.0], 2.0, 3)
    bits, *_ = orc.assign_bits(sims, thr0, g, pin=0)
    assert list(bits[0, 0]) == [16, 16, 16, 16]


def test_four_widths_and_pin_without_16(orc):
    thr = orc.thresholds([0.5], 2.0, 4)                         # (0.2689, 0.5, 0.7311)
    sims = np.array([[0.1, 0.1, 0.3, 0.5, 0.6, 0.75]])
    g = _g(orc, 6, widths=(2, 4, 8, 16))
    bits, *_ = orc.assign_bits(sims, thr, g, pin=0)
    assert list(bits[0, 0]) == [2, 2, 4, 8, 8, 16]
    g3 = _g(orc, 6, widths=(2, 4, 8))                           # C1: no 16 width
    thr3 = orc.thresholds([0.5], 2.0, 3)
    bits, rank, perm, seg = orc.assign_bits(sims, thr3, g3, pin=1)
    assert list(bits[0, 0]) == [16, 2, 4, 4, 4, 8]
    assert list(seg[0, 0]) == [0, 1, 4, 5, 6]                    # pinned window in class 16
    assert list(perm[0, 0]) == [1, 2, 3, 4, 5, 0]


def test_stable_partition_spec_example(orc):
    p = GOLD["stable_partition"]
    sims = np.array([[0.9, 0.1, 0.5, 0.9, 0.1, 0.5]])
    g = _g(orc, 6)
    bits, rank, perm, seg = orc.assign_bits(sims, np.array([[0.2, 0.8]]), g, pin=0)
    assert list(bits[0, 0]) == p["widths"]
    assert list(perm[0, 0]) == p["perm"]
    assert list(seg[0, 0]) == p["seg_off"]
    assert list(rank[0]) == [0, 4, 2, 1, 5, 3]                   # ties -> lower index first (Q7)


def test_vote_examples(orc):
    """P:395 / SPEC S:305-308: mode over the batch, ties toward the higher width."""
    thr = np.array([[0.2, 0.8]])
    val = {2: 0.1, 4: 0.5, 16: 0.9}
    for case in GOLD["vote_examples"]["cases"]:
        B = len(case["votes"])
        sims = np.array([[0.0, val[v]] for v in case["votes"]])   # window 0 pinned
        g = _g(orc, 2, B=B)
        bits, *_ = orc.assign_bits(sims, thr, g, pin=1, vote=1)
        assert np.all(bits[0, :, 1] == case["result"]) and np.all(bits[0, :, 0] == 16)
    # idempotent for one request, invariant to the batch order
    rng = np.random.default_rng(5)
    sims = rng.uniform(0, 1, (5, 20))
    g = _g(orc, 20, B=5)
    b1, *_ = orc.assign_bits(sims, thr, g, pin=1, vote=1)
    b2, *_ = orc.assign_bits(sims[::-1].copy(), thr, g, pin=1, vote=1)
    assert np.array_equal(b1, b2)
    g1 = _g(orc, 20, B=1)
    a, *_ = orc.assign_bits(sims[:1], thr, g1, pin=1, vote=0)
    b, *_ = orc.assign_bits(sims[:1], thr, g1, pin=1, vote=1)
    assert np.array_equal(a, b)


def test_budget_hand_example(orc):
    """Q13 by hand: W=5, widths {2,4,8,16}, thresholds (0.2689, 0.5, 0.7311), pin.
    sims [*, 0.8, 0.6, 0.3, 0.1] -> bands [16, 16, 8, 4, 2] (sum 46).
    budget 6 bits avg -> limit 30.  Demote lowest-ranked first, one step at a time:
    w3 4->2 (44), w2 8->4 (40), w2 4->2 (38), w1 16->8 (30) -> stop."""
    thr = orc.thresholds([0.5], 2.0, 4)
    sims = np.array([[0.0, 0.8, 0.6, 0.3, 0.1]])
    g = _g(orc, 5, widths=(2, 4, 8, 16))
    bits, *_ = orc.assign_bits(sims, thr, g, budget=0.0, pin=1)
    assert list(bits[0, 0]) == [16, 16, 8, 4, 2]
    bits, *_ = orc.assign_bits(sims, thr, g, budget=6.0, pin=1)
    assert list(bits[0, 0]) == [16, 8, 2, 2, 2]
    with pytest.raises(ValueError):                           # 16 + 4*2 = 24 > 4.7*5 = 23.5
        orc.assign_bits(sims, thr, g, budget=4.7, pin=1)


def test_budget_invariants_random(orc):
    """North star: the assignment meets the budget and is monotone in the score."""
    rng = np.random.default_rng(11)
    L, B, W = 3, 4, 60
    sims = rng.uniform(0, 1, (B, W))
    thr = orc.thresholds([0.5, 0.3, 0.1], 2.0, 4)
    g = orc.geom(B, 1, 1, 64, W * 16, 16, (2, 4, 8, 16))
    for budget in (0.0, 3.0, 4.0, 6.5):
        bits, rank, perm, seg = orc.assign_bits(sims, thr, g, budget=budget, pin=1)
        for l, b in itertools.product(range(L), range(B)):
            bl = bits[l, b].astype(int)
            assert bl[0] == 16
            if budget > 0:
                assert bl.sum() <= budget * W + 1e-9
            order = np.argsort(-sims[b], kind="stable")
            o = [w for w in order if w != 0]
            assert all(bl[o[i]] >= bl[o[i + 1]] for i in range(len(o) - 1))
            # perm is a stable partition and a bijection
            p = perm[l, b]
            assert sorted(p) == list(range(W))
            cls = np.array([{2: 0, 4: 1, 8: 2, 16: 3}[x] for x in bl[p]])
            assert np.all(np.diff(cls) >= 0)
            for k in range(4):
                seg_w = p[seg[l, b, k]:seg[l, b, k + 1]]
                assert np.all(np.diff(seg_w) > 0) and np.all(cls[seg[l, b, k]:seg[l, b, k + 1]] == k)


# --------------------------------------------------------------------------------------
# Byte accounting
# --------------------------------------------------------------------------------------
def test_memory_reduction_paper(orc):
    p = GOLD["memory_reduction"]
    t = p["tokens"]
    fp16 = orc.kv_code_bytes([0, 0, 0, t["int2"] + t["int4"] + t["fp16"]], p["d"], p["H"])
    wq = orc.kv_code_bytes([t["int2"], t["int4"], 0, t["fp16"]], p["d"], p["H"])
    assert fp16 - wq == p["bytes_saved_per_layer"]
    total_mb = round((fp16 - wq) / 2 ** 20, 2) * p["layers"]
    assert abs(total_mb - p["total_MB"]) < p["total_tol_MB"]


def test_record_bytes_closed_form(orc):
    # d=128, S=32: 2-bit 2*32*128*2/8 + 4*128 + 4*32 = 2688; 16-bit 4*32*128 = 16384
    assert orc.record_bytes(2, 128, 32) == 2688
    assert orc.record_bytes(4, 128, 32) == 4736
    assert orc.record_bytes(8, 128, 32) == 8832
    assert orc.record_bytes(16, 128, 32) == 16384
    g = orc.geom(1, 4, 28, 128, 32 * 10, 32, (2, 4, 8, 16))
    assert orc.packed_bytes(g, [4, 3, 2, 1]) == 4 * 2688 + 3 * 4736 + 2 * 8832 + 16384
    assert orc.packed_bytes(g, [1, 0, 0, 0], code_only=True) == 2048


# --------------------------------------------------------------------------------------
# Packing layout (D-1) and the SPEC golden bytes
# --------------------------------------------------------------------------------------
def test_packing_golden_bytes(orc):
    """SPEC S:164-169 bit order: consecutive codes of a byte fill it from bit 0.
    In D-1 the four pairs of lane 0 / k-tile 0 hold elements (0,0), (8,0), (0,8),
    (8,8) as their first elements, packed into byte 0 in that order."""
    pk = GOLD["packing"]
    elems = [(0, 0), (8, 0), (0, 8), (8, 8)]
    for b, key in ((2, "int2"), (4, "int4"), (2, "int2_single")):
        codes = pk[key]["codes"]
        byte = 0
        for (t, c), code in zip(elems, codes):
            off, bit = orc.code_pos(0, 64, b, t, c)
            assert off == 0 and bit == b * elems.index((t, c))
            byte |= code << bit
        assert byte == pk[key]["byte"]


@pytest.mark.parametrize("is_v,d,b", [(0, 64, 2), (1, 64, 4), (0, 128, 8), (1, 128, 2), (0, 128, 16), (1, 64, 16)])
def test_code_layout_is_a_bijection(orc, is_v, d, b):
    """Every bit of a tile is used exactly once (b < 16) / every fp16 slot once."""
    used = np.zeros(2 * d * b * 8, np.int32)
    for t in range(16):
        for c in range(d):
            off, bit = orc.code_pos(is_v, d, b, t, c)
            start = off * 8 + bit
            used[start:start + b] += 1
    assert np.all(used == 1)


def test_code_layout_fragment_rule(orc):
    """Spot-check the D-1 rule: K element (t=9, c=27): row 9 -> g=1, r&1=1;
    c=27 -> m=1, c%16=11 -> (r>>1)=1, q=1, e=1; so r=3, lane 4*1+1=5."""
    off, bit = orc.code_pos(0, 64, 2, 9, 27)
    # pair P = 4*1 + 3 = 7, word 0 (8 pairs/word), slot 7, e = 1 -> bit 16 + 14
    assert off == (4 * 1 + 1) * (64 * 2 // 16) and bit == 30
    off, bit = orc.code_pos(1, 64, 4, 3, 40)                    # V: channel 40, token 3
    # m = 2, row 8 -> g=0, rhi=1; col 3 -> q=1, h=0, e=1; r=1; P=9; 4 pairs/word: word 2 slot 1
    assert off == 1 * (64 * 4 // 16) + 2 * 4 and bit == 16 + 4


# --------------------------------------------------------------------------------------
# Quantizer Eq.14-16 under Q17 (hand-derived goldens in DESIGN.md §3)
# --------------------------------------------------------------------------------------
QGOLD = [
    # values, bits, scale fp16 bits, codes
    ([0, 1, 2, 3], 2, 0x3C00, [0, 1, 2, 3]),
    ([-1, 1], 4, 0x3045, [0, 15]),                    # RU(2/15) = 1093 * 2^-13
    ([5.5] * 4, 2, 0x0001, [0, 0, 0, 0]),             # degenerate: 2^-24 floor (Q21)
    ([-1, -0.5, 0, 0.5, 1], 2, None, [0, 1, 1, 2, 3]),   # s = RU(2/3) = 0.6669922
    ([0.1, 0.2, 0.3, 0.7], 4, None, [0, 2, 5, 15]),   # s = 1312 * 2^-15
    ([3.0, 3.001953125, 3.001953125], 8, 129, [0, 254, 254]),  # subnormal s = 129 * 2^-24
]


@pytest.mark.parametrize("vals,bits,sbits,codes", QGOLD)
def test_quantizer_goldens(orc, vals, bits, sbits, codes):
    s, mn, c = orc.quantize_group(np.array(vals, np.float16), bits)
    if sbits is not None:
        assert s == sbits
    assert list(c) == codes
    assert np.float16(vals[0]).view(np.uint16) == mn or min(vals) == np.array([mn], np.uint16).view(np.float16)[0]


def test_quantizer_scale_values(orc):
    s, _, _ = orc.quantize_group(np.array([-1, -0.5, 0, 0.5, 1], np.float16), 2)
    assert np.array([s], np.uint16).view(np.float16)[0] == np.float16(1366 * 2 ** -11)
    s, _, _ = orc.quantize_group(np.array([0.1, 0.2, 0.3, 0.7], np.float16), 4)
    assert np.array([s], np.uint16).view(np.float16)[0] == np.float16(1312 * 2 ** -15)


SZ = [
    # Q17 mn = IEEE 754-2019 minimum (section 9.6: -0 < +0), independent of element order
    ([0x0000, 0x8000, 0x3C00, 0x4000], 0x8000),       # [+0, -0, 1, 2] -> mn = -0
    ([0x8000, 0x0000, 0x3C00, 0x4000], 0x8000),       # [-0, +0, 1, 2] -> mn = -0
    ([0x3C00, 0x0000, 0x4000, 0x8000], 0x8000),       # -0 last
    ([0x0000, 0x0000, 0x3C00], 0x0000),               # only +0 -> +0
    ([0x8000, 0x8000, 0x3C00], 0x8000),               # only -0 -> -0
    ([0x0000, 0x8000, 0xBC00], 0xBC00),               # a negative value below both zeros
    ([0x8000, 0x0000], 0x8000),                       # all zeros: mn = -0, codes 0
]


@pytest.mark.parametrize("bits16,mn_bits", SZ)
def test_quantizer_signed_zero_minimum(orc, bits16, mn_bits):
    """Reading Q17 fixes mn as the IEEE 754-2019 minimum, so a group whose minimum is a
    zero stores the sign bit of -0 iff a -0 is present (both element orders give the
    same bytes); zeros of either sign get code 0 and dequantize to a zero."""
    x = np.array(bits16, np.uint16).view(np.float16)
    for bits in (2, 4, 8):
        s, mn, c = orc.quantize_group(x, bits)
        assert mn == mn_bits, (bits16, hex(mn))
        for i, v in enumerate(bits16):
            if v in (0x0000, 0x8000):
                assert c[i] == (0 if mn_bits in (0x0000, 0x8000) else c[i])
        sv = float(np.array([s], np.uint16).view(np.float16)[0])
        mv = float(np.array([mn], np.uint16).view(np.float16)[0])
        assert np.all(np.abs(x.astype(np.float64) - (mv + sv * c)) <= sv * (0.5 + 2 ** -14))


def test_quantizer_degenerate_groups(orc):
    """Edge groups: a constant group takes the 2^-24 scale floor (Q21) and every code is 0;
    values at the fp16 extremes +-65504 give s = RU(131008 / q_max) exactly (closed form)
    and the codes 0 / q_max at the ends; a range of one subnormal step is a subnormal scale."""
    for bits in (2, 4, 8):
        qmax = 2 ** bits - 1
        s, mn, c = orc.quantize_group(np.full(32, -3.25, np.float16), bits)
        assert s == 0x0001 and np.all(c == 0)
        x = np.array([65504, -65504, 0, 1, -1], np.float16)
        s, mn, c = orc.quantize_group(x, bits)
        sv = float(np.array([s], np.uint16).view(np.float16)[0])
        exact = 131008.0 / qmax
        # RU to fp16: the smallest fp16 >= fl32(131008 / q_max)
        assert sv >= np.float32(exact) and float(np.nextafter(np.float16(sv), np.float16(0))) < np.float32(exact)
        assert mn == 0xFBFF and c[0] == qmax and c[1] == 0
        x = np.array([2 ** -24, 0, 2 ** -24, 0], np.float16)     # range = one subnormal step
        s, mn, c = orc.quantize_group(x, bits)
        assert s == 0x0001 and list(c) == [1, 0, 1, 0]


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_quantizer_error_bound_and_monotone(orc, bits):
    """North star: |x - x^| <= s/2 (Q17 guarantees s*(1/2 + 2^-14)); codes monotone;
    code(min) = 0; the round trip of on-lattice values is exact."""
    rng = np.random.default_rng(bits)
    for i in range(300):
        n = int(rng.choice([16, 32, 64, 128]))
        scale = 10.0 ** rng.uniform(-3, 1.5)
        x = (rng.standard_normal(n) * scale + rng.uniform(-20, 20)).astype(np.float16)
        s, mn, c = orc.quantize_group(x, bits)
        sv = float(np.array([s], np.uint16).view(np.float16)[0])
        mv = float(np.array([mn], np.uint16).view(np.float16)[0])
        xh = mv + sv * c.astype(np.float64)
        err = np.abs(x.astype(np.float64) - xh)
        assert np.all(err <= sv * (0.5 + 2 ** -14)), (i, err.max() / sv)
        assert mv == float(x.min())
        assert c[np.argmin(x)] == 0 and c.max() <= 2 ** bits - 1
        o = np.argsort(x.astype(np.float64), kind="stable")
        assert np.all(np.diff(c[o].astype(int)) >= 0)


# --------------------------------------------------------------------------------------
# Reorder+quantize+pack and decode (Alg.2, Eq.2-3, Eq.12-13)
# --------------------------------------------------------------------------------------
def _small_case(orc, widths=(2, 4, 8, 16), B=2, H=2, Hq=4, d=64, S=16, W=6, tail=5, R=9, seed=0,
                all16=False):
    rng = np.random.default_rng(seed)
    M = W * S + tail
    K = (rng.standard_normal((B, H, M, d)) * rng.uniform(0.3, 2, (1, H, 1, d)) +
         rng.standard_normal((1, H, 1, d)) * 3).astype(np.float16)
    V = (rng.standard_normal((B, H, M, d)) * np.exp(0.5 * rng.standard_normal((B, H, M, 1)))).astype(np.float16)
    q = rng.standard_normal((B, Hq, d)).astype(np.float16)
    kr = rng.standard_normal((B, H, R, d)).astype(np.float16)
    vr = rng.standard_normal((B, H, R, d)).astype(np.float16)
    rest_len = np.array([R - b for b in range(B)], np.int32)
    g = orc.geom(B, H, Hq, d, M, S, widths)
    sims = rng.uniform(0, 1, (B, W))
    if all16:
        g16 = orc.geom(B, H, Hq, d, M, S, (16,))
        bits, rank, perm, seg = orc.assign_bits(sims, np.zeros((1, 0)), g16, pin=1)
    else:
        thr = orc.thresholds([0.5], 2.0, len(widths))
        bits, rank, perm, seg = orc.assign_bits(sims, thr, g, pin=1)
    return dict(g=g, K=K, V=V, q=q, kr=kr, vr=vr, rest_len=rest_len, perm=perm[0], seg=seg[0],
                bits=bits[0], W=W, S=S, d=d)


def test_decode_spec_example(orc):
    """SPEC S:467 (corrected, Q31): q=[1,0], K=V=I2, d_k=2 -> [0.669762, 0.330238]."""
    p = GOLD["decode_example"]
    d = 64
    g = orc.geom(1, 1, 1, d, 16, 16, (16,))
    q = np.zeros((1, 1, d), np.float16)
    q[0, 0, :2] = p["q"]
    kr = np.zeros((1, 1, 2, d), np.float16)
    vr = np.zeros((1, 1, 2, d), np.float16)
    kr[0, 0, :, :2] = p["K"]
    vr[0, 0, :, :2] = p["V"]
    K = np.zeros((1, 1, 16, d), np.float16)
    out = orc.bruteforce_attention(q, K, K, 0, g, np.zeros((1, 1), np.int32), np.zeros(1, np.int32),
                                   kr, vr, np.array([2], np.int32), 1 / math.sqrt(2))
    assert np.allclose(out[0, 0, :2], p["out"], atol=p["tol"])
    # the same through decode_attention with an empty packed image
    seg = np.zeros((1, 5), np.int32)
    out2 = orc.decode_attention(q, np.zeros(16, np.uint8), np.zeros(2, np.int64), seg,
                                np.zeros((1, 1), np.int32), g, kr, vr, np.array([2], np.int32),
                                1 / math.sqrt(2))
    assert np.array_equal(out, out2)


def test_all16_decode_equals_bruteforce(orc):
    """North star: with every window at 16 bits the oracle decode equals fp64
    brute-force attention (exactly: same fp64 values in the same token order)."""
    c = _small_case(orc, all16=True)
    packed, offs = orc.reorder_quantize_pack(c["K"], c["V"], 0, c["g"], c["perm"], c["seg"])
    sm = 1 / math.sqrt(c["d"])
    out = orc.decode_attention(c["q"], packed, offs, c["seg"], c["perm"], c["g"], c["kr"], c["vr"],
                               c["rest_len"], sm)
    B = c["g"].B
    win = np.tile(np.arange(c["W"], dtype=np.int32), (B, 1))
    ref = orc.bruteforce_attention(c["q"], c["K"], c["V"], 0, c["g"], win, np.full(B, c["W"], np.int32),
                                   c["kr"], c["vr"], c["rest_len"], sm)
    assert np.array_equal(out, ref)


def test_reorder_invariance_bruteforce(orc):
    """Eq.12-13: any window order gives the same attention output."""
    c = _small_case(orc)
    B = c["g"].B
    sm = 1 / math.sqrt(c["d"])
    win = np.tile(np.arange(c["W"], dtype=np.int32), (B, 1))
    ref = orc.bruteforce_attention(c["q"], c["K"], c["V"], 0, c["g"], win, np.full(B, c["W"], np.int32),
                                   c["kr"], c["vr"], c["rest_len"], sm)
    rng = np.random.default_rng(2)
    for _ in range(3):
        wp = np.stack([rng.permutation(c["W"]).astype(np.int32) for _ in range(B)])
        out = orc.bruteforce_attention(c["q"], c["K"], c["V"], 0, c["g"], wp, np.full(B, c["W"], np.int32),
                                       c["kr"], c["vr"], c["rest_len"], sm)
        assert np.max(np.abs(out - ref)) < 1e-12


def test_packed_image_dequant_error_bound(orc):
    """The byte image decodes (through the layout) to values within s/2 of the
    original fp16 K/V for every quantized window; 16-bit windows round-trip exactly."""
    c = _small_case(orc, widths=(2, 4, 8, 16), seed=4)
    packed, offs = orc.reorder_quantize_pack(c["K"], c["V"], 0, c["g"], c["perm"], c["seg"])
    g, S, d = c["g"], c["S"], c["d"]
    for b in range(g.B):
        for h in range(g.H):
            off = int(offs[b * g.H + h])
            for slot in range(c["seg"][b, 4]):
                k = int(np.searchsorted(c["seg"][b, 1:], slot, side="right"))
                bits = (2, 4, 8, 16)[k]
                w = c["perm"][b, slot]
                rb = orc.record_bytes(bits, d, S)
                kh, vh = orc.dequant_record(packed[off:off + rb], bits, d, S)
                off += rb
                Kw = c["K"][b, h, w * S:(w + 1) * S].astype(np.float64)
                Vw = c["V"][b, h, w * S:(w + 1) * S].astype(np.float64)
                if bits == 16:
                    assert np.array_equal(kh, Kw) and np.array_equal(vh, Vw)
                    continue
                ks = (Kw.max(0) - Kw.min(0)) / (2 ** bits - 1)     # per-channel s (before RU)
                vs = (Vw.max(1) - Vw.min(1)) / (2 ** bits - 1)     # per-token s
                tolk = np.maximum(ks * (1 + 2 ** -10), 2 ** -24) * (0.5 + 2 ** -14) + 1e-12
                tolv = np.maximum(vs * (1 + 2 ** -10), 2 ** -24) * (0.5 + 2 ** -14) + 1e-12
                assert np.all(np.abs(kh - Kw) <= tolk[None, :])
                assert np.all(np.abs(vh - Vw) <= tolv[:, None])
            assert off == offs[b * g.H + h + 1]


def test_decode_mixed_properties(orc):
    """Convex hull and reorder invariance of the dequantized cache."""
    c = _small_case(orc, seed=9)
    packed, offs = orc.reorder_quantize_pack(c["K"], c["V"], 0, c["g"], c["perm"], c["seg"])
    sm = 1 / math.sqrt(c["d"])
    out = orc.decode_attention(c["q"], packed, offs, c["seg"], c["perm"], c["g"], c["kr"], c["vr"],
                               c["rest_len"], sm)
    assert np.all(np.isfinite(out))
    # convex hull: every output coordinate within [min, max] of dequantized V column + rest
    g = c["g"]
    for b in range(g.B):
        for h in range(g.H):
            off = int(offs[b * g.H + h])
            vs = []
            for slot in range(c["seg"][b, 4]):
                k = int(np.searchsorted(c["seg"][b, 1:], slot, side="right"))
                bits = (2, 4, 8, 16)[k]
                rb = orc.record_bytes(bits, c["d"], c["S"])
                vs.append(orc.dequant_record(packed[off:off + rb], bits, c["d"], c["S"])[1])
                off += rb
            vs.append(c["vr"][b, h, :c["rest_len"][b]].astype(np.float64))
            allv = np.concatenate(vs)
            grp = g.Hq // g.H
            o = out[b, h * grp:(h + 1) * grp]
            assert np.all(o <= allv.max(0) + 1e-12) and np.all(o >= allv.min(0) - 1e-12)


def test_merge_identity_and_split(orc):
    """LSE merge: G=1 is the identity; merging shard partials equals the unsplit
    result (the C5 sequence split, §8(e))."""
    c = _small_case(orc, seed=12)
    g = c["g"]
    sm = 1 / math.sqrt(c["d"])
    packed, offs = orc.reorder_quantize_pack(c["K"], c["V"], 0, g, c["perm"], c["seg"])
    full, part = orc.decode_attention(c["q"], packed, offs, c["seg"], c["perm"], g, c["kr"], c["vr"],
                                      c["rest_len"], sm, want_partial=True)
    assert np.max(np.abs(orc.merge(part[None]) - full)) < 1e-13
    # two shards: each keeps ~half of every segment; shard 1 has no rest tokens
    parts = []
    for r in range(2):
        perm_r = np.zeros_like(c["perm"])
        seg_r = np.zeros_like(c["seg"])
        for b in range(g.B):
            slots = []
            for k in range(4):
                lo, hi = c["seg"][b, k], c["seg"][b, k + 1]
                mid = lo + (hi - lo) // 2
                seg_r[b, k] = len(slots)
                slots += list(c["perm"][b, lo:mid] if r == 0 else c["perm"][b, mid:hi])
            seg_r[b, 4] = len(slots)
            perm_r[b, :len(slots)] = slots
        pk, of = orc.reorder_quantize_pack(c["K"], c["V"], 0, g, perm_r, seg_r)
        rl = c["rest_len"] if r == 0 else np.zeros_like(c["rest_len"])
        _, p = orc.decode_attention(c["q"], pk, of, seg_r, perm_r, g, c["kr"], c["vr"], rl, sm,
                                    want_partial=True)
        parts.append(p)
    assert np.max(np.abs(orc.merge(np.stack(parts)) - full)) < 1e-12


def test_code_layout_interleaved_groups(orc):
    """D-1 interleaving: d=128, b=4 -> 32-byte lane chunks stored as 16-byte groups
    across lanes.  K element (t=0, c=32): m=2, r=0, lane 0 -> pair P=8, word 2
    (4 pairs/word), so group 0, byte 0*512 + 0*16 + 2*4 = 8.  K element (t=1, c=64):
    g=1 -> lane 4, m=4 -> P=16 -> word 4 -> group 1: byte 512 + 4*16 + 0 = 576."""
    assert orc.code_pos(0, 128, 4, 0, 32) == (8, 0)
    assert orc.code_pos(0, 128, 4, 1, 64) == (576, 0)
    # 8-byte chunks (d=64, b=2) stay lane-linear: K (t=1, c=18): g=1, m=1, q=1, r=0
    # -> lane 5, P=4 -> word 0, slot 4 -> byte 5*8 = 40, bit 8
    assert orc.code_pos(0, 64, 2, 1, 18) == (40, 8)


def test_param_layout_hand_derived(orc):
    """D-1 params: K group (q, m) = {mn(c0), mn(c0+1), s(c0), s(c0+1), mn(c0+8), mn(c0+9),
    s(c0+8), s(c0+9)} with c0 = 16m + 2q; V group (i, q) = {s(t0), s(t0+1), s(t0+8), s(t0+9),
    mn(t0), ...}.  K c=9 (d=64): m=0, q=0, second half (c0+8), e=1 -> mn at half 5, s at half 7.
    K c=34 (d=128): m=2, q=1, first half, e=0 -> group 4*2+1=9 -> s at byte 144+4.
    V t=9: group 0, second half, e=1 -> s at half 3, mn at half 7."""
    assert orc.param_pos(0, 64, 9, 1) == 10 and orc.param_pos(0, 64, 9, 0) == 14
    assert orc.param_pos(0, 128, 34, 0) == 148 and orc.param_pos(0, 128, 34, 1) == 144
    assert orc.param_pos(1, 64, 9, 0) == 6 and orc.param_pos(1, 64, 9, 1) == 14
    # every param slot used exactly once (K: 2 x d halves in 4d bytes)
    used = sorted(orc.param_pos(0, 128, c, m) for c in range(128) for m in (0, 1))
    assert used == list(range(0, 4 * 128, 2))


# --------------------------------------------------------------------------------------
# T9 unfused baseline: dequantize the image to FP16
# --------------------------------------------------------------------------------------
def test_f64_to_f16_rn_matches_numpy(orc):
    """RN to fp16 from fp64 (incl. exact ties of dyadic values) against numpy's astype."""
    x = _boundary_floats().astype(np.float64)
    h = np.arange(0, 0x7BFF, dtype=np.uint16).view(np.float16).astype(np.float64)
    ties = (h[:-1] + h[1:]) / 2                         # exact midpoints: ties to even
    x = np.concatenate([x, ties, -ties, ties + 2.0 ** -40, ties - 2.0 ** -40])
    x = x[np.abs(x) < 65520]
    got = np.array([orc.f64_to_f16_rn(float(v)) for v in x], np.uint16)
    assert np.array_equal(got, x.astype(np.float16).view(np.uint16))


def test_dequantize_image_values(orc):
    """Every FP16 record holds RN_fp16 of the exact dequantized values (numpy rounding of
    the fp64 record dequantization); FP16 windows are copied; slot order is kept."""
    c = _small_case(orc, seed=13)
    g = c["g"]
    packed, offs = orc.reorder_quantize_pack(c["K"], c["V"], 0, g, c["perm"], c["seg"])
    img16, offs16, seg16 = orc.dequantize_image(packed, offs, c["seg"], g)
    assert np.array_equal(seg16[:, :4], np.zeros_like(seg16[:, :4]))
    assert np.array_equal(seg16[:, 4], c["seg"][:, 4])
    rb16 = orc.record_bytes(16, c["d"], c["S"])
    for b in range(g.B):
        for h in range(g.H):
            off, off16 = int(offs[b * g.H + h]), int(offs16[b * g.H + h])
            for slot in range(c["seg"][b, 4]):
                k = int(np.searchsorted(c["seg"][b, 1:], slot, side="right"))
                bits = (2, 4, 8, 16)[k]
                rb = orc.record_bytes(bits, c["d"], c["S"])
                kx, vx = orc.dequant_record(packed[off:off + rb], bits, c["d"], c["S"])
                k16, v16 = orc.dequant_record(img16[off16 + slot * rb16:off16 + (slot + 1) * rb16], 16, c["d"], c["S"])
                assert np.array_equal(k16, kx.astype(np.float16).astype(np.float64))
                assert np.array_equal(v16, vx.astype(np.float16).astype(np.float64))
                off += rb


def test_dequantize_image_decode_close_to_fused(orc):
    """Attention over the FP16 image differs from the fused (exact-dequant) attention
    only by the fp16 rounding of the dequantized values."""
    c = _small_case(orc, seed=14)
    g = c["g"]
    packed, offs = orc.reorder_quantize_pack(c["K"], c["V"], 0, g, c["perm"], c["seg"])
    img16, offs16, seg16 = orc.dequantize_image(packed, offs, c["seg"], g)
    sm = 1 / math.sqrt(c["d"])
    a = orc.decode_attention(c["q"], packed, offs, c["seg"], c["perm"], g, c["kr"], c["vr"], c["rest_len"], sm)
    b = orc.decode_attention(c["q"], img16, offs16, seg16, c["perm"], g, c["kr"], c["vr"], c["rest_len"], sm)
    assert np.max(np.abs(a - b)) / np.max(np.abs(a)) < 5e-3
    assert not np.array_equal(a, b)


# --------------------------------------------------------------------------------------
# T11 similarity variant: Pearson correlation in Eq.8
# --------------------------------------------------------------------------------------
def test_pearson_scores_vs_numpy_and_invariants(orc):
    rng = np.random.default_rng(21)
    S, N, D = 16, 5, 24
    vis = rng.standard_normal((1, 3 * S, D)).astype(np.float16)
    txt = rng.standard_normal((1, N, D)).astype(np.float16)
    got = orc.window_scores_pearson(vis, txt, S)
    v64, t64 = vis[0].astype(np.float64), txt[0].astype(np.float64)
    for w in range(3):
        c = np.corrcoef(np.concatenate([t64, v64[w * S:(w + 1) * S]]))[:N, N:]
        assert abs(got[0, w] - c.mean()) < 1e-12
    # invariant under affine maps x -> a x + b (a > 0) of any row; equals cosine for centred rows
    vis2 = vis.copy()
    vis2[0, 3] = (vis[0, 3].astype(np.float32) * 0.5 + 0.25).astype(np.float16)
    exact = np.allclose(vis2[0, 3].astype(np.float64), vis[0, 3].astype(np.float64) * 0.5 + 0.25, rtol=0, atol=0)
    if exact:
        assert abs(orc.window_scores_pearson(vis2, txt, S)[0, 0] - got[0, 0]) < 1e-12
    vc = (v64 - v64.mean(1, keepdims=True)).astype(np.float16)[None]
    tc = (t64 - t64.mean(1, keepdims=True)).astype(np.float16)[None]
    vc64, tc64 = vc[0].astype(np.float64), tc[0].astype(np.float64)
    if np.allclose(vc64.mean(1), 0, atol=0) and np.allclose(tc64.mean(1), 0, atol=0):
        assert np.allclose(orc.window_scores_pearson(vc, tc, S), orc.window_scores(vc, tc, S), atol=1e-12)
    # perfectly correlated / anti-correlated / constant rows
    base = rng.standard_normal(D).astype(np.float16)
    v = np.tile(base, (S, 1))[None]
    t = np.stack([base, (-base.astype(np.float32)).astype(np.float16)])[None]
    assert abs(orc.window_scores_pearson(v, t[:, :1], S)[0, 0] - 1.0) < 1e-12
    assert abs(orc.window_scores_pearson(v, t[:, 1:], S)[0, 0] + 1.0) < 1e-12
    const = np.full((1, S, D), 0.5, np.float16)
    assert orc.window_scores_pearson(const, t[:, :1], S)[0, 0] == 0.0


def test_alpha_sweep_trend(orc):
    """Fig. thre_para: for fixed scores, raising alpha lowers T_low = f1(s) and
    raises T_high = f2(s) (Eq.10-11), so INT2 and FP16 windows never grow and INT4 never
    shrinks (3 widths {2,4,16}, no budget, no pin)."""
    rng = np.random.default_rng(11)
    W = 400
    g = orc.geom(1, 1, 1, 64, W * 16, 16, (2, 4, 16))
    sc = rng.uniform(0, 1, (1, W))
    prev = None
    for a in (0.25, 0.5, 1.0, 2.0, 4.0, 8.0, 16.0):
        thr = orc.thresholds([0.5], a, 3)
        bits, _, _, _ = orc.assign_bits(sc, thr, g, pin=0)
        n = [int((bits == b).sum()) for b in (2, 4, 16)]
        if prev is not None:
            assert n[0] <= prev[0] and n[2] <= prev[2] and n[1] >= prev[1]
        prev = n
    assert prev[1] > prev[0] and prev[1] > prev[2]


# --------------------------------------------------------------------------------------
# Per-layer scorer (reading Q36)
# --------------------------------------------------------------------------------------
def test_layer_scorer_reduces_to_embedding_scorer(orc):
    """H = Hq = 1: the per-layer scorer IS Eq.8 on the key rows and the query rows (the
    pinned embedding scorer); with H kv heads and identical queries inside each GQA group,
    it equals the embedding scorer on the head-concatenated rows (group mean of equal rows)."""
    rng = np.random.default_rng(21)
    B, T, d, N, S, vis_off = 2, 7 + 5 * 16, 64, 6, 16, 7
    M = T - vis_off
    k = rng.standard_normal((B, 1, T, d)).astype(np.float16)
    q = rng.standard_normal((B, 1, N, d)).astype(np.float16)
    got = orc.window_scores_layer(k, vis_off, q, M, S)
    ref = orc.window_scores(np.ascontiguousarray(k[:, 0, vis_off:]), np.ascontiguousarray(q[:, 0]), S)
    assert np.max(np.abs(got - ref)) <= 1e-13
    H, grp = 3, 4
    k = rng.standard_normal((B, H, T, d)).astype(np.float16)
    qh = rng.standard_normal((B, H, N, d)).astype(np.float16)
    q = np.repeat(qh, grp, axis=1)                                  # identical queries in a group
    got = orc.window_scores_layer(k, vis_off, q, M, S)
    vis = np.ascontiguousarray(k[:, :, vis_off:].transpose(0, 2, 1, 3).reshape(B, M, H * d))
    txt = np.ascontiguousarray(qh.transpose(0, 2, 1, 3).reshape(B, N, H * d))
    assert np.max(np.abs(got - orc.window_scores(vis, txt, S))) <= 1e-12


def test_layer_scorer_invariants(orc):
    """Permuting the kv heads (keys and their query groups together) and scaling a key
    row by c > 0 leave the scores unchanged; a query group and its mean give one score."""
    rng = np.random.default_rng(22)
    B, H, grp, T, d, N, S = 1, 4, 2, 4 * 32, 128, 5, 32
    k = rng.standard_normal((B, H, T, d)).astype(np.float16)
    q = rng.standard_normal((B, H * grp, N, d)).astype(np.float16)
    base = orc.window_scores_layer(k, 0, q, T, S)
    perm = [2, 0, 3, 1]
    qperm = np.concatenate([q[:, h * grp:(h + 1) * grp] for h in perm], axis=1)
    assert np.max(np.abs(orc.window_scores_layer(np.ascontiguousarray(k[:, perm]), 0, np.ascontiguousarray(qperm),
                                                 T, S) - base)) <= 1e-12
    k2 = k.copy()
    k2[:, :, 5] = (k2[:, :, 5].astype(np.float32) * 2).astype(np.float16)     # whole token row x2 (exact)
    assert np.max(np.abs(orc.window_scores_layer(k2, 0, q, T, S) - base)) <= 1e-12


# --------------------------------------------------------------------------------------
# Paper-literal group quantization (reading Q37)
# --------------------------------------------------------------------------------------
def _group_case(orc, K, V, S, d, bits):
    """One request, one head, one window of class `bits` -> (record bytes, image)."""
    g = orc.geom(1, 1, 1, d, S, S, [bits])
    perm = np.zeros((1, 1), np.int32)
    cls = {2: 0, 4: 1, 8: 2, 16: 3}[bits]
    seg = np.array([[0] * (cls + 1) + [1] * (4 - cls)], np.int32)
    pk, offs = orc.reorder_quantize_pack(K.reshape(1, 1, S, d), V.reshape(1, 1, S, d), 0, g, perm, seg, gran=1)
    return pk[:int(offs[-1])], offs


def test_group_record_bytes_closed_form(orc):
    for d in (64, 128):
        for S in (16, 32, 64, 128):
            for b in (2, 4, 8):
                assert orc.record_bytes(b, d, S, 1) == S * d * b // 4 + 16
            assert orc.record_bytes(16, d, S, 1) == 4 * S * d


def test_group_quantizer_hand_golden(orc):
    """K values cycling through -3..3 (fp16-exact), V = 2 * K; 2-bit groups: mn_K = -3, range 6,
    s_K = RU(6/3) = 2 (0x4000), codes rint((x + 3) / 2) half-even: -3,-2 -> 0, -1 -> 1,
    0 -> 2 (1.5 -> 2), 1 -> 2, 2 -> 2 (2.5 -> 2), 3 -> 3; V: mn_V = -6 (0xC600), s_V = 4 (0x4400),
    the same codes.  The 16-byte block reads {mn_K, s_K, mn_V, s_V, 0, 0, 0, 0}."""
    S, d = 16, 64
    t, c = np.meshgrid(np.arange(S), np.arange(d), indexing="ij")
    K = (((t * d + c) % 7) - 3).astype(np.float16)
    V = (2 * K.astype(np.float32)).astype(np.float16)
    rec, _ = _group_case(orc, K, V, S, d, 2)
    assert len(rec) == S * d * 2 // 4 + 16
    blk = rec[2 * S * d * 2 // 8:].view(np.uint16)
    assert list(blk) == [0xC200, 0x4000, 0xC600, 0x4400, 0, 0, 0, 0]
    code_of = {-3: 0, -2: 0, -1: 1, 0: 2, 1: 2, 2: 2, 3: 3}
    kh, vh = orc.dequant_record(rec, 2, d, S, gran=1)
    want = np.vectorize(lambda x: -3 + 2 * code_of[int(x)])(K.astype(np.float64))
    assert np.array_equal(kh, want)
    assert np.array_equal(vh, 2 * want)


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_group_quantizer_error_bound(orc, bits):
    """Every element of the window is within s (1/2 + 2^-14) of its dequantized value, with the
    group's single scale s = the smallest fp16 >= fl32(range / q_max) over ALL S*d values
    (range from numpy, the rounding-up from numpy's float16: independent of the oracle)."""
    rng = np.random.default_rng(40 + bits)
    S, d = 32, 128
    qmax = 2 ** bits - 1
    for _ in range(6):
        K = (rng.standard_normal((S, d)) * rng.uniform(0.3, 2, d) + rng.standard_normal(d) * 3).astype(np.float16)
        V = (rng.standard_normal((S, d)) * np.exp(0.5 * rng.standard_normal((S, 1)))).astype(np.float16)
        rec, _ = _group_case(orc, K, V, S, d, bits)
        kh, vh = orc.dequant_record(rec, bits, d, S, gran=1)
        for X, Xh, off in ((K, kh, 2), (V, vh, 6)):
            x = X.astype(np.float64)
            rng32 = np.float32(np.float32(x.max()) - np.float32(x.min())) / np.float32(qmax)
            s = _ru_reference(np.array([rng32], np.float32))[0].view(np.float16).astype(np.float64)
            blk = rec[2 * S * d * bits // 8:].view(np.uint16)
            assert blk[off // 2] == np.float16(s).view(np.uint16)
            assert np.all(np.abs(x - Xh) <= s * (0.5 + 2 ** -14))


def test_group_decode_exact_on_lattice(orc):
    """Windows whose K and V values lie on a power-of-two lattice of their group (x = mn + s k,
    k in [0, q_max], both extremes present) round-trip exactly, so the group-quantized decode
    (gran 1) equals fp64 brute-force attention on the original fp16 tokens."""
    rng = np.random.default_rng(44)
    B, H, Hq, d, S, W = 2, 2, 6, 64, 16, 5
    M = W * S
    bits_w = [16, 2, 4, 8, 2]
    K = np.zeros((B, H, M, d), np.float16)
    V = np.zeros((B, H, M, d), np.float16)
    for b in range(B):
        for h in range(H):
            for w, bw in enumerate(bits_w):
                qm = 2 ** min(bw, 8) - 1
                for X in (K, V):
                    s, mn = 2.0 ** int(rng.integers(-4, 0)), float(rng.integers(-8, 8))
                    k = rng.integers(0, qm + 1, (S, d))
                    k.flat[0], k.flat[1] = 0, qm
                    X[b, h, w * S:(w + 1) * S] = (mn + s * k).astype(np.float16)
    order = [i for cls in (2, 4, 8, 16) for i, x in enumerate(bits_w) if x == cls]
    perm = np.array([order] * B, np.int32)
    seg = np.array([[0, 2, 3, 4, 5]] * B, np.int32)
    g = orc.geom(B, H, Hq, d, M, S, [2, 4, 8, 16])
    pk, offs = orc.reorder_quantize_pack(K, V, 0, g, perm, seg, gran=1)
    q = rng.standard_normal((B, Hq, d)).astype(np.float16)
    kr = rng.standard_normal((B, H, 3, d)).astype(np.float16)
    vr = rng.standard_normal((B, H, 3, d)).astype(np.float16)
    rl = np.array([3, 2], np.int32)
    got = orc.decode_attention(q, pk, offs, seg, perm, g, kr, vr, rl, 0.125, gran=1)
    win = np.tile(np.arange(W, dtype=np.int32), (B, 1))
    ref = orc.bruteforce_attention(q, K, V, 0, g, win, np.array([W] * B, np.int32), kr, vr, rl, 0.125)
    assert np.max(np.abs(got - ref)) <= 1e-12
