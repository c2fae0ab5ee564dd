"""CPU oracle for the WindowQuant hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference leg may import this package.  The product path
(``paper_2605_02262_b200``) never imports it and shares no code with it; the
two meet only on the seeded input tensors of ``paper_2605_02262_b200.synth``.

This module builds ``liboracle.so`` from ``wqo.c`` with gcc and exposes numpy
wrappers with the names of the C functions (``wqo_*`` minus the prefix).
fp16 arrays are passed as their raw bit patterns.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wqo.c")
_HDR = os.path.join(_HERE, "wqo.h")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c99", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
          "-fopenmp", "-shared", "-fPIC", "-Wall", "-Wno-unused-function"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2 -ffp-contract=off -fno-fast-math)."""
    stale = (not os.path.exists(_LIB_PATH) or
             os.path.getmtime(_LIB_PATH) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Geom(C.Structure):
    _fields_ = [("B", C.c_int32), ("H", C.c_int32), ("Hq", C.c_int32), ("d", C.c_int32),
                ("M", C.c_int32), ("S", C.c_int32), ("n_widths", C.c_int32),
                ("widths", C.c_int32 * 4)]


def geom(B, H, Hq, d, M, S, widths) -> Geom:
    w = list(widths) + [0] * (4 - len(widths))
    return Geom(B, H, Hq, d, M, S, len(widths), (C.c_int32 * 4)(*w))


P = C.c_void_p
I32, I64, F32, F64 = C.c_int32, C.c_int64, C.c_float, C.c_double


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB_PATH)
            sig = {
                "wqo_f16_to_f64": (F64, [C.c_uint16]),
                "wqo_f32_to_f16_ru": (C.c_uint16, [F32]),
                "wqo_f32_to_f16_rn": (C.c_uint16, [F32]),
                "wqo_f1": (F64, [F64, F64]),
                "wqo_f2": (F64, [F64, F64]),
                "wqo_thresholds": (C.c_int, [P, I32, F64, I32, P]),
                "wqo_window_score": (F64, [P, I64, P, I64, I32, I32, I32, I32]),
                "wqo_window_scores": (None, [P, I64, I64, P, I64, I64, I32, I32, I32, I32, I32, P]),
                "wqo_window_scores_pearson": (None, [P, I64, I64, P, I64, I64, I32, I32, I32, I32, I32, P]),
                "wqo_window_scores_layer": (None, [P, P, I32, P, P, I32, I32, I32, I32, I32, I32, I32, P]),
                "wqo_assign_bits": (C.c_int, [P, P, I32, C.POINTER(Geom), F64, I32, I32, P, P, P, P]),
                "wqo_record_bytes": (I64, [I32, I32, I32]),
                "wqo_packed_bytes": (I64, [C.POINTER(Geom), P, I32]),
                "wqo_kv_code_bytes": (I64, [P, I32, I32]),
                "wqo_layer_layout": (None, [C.POINTER(Geom), P, P]),
                "wqo_quantize_group": (None, [P, I32, I64, I32, P, P, P]),
                "wqo_code_pos": (None, [I32, I32, I32, I32, I32, P, P]),
                "wqo_param_pos": (C.c_int64, [I32, I32, I32, I32]),
                "wqo_reorder_quantize_pack": (None, [P, P, P, I32, C.POINTER(Geom), P, I32, P, P, P]),
                "wqo_dequant_record": (None, [P, I32, I32, I32, P, P]),
                "wqo_decode_attention": (None, [P, P, P, P, P, I32, C.POINTER(Geom), P, P, P, P,
                                                F32, P, P]),
                "wqo_bruteforce_attention": (None, [P, P, P, P, I32, C.POINTER(Geom), P, I32, P,
                                                    P, P, P, P, F32, P]),
                "wqo_merge": (None, [P, I32, I32, I32, P]),
                "wqo_f64_to_f16_rn": (C.c_uint16, [F64]),
                "wqo_dequantize_image": (None, [P, P, P, C.POINTER(Geom), P, P]),
                "wqo_record_bytes_g": (I64, [I32, I32, I32, I32]),
                "wqo_layer_layout_g": (None, [C.POINTER(Geom), P, P, I32]),
                "wqo_reorder_quantize_pack_g": (None, [P, P, P, I32, C.POINTER(Geom), P, I32, P, P, P, I32]),
                "wqo_dequant_record_g": (None, [P, I32, I32, I32, P, P, I32]),
                "wqo_decode_attention_g": (None, [P, P, P, P, P, I32, C.POINTER(Geom), P, P, P, P, F32, P, P, I32]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def _u16(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    return a.view(np.uint16) if a.dtype == np.float16 else a.astype(np.uint16)


# --- scalar conversions ------------------------------------------------------
def f16_to_f64(h: int) -> float:
    return lib().wqo_f16_to_f64(h)


def f32_to_f16_ru(x: float) -> int:
    return lib().wqo_f32_to_f16_ru(x)


def f32_to_f16_rn(x: float) -> int:
    return lib().wqo_f32_to_f16_rn(x)


# --- Eq.10-11 -----------------------------------------------------------------
def f1(s, alpha):
    return lib().wqo_f1(s, alpha)


def f2(s, alpha):
    return lib().wqo_f2(s, alpha)


def thresholds(s, alpha, n_widths):
    s = np.ascontiguousarray(s, dtype=np.float64)
    thr = np.zeros((len(s), max(n_widths - 1, 0)), np.float64)
    rc = lib().wqo_thresholds(_p(s), len(s), alpha, n_widths, _p(thr) if thr.size else None)
    if rc:
        raise ValueError("wqo_thresholds: invalid argument")
    return thr


# --- Eq.8 -----------------------------------------------------------------------
def window_scores(vis: np.ndarray, txt: np.ndarray, S: int) -> np.ndarray:
    """vis [B][M][D] fp16, txt [B][N][D] fp16 -> scores [B][M//S] fp64."""
    vis, txt = _u16(vis), _u16(txt)
    B, M, D = vis.shape
    N = txt.shape[1]
    out = np.zeros((B, M // S), np.float64)
    lib().wqo_window_scores(_p(vis), D, M * D, _p(txt), D, N * D, B, M, N, D, S, _p(out))
    return out


def window_scores_pearson(vis: np.ndarray, txt: np.ndarray, S: int) -> np.ndarray:
    """T11 variant: Eq.8 with the Pearson correlation of every (text, window) token pair."""
    vis, txt = _u16(vis), _u16(txt)
    B, M, D = vis.shape
    N = txt.shape[1]
    out = np.zeros((B, M // S), np.float64)
    lib().wqo_window_scores_pearson(_p(vis), D, M * D, _p(txt), D, N * D, B, M, N, D, S, _p(out))
    return out


def window_scores_layer(k: np.ndarray, vis_off: int, q_text: np.ndarray, M: int, S: int) -> np.ndarray:
    """Per-layer scorer (reading Q36): k fp16 [B][H][T][d], q_text fp16 [B][Hq][N][d] -> [B][M//S]."""
    k, q_text = _u16(k), _u16(q_text)
    B, H, T, d = k.shape
    Hq, N = q_text.shape[1], q_text.shape[2]
    ks = np.array([H * T * d, T * d, d], np.int64)
    qs = np.array([Hq * N * d, N * d, d], np.int64)
    out = np.zeros((B, M // S), np.float64)
    lib().wqo_window_scores_layer(_p(k), _p(ks), vis_off, _p(q_text), _p(qs), B, H, Hq, d, M, N, S, _p(out))
    return out


def window_score(vis_b: np.ndarray, txt_b: np.ndarray, S: int, w: int) -> float:
    vis_b, txt_b = _u16(vis_b), _u16(txt_b)
    M, D = vis_b.shape
    N = txt_b.shape[0]
    return lib().wqo_window_score(_p(vis_b), D, _p(txt_b), D, N, D, S, w)


# --- Alg.1 + Alg.2 partition ----------------------------------------------------------
def assign_bits(scores, thr, g: Geom, budget=0.0, pin=1, vote=0):
    scores = np.ascontiguousarray(scores, np.float64)
    thr = np.ascontiguousarray(thr, np.float64)
    L = thr.shape[0]
    B, W = g.B, g.M // g.S
    bits = np.zeros((L, B, W), np.uint8)
    rank = np.zeros((B, W), np.int32)
    perm = np.zeros((L, B, W), np.int32)
    seg = np.zeros((L, B, 5), np.int32)
    rc = lib().wqo_assign_bits(_p(scores), _p(thr) if thr.size else None, L, C.byref(g),
                               float(budget), int(pin), int(vote), _p(bits), _p(rank), _p(perm),
                               _p(seg))
    if rc == 3:
        raise ValueError("budget infeasible")
    return bits, rank, perm, seg


# --- byte accounting -------------------------------------------------------------
def record_bytes(bits, d, S, gran=0):
    return lib().wqo_record_bytes_g(bits, d, S, gran)


def packed_bytes(g: Geom, n_per_class, code_only=False):
    n = np.ascontiguousarray(n_per_class, np.int32)
    return lib().wqo_packed_bytes(C.byref(g), _p(n), int(code_only))


def kv_code_bytes(tokens_per_class, d, H):
    t = np.ascontiguousarray(tokens_per_class, np.int64)
    return lib().wqo_kv_code_bytes(_p(t), d, H)


def layer_layout(g: Geom, seg_off_l: np.ndarray, gran=0) -> np.ndarray:
    seg_off_l = np.ascontiguousarray(seg_off_l, np.int32)
    offs = np.zeros(g.B * g.H + 1, np.int64)
    lib().wqo_layer_layout_g(C.byref(g), _p(seg_off_l), _p(offs), int(gran))
    return offs


# --- Eq.14-16 -------------------------------------------------------------------------
def quantize_group(x: np.ndarray, bits: int):
    """x: 1-D fp16 -> (s_bits u16, mn_bits u16, codes u8[n])."""
    x = _u16(x)
    s = np.zeros(1, np.uint16)
    mn = np.zeros(1, np.uint16)
    codes = np.zeros(len(x), np.uint8)
    lib().wqo_quantize_group(_p(x), len(x), 1, bits, _p(s), _p(mn), _p(codes))
    return int(s[0]), int(mn[0]), codes


def param_pos(is_v, d, i, is_min):
    """Byte offset of K channel / V token i's scale (is_min=0) or zero point inside the params."""
    return int(lib().wqo_param_pos(is_v, d, i, is_min))


def code_pos(is_v, d, b, t, c):
    bo = np.zeros(1, np.int64)
    bit = np.zeros(1, np.int32)
    lib().wqo_code_pos(is_v, d, b, t, c, _p(bo), _p(bit))
    return int(bo[0]), int(bit[0])


def reorder_quantize_pack(k, v, vis_off, g: Geom, perm_l, seg_off_l, offs=None, gran=0):
    """k, v: fp16 [B][H][T][d] -> packed u8 image of one layer (D-1; gran 1: P:508 groups)."""
    k, v = _u16(k), _u16(v)
    perm_l = np.ascontiguousarray(perm_l, np.int32)
    seg_off_l = np.ascontiguousarray(seg_off_l, np.int32)
    if offs is None:
        offs = layer_layout(g, seg_off_l, gran)
    B, H, T, d = k.shape
    strides = np.array([H * T * d, T * d, d], np.int64)
    packed = np.zeros(max(int(offs[-1]), 16), np.uint8)
    lib().wqo_reorder_quantize_pack_g(_p(k), _p(v), _p(strides), vis_off, C.byref(g), _p(perm_l),
                                      perm_l.shape[-1], _p(seg_off_l), _p(offs), _p(packed), int(gran))
    return packed, offs


def dequant_record(rec: np.ndarray, bits, d, S, gran=0):
    rec = np.ascontiguousarray(rec, np.uint8)
    kh = np.zeros((S, d), np.float64)
    vh = np.zeros((S, d), np.float64)
    lib().wqo_dequant_record_g(_p(rec), bits, d, S, _p(kh), _p(vh), int(gran))
    return kh, vh


def decode_attention(q, packed, offs, seg_off_l, perm_l, g: Geom, k_rest, v_rest, rest_len,
                     sm_scale, want_partial=False, gran=0):
    """q fp16 [B][Hq][d]; k_rest/v_rest fp16 [B][H][R][d]; -> out fp64 [B][Hq][d] (, partial)."""
    q, k_rest, v_rest = _u16(q), _u16(k_rest), _u16(v_rest)
    B, H, R, d = k_rest.shape
    rs = np.array([H * R * d, R * d], np.int64)
    rest_len = np.clip(np.ascontiguousarray(rest_len, np.int32), 0, R)   # contract: clamped to R_max
    perm_l = np.ascontiguousarray(perm_l, np.int32)
    seg_off_l = np.ascontiguousarray(seg_off_l, np.int32)
    out = np.zeros((g.B, g.Hq, g.d), np.float64)
    part = np.zeros((g.B, g.Hq, g.d + 2), np.float64) if want_partial else None
    lib().wqo_decode_attention_g(_p(q), _p(np.ascontiguousarray(packed)), _p(np.ascontiguousarray(offs)),
                                 _p(seg_off_l), _p(perm_l), perm_l.shape[-1], C.byref(g),
                                 _p(k_rest), _p(v_rest), _p(rs), _p(rest_len), float(sm_scale),
                                 _p(out), _p(part), int(gran))
    return (out, part) if want_partial else out


def bruteforce_attention(q, k, v, vis_off, g: Geom, win_l, n_win, k_rest, v_rest, rest_len, sm_scale):
    q, k, v, k_rest, v_rest = _u16(q), _u16(k), _u16(v), _u16(k_rest), _u16(v_rest)
    B, H, T, d = k.shape
    strides = np.array([H * T * d, T * d, d], np.int64)
    R = k_rest.shape[2]
    rs = np.array([H * R * d, R * d], np.int64)
    win_l = np.ascontiguousarray(win_l, np.int32)
    n_win = np.ascontiguousarray(n_win, np.int32)
    rest_len = np.ascontiguousarray(rest_len, np.int32)
    out = np.zeros((g.B, g.Hq, g.d), np.float64)
    lib().wqo_bruteforce_attention(_p(q), _p(k), _p(v), _p(strides), vis_off, C.byref(g), _p(win_l),
                                   win_l.shape[-1], _p(n_win), _p(k_rest), _p(v_rest), _p(rs),
                                   _p(rest_len), float(sm_scale), _p(out))
    return out


def merge(parts: np.ndarray) -> np.ndarray:
    """parts fp64 [G][B][Hq][d+2] -> out fp64 [B][Hq][d]."""
    parts = np.ascontiguousarray(parts, np.float64)
    G, B, Hq, d2 = parts.shape
    out = np.zeros((B, Hq, d2 - 2), np.float64)
    lib().wqo_merge(_p(parts), G, B * Hq, d2 - 2, _p(out))
    return out


def f64_to_f16_rn(x: float) -> int:
    return int(lib().wqo_f64_to_f16_rn(float(x)))


def dequantize_image(packed, offs, seg_off_l, g: Geom):
    """T9 unfused baseline: the FP16 image (u8) of a packed layer image and its (b, h) offsets."""
    seg_off_l = np.ascontiguousarray(seg_off_l, np.int32)
    seg16 = np.zeros_like(seg_off_l)
    seg16[:, 4] = seg_off_l[:, 4]
    offs16 = layer_layout(g, seg16)
    img16 = np.zeros(max(int(offs16[-1]), 16), np.uint8)
    lib().wqo_dequantize_image(_p(np.ascontiguousarray(packed, np.uint8)), _p(np.ascontiguousarray(offs, np.int64)),
                               _p(seg_off_l), C.byref(g), _p(offs16), _p(img16))
    return img16, offs16, seg16
