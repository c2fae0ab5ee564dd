"""Thin Python binding of libwq.so (include/wq.h) -- argument marshalling only.

Every function has the name of the C entry point it calls; tensors are passed as
raw device pointers on torch's current CUDA stream.  All computation happens in
the CUDA kernels of ``csrc/``; when the library is missing this module raises
instead of falling back to anything else.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import build as _build

_LIB = None

P = C.c_void_p
I32, I64, F32, F64, SZ = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_size_t

WQ_OK, WQ_EINVAL, WQ_ESHAPE, WQ_EBUDGET, WQ_EUNSUPPORTED, WQ_ECUDA = range(6)
CLASS_BITS = (2, 4, 8, 16)


class WQError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"wq status {status}: {msg}")
        self.status = status


class Geom(C.Structure):
    _fields_ = [("B", I32), ("H", I32), ("Hq", I32), ("d", I32), ("M", I32), ("S", I32),
                ("n_widths", I32), ("widths", I32 * 4)]


class AssignOpts(C.Structure):
    _fields_ = [("budget_avg_bits", F64), ("pin_first", I32), ("batch_vote", I32)]


def geom(B, H, Hq, d, M, S, widths) -> Geom:
    w = list(widths) + [0] * (4 - len(widths))
    return Geom(B, H, Hq, d, M, S, len(widths), (I32 * 4)(*w))


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libwq.so (building it in-tree with nvcc if it is missing)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _build.LIB
    if not os.path.exists(path):
        if not build_if_missing:
            raise FileNotFoundError(f"{path} missing: run python -m paper_2605_02262_b200.build")
        _build.build()
    L = C.CDLL(path)
    sig = {
        "wq_thresholds": [P, I32, F64, I32, P],
        "wq_window_scores_workspace": [I32, I32, P],
        "wq_window_scores": [P, I64, I64, P, I64, I64, I32, I32, I32, I32, I32, P, P, SZ, P],
        "wq_window_scores_ex": [P, I64, I64, P, I64, I64, I32, I32, I32, I32, I32, I32, P, P, SZ, P],
        "wq_window_scores_layer": [P, P, I32, P, P, I32, I32, I32, I32, I32, I32, I32, P, P, SZ, P],
        "wq_assign_bits": [P, P, I32, C.POINTER(Geom), C.POINTER(AssignOpts), P, P, P, P, P],
        "wq_search_workspace": [I32, I32, I32, P],
        "wq_search": [P, I64, I64, P, I64, I64, I32, I32, I32, P, I32, C.POINTER(Geom), C.POINTER(AssignOpts), P, P,
                      P, P, P, P, SZ, P],
        "wq_packed_bytes": [C.POINTER(Geom), P, I32, P],
        "wq_packed_bytes_ex": [C.POINTER(Geom), P, I32, I32, P],
        "wq_layer_layout": [C.POINTER(Geom), P, P, P],
        "wq_layer_layout_ex": [C.POINTER(Geom), P, I32, P, P],
        "wq_reorder_quantize_pack": [P, P, P, I32, C.POINTER(Geom), P, I32, P, P, P, P],
        "wq_reorder_quantize_pack_ex": [P, P, P, I32, C.POINTER(Geom), P, I32, P, P, I32, P, P],
        "wq_decode_workspace": [C.POINTER(Geom), P],
        "wq_decode_attention": [P, P, P, P, C.POINTER(Geom), P, P, P, P, I32, F32, P, P, P, SZ, P],
        "wq_decode_attention_ex": [P, P, P, P, C.POINTER(Geom), P, P, P, P, I32, F32, P, P, P, SZ, C.c_uint32, P],
        "wq_merge_partials": [P, I32, C.POINTER(Geom), P, P],
        "wq_shard_slots": [P, P, I32, I32, I32, I32, P, P, P],
        "wq_dequant_layout": [C.POINTER(Geom), P, P, P, P],
        "wq_dequantize_image": [P, P, P, C.POINTER(Geom), P, P, P],
        "wq_unreordered_layout": [C.POINTER(Geom), P, P, P],
        "wq_peer_buffer_bytes": [C.POINTER(Geom), I32, P],
        "wq_peer_error_offset": [C.POINTER(Geom), I32, P],
        "wq_decode_attention_peer": [P, P, P, P, C.POINTER(Geom), P, P, P, P, I32, F32, P, P, SZ, P, P, I32, I32,
                                     C.c_uint32, P],
        "wq_decode_attention_peer_emulated": [I32, P, P, P, P, C.POINTER(Geom), P, P, P, P, I32, F32, P, P, SZ, P,
                                              P, C.c_uint32, P],
        "wq_unreorder_image": [P, P, P, P, C.POINTER(Geom), P, P, P],
        "wq_decode_attention_unreordered": [P, P, P, P, P, C.POINTER(Geom), P, P, P, P, I32, F32, P, P, P, SZ, P],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.wq_last_error.restype = C.c_char_p
    L.wq_last_error.argtypes = []
    L.wq_version.restype = C.c_char_p
    L.wq_version.argtypes = []
    _LIB = L
    return L


def exported_symbols():
    return ["wq_thresholds", "wq_window_scores_workspace", "wq_window_scores", "wq_window_scores_ex",
            "wq_window_scores_layer", "wq_assign_bits", "wq_search_workspace", "wq_search",
            "wq_packed_bytes", "wq_packed_bytes_ex", "wq_layer_layout", "wq_layer_layout_ex",
            "wq_reorder_quantize_pack", "wq_reorder_quantize_pack_ex", "wq_decode_workspace",
            "wq_decode_attention", "wq_decode_attention_ex", "wq_merge_partials", "wq_shard_slots", "wq_dequant_layout", "wq_dequantize_image",
            "wq_unreordered_layout", "wq_unreorder_image", "wq_decode_attention_unreordered",
            "wq_peer_buffer_bytes", "wq_peer_error_offset", "wq_decode_attention_peer",
            "wq_decode_attention_peer_emulated", "wq_last_error", "wq_version"]


def _check(rc: int):
    if rc != WQ_OK:
        raise WQError(rc, load().wq_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return C.c_void_p(t.data_ptr())
    return t


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _host_ptr(a):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------------------------------
def wq_version() -> str:
    return load().wq_version().decode()


def wq_thresholds(s, alpha: float, n_widths: int):
    """Eq.10-11 (host).  s: sequence of per-layer sensitivities -> numpy [L][n-1]."""
    import numpy as np
    s = np.ascontiguousarray(s, dtype=np.float64)
    thr = np.zeros((len(s), max(n_widths - 1, 1)), np.float64)
    _check(load().wq_thresholds(_host_ptr(s), len(s), float(alpha), int(n_widths), _host_ptr(thr)))
    return thr[:, :max(n_widths - 1, 0)]


def wq_window_scores_workspace(B: int, D: int) -> int:
    n = C.c_size_t(0)
    _check(load().wq_window_scores_workspace(B, D, C.byref(n)))
    return n.value


WQ_SIM_COSINE, WQ_SIM_PEARSON = 0, 1


def wq_window_scores(vis: torch.Tensor, txt: torch.Tensor, S: int, scores=None, workspace=None, stream=None,
                     metric: int = WQ_SIM_COSINE):
    """vis fp16 [B][M][D] (rows contiguous), txt fp16 [B][N][D] -> scores fp64 [B][M//S].
    metric: WQ_SIM_COSINE (Eq.8) or WQ_SIM_PEARSON (T11 variant) -> wq_window_scores_ex."""
    B, M, D = vis.shape
    N = txt.shape[1]
    if scores is None:
        scores = torch.empty((B, M // S), dtype=torch.float64, device=vis.device)
    if workspace is None:
        workspace = torch.empty(wq_window_scores_workspace(B, D), dtype=torch.uint8, device=vis.device)
    if metric == WQ_SIM_COSINE:
        _check(load().wq_window_scores(_ptr(vis), vis.stride(1), vis.stride(0), _ptr(txt), txt.stride(1),
                                       txt.stride(0), B, M, N, D, S, _ptr(scores), _ptr(workspace),
                                       workspace.numel(), _stream(stream)))
    else:
        _check(load().wq_window_scores_ex(_ptr(vis), vis.stride(1), vis.stride(0), _ptr(txt), txt.stride(1),
                                          txt.stride(0), B, M, N, D, S, int(metric), _ptr(scores),
                                          _ptr(workspace), workspace.numel(), _stream(stream)))
    return scores


def wq_assign_bits(scores: torch.Tensor, thr, L: int, g: Geom, opts: AssignOpts | None = None,
                   bits=None, rank=None, perm=None, seg_off=None, want_rank=True, stream=None):
    import numpy as np
    B, W = g.B, g.M // g.S
    dev = scores.device
    if bits is None:
        bits = torch.empty((L, B, W), dtype=torch.uint8, device=dev)
    if perm is None:
        perm = torch.empty((L, B, W), dtype=torch.int32, device=dev)
    if seg_off is None:
        seg_off = torch.empty((L, B, 5), dtype=torch.int32, device=dev)
    if rank is None and want_rank:
        rank = torch.empty((B, W), dtype=torch.int32, device=dev)
    if opts is None:
        opts = AssignOpts(0.0, 1, 0)
    thr = np.ascontiguousarray(thr, dtype=np.float64).reshape(L, -1)
    thr_p = _host_ptr(thr) if thr.size else None
    _check(load().wq_assign_bits(_ptr(scores), thr_p, L, C.byref(g), C.byref(opts), _ptr(bits), _ptr(rank),
                                 _ptr(perm), _ptr(seg_off), _stream(stream)))
    return bits, rank, perm, seg_off


WQ_GRAN_CHANNEL_TOKEN, WQ_GRAN_GROUP = 0, 1


def wq_packed_bytes(g: Geom, n_per_class, code_bytes_only: bool = False, gran: int = 0) -> int:
    """gran: WQ_GRAN_* (non-zero calls wq_packed_bytes_ex)."""
    import numpy as np
    n = np.ascontiguousarray(n_per_class, dtype=np.int32)
    out = C.c_int64(0)
    if gran:
        _check(load().wq_packed_bytes_ex(C.byref(g), _host_ptr(n), int(code_bytes_only), int(gran), C.byref(out)))
    else:
        _check(load().wq_packed_bytes(C.byref(g), _host_ptr(n), int(code_bytes_only), C.byref(out)))
    return out.value


def wq_layer_layout(g: Geom, seg_off_l: torch.Tensor, offs=None, stream=None, gran: int = 0) -> torch.Tensor:
    if offs is None:
        offs = torch.empty(g.B * g.H + 1, dtype=torch.int64, device=seg_off_l.device)
    if gran:
        _check(load().wq_layer_layout_ex(C.byref(g), _ptr(seg_off_l), int(gran), _ptr(offs), _stream(stream)))
    else:
        _check(load().wq_layer_layout(C.byref(g), _ptr(seg_off_l), _ptr(offs), _stream(stream)))
    return offs


def wq_reorder_quantize_pack(k: torch.Tensor, v: torch.Tensor, vis_off: int, g: Geom, perm_l: torch.Tensor,
                             seg_off_l: torch.Tensor, offs: torch.Tensor, packed: torch.Tensor, stream=None,
                             gran: int = 0):
    """k, v fp16 [B][H][T][d] (channel stride 1); perm_l i32 [B][Ws]; seg_off_l i32 [B][5].
    gran: WQ_GRAN_* (non-zero calls wq_reorder_quantize_pack_ex)."""
    assert k.stride() == v.stride() and k.stride(3) == 1
    strides = (C.c_int64 * 3)(k.stride(0), k.stride(1), k.stride(2))
    L = load()
    head = (_ptr(k), _ptr(v), strides, vis_off, C.byref(g), _ptr(perm_l), perm_l.shape[-1], _ptr(seg_off_l),
            _ptr(offs))
    if gran:
        _check(L.wq_reorder_quantize_pack_ex(*head, int(gran), _ptr(packed), _stream(stream)))
    else:
        _check(L.wq_reorder_quantize_pack(*head, _ptr(packed), _stream(stream)))
    return packed


def wq_decode_workspace(g: Geom) -> int:
    n = C.c_size_t(0)
    _check(load().wq_decode_workspace(C.byref(g), C.byref(n)))
    return n.value


WQ_DECODE_EARLY = 1
WQ_DECODE_GROUP = 2     # the image is WQ_GRAN_GROUP


def wq_decode_attention(q: torch.Tensor, packed: torch.Tensor, offs: torch.Tensor, seg_off_l: torch.Tensor,
                        g: Geom, k_rest, v_rest, rest_len, sm_scale: float, out=None, partial=None,
                        workspace=None, stream=None, flags: int = 0):
    """q fp16 [B][Hq][d]; k_rest/v_rest fp16 [B][H][R_max][d] (or None); rest_len i32 [B].
    flags: WQ_DECODE_EARLY | WQ_DECODE_GROUP (see include/wq.h) calls wq_decode_attention_ex."""
    if workspace is None:
        workspace = torch.zeros(wq_decode_workspace(g), dtype=torch.uint8, device=q.device)
    R_max = 0 if k_rest is None else k_rest.shape[2]
    rs = (C.c_int64 * 2)(*(k_rest.stride(0), k_rest.stride(1))) if k_rest is not None else None
    args = (_ptr(q), _ptr(packed), _ptr(offs), _ptr(seg_off_l), C.byref(g), _ptr(k_rest), _ptr(v_rest), rs,
            _ptr(rest_len), R_max, float(sm_scale), _ptr(out), _ptr(partial), _ptr(workspace), workspace.numel())
    if flags:
        _check(load().wq_decode_attention_ex(*args, int(flags), _stream(stream)))
    else:
        _check(load().wq_decode_attention(*args, _stream(stream)))
    return out, partial


def wq_merge_partials(parts: torch.Tensor, g: Geom, out=None, stream=None) -> torch.Tensor:
    """parts fp32 [G][B][Hq][d+2] -> out fp16 [B][Hq][d]."""
    if out is None:
        out = torch.empty((g.B, g.Hq, g.d), dtype=torch.float16, device=parts.device)
    _check(load().wq_merge_partials(_ptr(parts), parts.shape[0], C.byref(g), _ptr(out), _stream(stream)))
    return out


def wq_shard_slots(perm_l: torch.Tensor, seg_off_l: torch.Tensor, G: int, r: int, perm_r=None, seg_off_r=None,
                   stream=None):
    """Rank r's slots of the sequence split: perm_l i32 [B][W], seg_off_l i32 [B][5]."""
    B, W = perm_l.shape
    if perm_r is None:
        perm_r = torch.zeros_like(perm_l)
    if seg_off_r is None:
        seg_off_r = torch.empty_like(seg_off_l)
    _check(load().wq_shard_slots(_ptr(perm_l), _ptr(seg_off_l), B, W, G, r, _ptr(perm_r), _ptr(seg_off_r),
                                 _stream(stream)))
    return perm_r, seg_off_r


def wq_dequant_layout(g: Geom, seg_off_l: torch.Tensor, stream=None):
    """(seg16 i32 [B][5], offs16 i64 [B*H+1]) of the FP16 image of the unfused baseline (T9)."""
    seg16 = torch.empty_like(seg_off_l)
    offs16 = torch.empty(g.B * g.H + 1, dtype=torch.int64, device=seg_off_l.device)
    _check(load().wq_dequant_layout(C.byref(g), _ptr(seg_off_l), _ptr(seg16), _ptr(offs16), _stream(stream)))
    return seg16, offs16


def wq_dequantize_image(packed: torch.Tensor, offs: torch.Tensor, seg_off_l: torch.Tensor, g: Geom,
                        offs16: torch.Tensor, img16: torch.Tensor, stream=None) -> torch.Tensor:
    """Dequantize every record of a packed layer image into the FP16 image img16 (T9 unfused path)."""
    _check(load().wq_dequantize_image(_ptr(packed), _ptr(offs), _ptr(seg_off_l), C.byref(g), _ptr(offs16),
                                      _ptr(img16), _stream(stream)))
    return img16


def wq_unreordered_layout(g: Geom, bits_l: torch.Tensor, woff=None, stream=None) -> torch.Tensor:
    """woff i64 [B][W+1]: original-order record offsets of the unreordered image (T8 baseline)."""
    B, W = bits_l.shape
    if woff is None:
        woff = torch.empty((B, W + 1), dtype=torch.int64, device=bits_l.device)
    _check(load().wq_unreordered_layout(C.byref(g), _ptr(bits_l), _ptr(woff), _stream(stream)))
    return woff


def wq_unreorder_image(packed, offs, seg_off_l, perm_l, g: Geom, woff, uimg, stream=None):
    """Copy the packed (reordered) image's records into original window order (T8 baseline)."""
    _check(load().wq_unreorder_image(_ptr(packed), _ptr(offs), _ptr(seg_off_l), _ptr(perm_l), C.byref(g),
                                     _ptr(woff), _ptr(uimg), _stream(stream)))
    return uimg


def wq_decode_attention_unreordered(q, uimg, offs, seg_off_l, woff, g: Geom, k_rest, v_rest, rest_len,
                                    sm_scale: float, out=None, partial=None, workspace=None, stream=None):
    """Decode over the unreordered image (windows in original order, per-window width)."""
    if workspace is None:
        workspace = torch.zeros(wq_decode_workspace(g), dtype=torch.uint8, device=q.device)
    R_max = 0 if k_rest is None else k_rest.shape[2]
    rs = (C.c_int64 * 2)(*(k_rest.stride(0), k_rest.stride(1))) if k_rest is not None else None
    _check(load().wq_decode_attention_unreordered(_ptr(q), _ptr(uimg), _ptr(offs), _ptr(seg_off_l), _ptr(woff),
                                                  C.byref(g), _ptr(k_rest), _ptr(v_rest), rs, _ptr(rest_len), R_max,
                                                  float(sm_scale), _ptr(out), _ptr(partial), _ptr(workspace),
                                                  workspace.numel(), _stream(stream)))
    return out, partial


def wq_peer_buffer_bytes(g: Geom, G: int) -> int:
    n = C.c_size_t(0)
    _check(load().wq_peer_buffer_bytes(C.byref(g), int(G), C.byref(n)))
    return n.value


def wq_decode_attention_peer(q, packed, offs, seg_off_l, g: Geom, k_rest, v_rest, rest_len, sm_scale: float,
                             out, peer_ptrs: torch.Tensor, local_ptr: int, G: int, rank: int, epoch: int,
                             workspace=None, stream=None):
    """Decode of this rank's shard with the fused cross-GPU LSE merge: out receives the merged
    result of all G ranks.  peer_ptrs: int64 device tensor [G] of the symmetric buffers."""
    if workspace is None:
        workspace = torch.zeros(wq_decode_workspace(g), dtype=torch.uint8, device=q.device)
    R_max = 0 if k_rest is None else k_rest.shape[2]
    rs = (C.c_int64 * 2)(*(k_rest.stride(0), k_rest.stride(1))) if k_rest is not None else None
    _check(load().wq_decode_attention_peer(_ptr(q), _ptr(packed), _ptr(offs), _ptr(seg_off_l), C.byref(g),
                                           _ptr(k_rest), _ptr(v_rest), rs, _ptr(rest_len), R_max, float(sm_scale),
                                           _ptr(out), _ptr(workspace), workspace.numel(), _ptr(peer_ptrs),
                                           C.c_void_p(local_ptr), int(G), int(rank), C.c_uint32(epoch),
                                           _stream(stream)))
    return out


def wq_peer_error_offset(g: Geom, G: int) -> int:
    n = C.c_size_t(0)
    _check(load().wq_peer_error_offset(C.byref(g), int(G), C.byref(n)))
    return n.value


def wq_decode_attention_peer_emulated(ranks, g: Geom, sm_scale: float, peer_ptrs: torch.Tensor, local_ptrs, epoch: int,
                                      stream=None):
    """G = 2 virtual ranks of wq_decode_attention_peer in ONE launch on one GPU (tests of
    the fused cross-GPU merge without a second device).  ranks: list of G dicts with the
    keys q, packed, offs, seg_off, k_rest, v_rest, rest_len, out, workspace (tensors)."""
    G = len(ranks)
    arr = lambda key: (C.c_void_p * G)(*[ranks[r][key].data_ptr() for r in range(G)])
    kr = ranks[0]["k_rest"]
    R_max = kr.shape[2]
    rs = (C.c_int64 * 2)(*(kr.stride(0), kr.stride(1)))
    loc = (C.c_void_p * G)(*[int(x) for x in local_ptrs])
    _check(load().wq_decode_attention_peer_emulated(
        G, arr("q"), arr("packed"), arr("offs"), arr("seg_off"), C.byref(g), arr("k_rest"), arr("v_rest"), rs,
        arr("rest_len"), R_max, float(sm_scale), arr("out"), arr("workspace"), ranks[0]["workspace"].numel(),
        _ptr(peer_ptrs), loc, C.c_uint32(epoch), _stream(stream)))


def wq_window_scores_layer(k: torch.Tensor, vis_off: int, q_text: torch.Tensor, M: int, S: int, scores=None,
                           workspace=None, stream=None) -> torch.Tensor:
    """Per-layer scorer (include/wq.h): k fp16 [B][H][T][d] (any strides, rows contiguous),
    q_text fp16 [B][Hq][N][d] -> scores fp64 [B][M // S]."""
    B, H, T, d = k.shape
    Hq, N = q_text.shape[1], q_text.shape[2]
    if scores is None:
        scores = torch.empty((B, M // S), dtype=torch.float64, device=k.device)
    if workspace is None:
        workspace = torch.empty(wq_window_scores_workspace(B, H * d), dtype=torch.uint8, device=k.device)
    ks = (C.c_int64 * 3)(k.stride(0), k.stride(1), k.stride(2))
    qs = (C.c_int64 * 3)(q_text.stride(0), q_text.stride(1), q_text.stride(2))
    _check(load().wq_window_scores_layer(_ptr(k), ks, int(vis_off), _ptr(q_text), qs, B, H, Hq, d, int(M), N, int(S),
                                         _ptr(scores), _ptr(workspace), workspace.numel(), _stream(stream)))
    return scores


def wq_search(vis: torch.Tensor, txt: torch.Tensor, thr, L: int, g: Geom, opts: AssignOpts | None = None,
              metric: int = 0, outs=None, workspace=None, stream=None):
    """The fused search (include/wq.h wq_search): scores + rank + assignment of L layers in one
    launch.  Returns (scores, bits, rank, perm, seg_off)."""
    import numpy as np
    B, M, D = vis.shape
    N = txt.shape[1]
    W = M // g.S
    dev = vis.device
    if outs is None:
        outs = (torch.empty((B, W), dtype=torch.float64, device=dev), torch.empty((L, B, W), dtype=torch.uint8, device=dev),
                torch.empty((B, W), dtype=torch.int32, device=dev), torch.empty((L, B, W), dtype=torch.int32, device=dev),
                torch.empty((L, B, 5), dtype=torch.int32, device=dev))
    scores, bits, rank, perm, seg = outs
    if workspace is None:
        n = C.c_size_t(0)
        _check(load().wq_search_workspace(B, D, W, C.byref(n)))
        workspace = torch.empty(n.value, dtype=torch.uint8, device=dev)
    thr = np.ascontiguousarray(thr, np.float64)
    _check(load().wq_search(_ptr(vis), vis.stride(1), vis.stride(0), _ptr(txt), txt.stride(1), txt.stride(0), N, D,
                            int(metric), _host_ptr(thr) if thr.size else None, int(L), C.byref(g),
                            C.byref(opts) if opts is not None else None, _ptr(scores), _ptr(bits), _ptr(rank),
                            _ptr(perm), _ptr(seg), _ptr(workspace), workspace.numel(), _stream(stream)))
    return scores, bits, rank, perm, seg
