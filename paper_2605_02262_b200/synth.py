"""Seeded synthetic inputs — shared by the CUDA
path, the oracle tests and bench.py.

This module holds NONE of the method's arithmetic (no similarity, threshold,
assignment, quantization or attention math): it only draws tensors shaped like
LLaVA-OneVision / Qwen2 video workloads.  Everything is produced with a
``torch.Generator`` seeded from (config seed, layer, purpose), on the requested
device; the oracle consumes the very same tensors copied to the host.
"""
from __future__ import annotations

import math

import torch

# Fig.11 token proportions per layer: INT2 12,564 / INT4 6,956 / FP16 215
RELEVANCE_MIX = ((0.637, 0.05, 0.25), (0.352, 0.35, 0.65), (0.011, 0.80, 0.95))


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0x7FFFFFFFFFFFFFFF)
    return g


def _randn(shape, g, device):
    return torch.randn(shape, generator=g, device=device, dtype=torch.float32)


def _rand(shape, g, device):
    return torch.rand(shape, generator=g, device=device, dtype=torch.float32)


def window_relevance(B: int, W: int, seed: int, device="cpu") -> torch.Tensor:
    """rho[B][W] drawn from the Fig.11 mixture (63.7/35.2/1.1 %)."""
    g = _gen(seed * 7 + 1, device)
    u = _rand((B, W), g, device)
    r = _rand((B, W), g, device)
    rho = torch.empty((B, W), device=device)
    c0 = RELEVANCE_MIX[0][0]
    c1 = c0 + RELEVANCE_MIX[1][0]
    for (lo_p, hi_p), (_, a, b) in zip(((0.0, c0), (c0, c1), (c1, 1.01)), RELEVANCE_MIX):
        m = (u >= lo_p) & (u < hi_p)
        rho[m] = a + (b - a) * r[m]
    return rho


def embeddings(B: int, M: int, N: int, D: int, S: int, seed: int, device="cpu"):
    """Visual tokens vis[B][M][D] and text tokens txt[B][N][D] (fp16).

    u: a random unit direction per request; text t_j = u + 0.3 eps_j; visual
    token of window w: v = rho_w u + sqrt(1 - rho_w^2) xi, eps, xi ~ N(0, I/D);
    tail tokens (M mod S) draw rho like a window.
    """
    g = _gen(seed * 7 + 2, device)
    u = _randn((B, 1, D), g, device)
    u = u / u.norm(dim=-1, keepdim=True)
    txt = u + 0.3 * _randn((B, N, D), g, device) / math.sqrt(D)
    W = M // S
    rho = window_relevance(B, W + 1, seed, device)                 # +1: the tail
    rho_tok = rho.repeat_interleave(S, dim=1)[:, :M].unsqueeze(-1)
    xi = _randn((B, M, D), g, device) / math.sqrt(D)
    vis = rho_tok * u + torch.sqrt(1 - rho_tok ** 2) * xi
    return vis.half().contiguous(), txt.half().contiguous()


def _rope(x: torch.Tensor, pos0: int, theta: float = 1.0e6) -> torch.Tensor:
    """Qwen2 (NeoX half-rotation) rotary embedding of x[..., T, d] at positions pos0.."""
    T, d = x.shape[-2], x.shape[-1]
    half = d // 2
    inv = theta ** (-torch.arange(0, half, device=x.device, dtype=torch.float64) / half)
    pos = torch.arange(pos0, pos0 + T, device=x.device, dtype=torch.float64)
    ang = torch.outer(pos, inv)
    cos, sin = ang.cos().float(), ang.sin().float()
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def kv_layer(B: int, H: int, T: int, d: int, S: int, seed: int, layer: int, device="cpu",
             pos0: int = 0):
    """One layer's visual-span K, V [B][H][T][d] fp16 (K post-RoPE, as prefill stores it).

    K[t, c] = mu_c + sigma_c z (4 % outlier channels with |mu_c| ~ U(8, 20),
    sigma_c ~ U(0.3, 1.5)); window-0 keys carry a shared "sink" direction
    (Fig. first_window); then RoPE (theta 1e6).  V[t, c] = sigma_t z,
    sigma_t ~ LogNormal(0, 0.5).
    """
    g = _gen(seed * 1009 + 31 * layer + 3, device)
    mu = _randn((1, H, 1, d), g, device)
    out = _rand((1, H, 1, d), g, device) < 0.04
    sgn = torch.where(_rand((1, H, 1, d), g, device) < 0.5, -1.0, 1.0)
    mu = torch.where(out, sgn * (8 + 12 * _rand((1, H, 1, d), g, device)), mu)
    sig = 0.3 + 1.2 * _rand((1, H, 1, d), g, device)
    K = mu + sig * _randn((B, H, T, d), g, device)
    sink = sink_direction(H, d, seed, layer, device)
    K[:, :, :min(S, T), :] += 8.0 * sink.view(1, H, 1, d)
    K = _rope(K, pos0)
    sv = torch.exp(0.5 * _randn((B, H, T, 1), g, device))
    V = sv * _randn((B, H, T, d), g, device)
    return K.half().contiguous(), V.half().contiguous()


def sink_direction(H: int, d: int, seed: int, layer: int, device="cpu") -> torch.Tensor:
    g = _gen(seed * 1009 + 31 * layer + 5, device)
    s = _randn((H, d), g, device)
    return s / s.norm(dim=-1, keepdim=True)


def rest_layer(B: int, H: int, R_max: int, d: int, seed: int, layer: int, device="cpu"):
    """FP16 "rest" tokens (text + generated) for one layer: [B][H][R_max][d] each."""
    g = _gen(seed * 1009 + 31 * layer + 7, device)
    mu = _randn((1, H, 1, d), g, device)
    K = mu + _randn((B, H, R_max, d), g, device)
    V = torch.exp(0.5 * _randn((B, H, R_max, 1), g, device)) * _randn((B, H, R_max, d), g, device)
    return K.half().contiguous(), V.half().contiguous()


def queries(B: int, Hq: int, H: int, d: int, seed: int, layer: int, step: int = 0, device="cpu"):
    """Decode queries q[B][Hq][d] fp16: 0.5 N(0, I) plus a component along the
    kv head's sink direction so window-0 logits stand out (~+3)."""
    g = _gen(seed * 1009 + 31 * layer + 11 + 7919 * step, device)
    sink = sink_direction(H, d, seed, layer, device)                 # [H][d]
    grp = Hq // H
    q = 0.5 * _randn((B, Hq, d), g, device)
    q = q + 5.0 * sink.repeat_interleave(grp, dim=0).unsqueeze(0)
    return q.half().contiguous()


def layer_tensors(cfg, layer: int, device="cpu", B=None):
    """Everything one layer call needs: K, V (visual span, vis_off = 0), the
    rest buffers with the M mod S tail copied in front, and rest_len."""
    B = cfg.B if B is None else B
    m = cfg.model
    K, V = kv_layer(B, m.H, cfg.M, m.d, cfg.S, cfg.seed, layer, device)
    kr, vr = rest_layer(B, m.H, cfg.R_max, m.d, cfg.seed, layer, device)
    t = cfg.tail
    if t:
        kr[:, :, :t] = K[:, :, cfg.M - t:]
        vr[:, :, :t] = V[:, :, cfg.M - t:]
    rest_len = torch.full((B,), t + cfg.n_text, dtype=torch.int32, device=device)
    return K, V, kr, vr, rest_len


def text_queries(B: int, Hq: int, N: int, d: int, seed: int, layer: int, device="cpu"):
    """Query states of the N text tokens of one layer, [B][Hq][N][d] fp16 (the per-layer
    scorer's text side, include/wq.h wq_window_scores_layer): N(0, 1) plus a common
    per-request direction so that text and visual keys correlate like the embeddings."""
    g = _gen(seed * 1009 + 31 * layer + 13, device)
    u = _randn((B, 1, 1, d), g, device)
    return (0.7 * _randn((B, Hq, N, d), g, device) + u).half().contiguous()
