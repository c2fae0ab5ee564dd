"""Workload table (BASELINE.json ``configs``).

Model shapes: LLaVA-OneVision-0.5B = Qwen2-0.5B (L24, H2/Hq14, d64, D896) and
LLaVA-OneVision-7B = Qwen2-7B (L28, H4/Hq28, d128, D3584).  196 visual tokens per
frame (M = T x K, Eq.5).  N = 32 text tokens; 50 generated tokens
("we generate 50 tokens").  No method arithmetic lives here.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

SEED_BASE = 0x57514E54          # 'WQNT'
TOKENS_PER_FRAME = 196
N_TEXT = 32
N_GEN = 50


@dataclass(frozen=True)
class Model:
    name: str
    L: int
    H: int
    Hq: int
    d: int
    D: int


QWEN2_05B = Model("llava-ov-0.5b", 24, 2, 14, 64, 896)
QWEN2_7B = Model("llava-ov-7b", 28, 4, 28, 128, 3584)


@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    model: Model
    layers: int            # layers exercised (C1: a single layer)
    B: int
    frames: int
    S: int
    widths: tuple
    budget: float = 0.0    # average-bit budget (<= 0: none)
    s_profile: tuple = field(default=())   # per-layer sensitivity s_l; () = 0.5 everywhere
    alpha: float = 2.0
    n_text: int = N_TEXT
    n_gen: int = N_GEN

    @property
    def M(self) -> int:
        return self.frames * TOKENS_PER_FRAME

    @property
    def W(self) -> int:
        return self.M // self.S

    @property
    def tail(self) -> int:
        return self.M % self.S

    @property
    def R_max(self) -> int:
        return self.tail + self.n_text + self.n_gen

    @property
    def seed(self) -> int:
        return SEED_BASE + self.idx

    def sensitivities(self) -> list:
        if self.s_profile:
            return list(self.s_profile)
        return [0.5] * self.layers

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


_C2_S = tuple([0.5] * 20 + [0.3, 0.2, 0.1, 0.05])

CONFIGS = {
    "C1": Config(1, "C1-0.5b-1layer-8f", QWEN2_05B, 1, 1, 8, 64, (2, 4, 8)),
    "C2": Config(2, "C2-0.5b-32f-b8-budget4", QWEN2_05B, 24, 8, 32, 32, (2, 4, 8, 16), budget=4.0,
                 s_profile=_C2_S),
    "C3": Config(3, "C3-7b-64f-b16", QWEN2_7B, 28, 16, 64, 32, (2, 4, 8, 16)),
    "C4": Config(4, "C4-7b-60f-b64-S32", QWEN2_7B, 28, 64, 60, 32, (2, 4, 8, 16)),
    "C5": Config(5, "C5-7b-256f-b4-longvideo", QWEN2_7B, 28, 4, 256, 32, (2, 4, 8, 16)),
}


def c4(S: int) -> Config:
    """C4 window-size sweep member (S = 16/32/64/128)."""
    return CONFIGS["C4"].with_(S=S, name=f"C4-7b-60f-b64-S{S}")
