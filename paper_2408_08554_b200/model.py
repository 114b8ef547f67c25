"""Model-level drop-in: the reference's toy LLaMA-style block
(toyblock.hpp:66-282) with every projection on the GPU engine.

As in the reference, normalisation, attention softmax, SiLU and the residual
adds stay in real (FP64) arithmetic on the host -- they are the hot path's
callers, not the hot path -- and are evaluated in the reference's own
operation order (sequential reductions, glibc exp via ``math.exp``, no FMA) so
that the activations reaching the engine are the reference's bit for bit.
Each projection is ``quant_linear`` (toyblock.hpp:196-223): balance pre-scale
x/s and w*s, per-token activation ReQuant and per-channel weight quantization
(``abq.quantize`` on the device, FP64-exact) and ``abq.quantized_linear``
(bit-plane GEMM + zero-point correction + FP64 dequant on the device).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Tuple

import numpy as np

from . import api

RMS_EPS = 1e-6  # toyblock.hpp:15
LAYERS = ("q_proj", "k_proj", "v_proj", "o_proj", "gate_proj", "up_proj", "down_proj")  # toyblock.hpp:18-25


@dataclasses.dataclass
class ToyBlock:
    """ToyBlock  toyblock.hpp:66-119 (weights stored out x in, FP64)."""
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    wgate: np.ndarray
    wup: np.ndarray
    wdown: np.ndarray
    heads: int = 4
    norm1_gain: Optional[np.ndarray] = None
    norm2_gain: Optional[np.ndarray] = None

    def __post_init__(self):
        if self.dim % self.heads != 0:
            raise api.ValueError("ToyBlock: dim must be divisible by heads")
        if self.norm1_gain is None:
            self.norm1_gain = np.ones(self.dim)
        if self.norm2_gain is None:
            self.norm2_gain = np.ones(self.dim)

    @property
    def dim(self) -> int:
        return self.wq.shape[0]

    @property
    def hidden(self) -> int:
        return self.wgate.shape[0]

    def weight(self, name: str) -> np.ndarray:
        return {"q_proj": self.wq, "k_proj": self.wk, "v_proj": self.wv, "o_proj": self.wo,
                "gate_proj": self.wgate, "up_proj": self.wup, "down_proj": self.wdown}[name]

    def init_params(self) -> "BlockQuantParams":
        """ToyBlock::init_params  toyblock.hpp:111-118."""
        return BlockQuantParams({n: LayerParams(np.ones(self.weight(n).shape[1])) for n in LAYERS},
                                np.ones(self.dim), np.zeros(self.hidden), 0)


@dataclasses.dataclass
class LayerParams:
    """LayerParams  toyblock.hpp:28-32."""
    s: np.ndarray
    alpha: float = 1.0
    beta: float = 1.0


@dataclasses.dataclass
class BlockQuantParams:
    """BlockQuantParams  toyblock.hpp:36-44 (compensation on down_proj, gated by gamma)."""
    layers: dict
    comp_a: np.ndarray
    comp_b: np.ndarray
    gamma: int = 0


@dataclasses.dataclass
class BlockSpecs:
    """BlockSpecs  toyblock.hpp:47-64."""
    act: api.QuantSpec
    weight: api.QuantSpec

    @staticmethod
    def make(bits_w: int, bits_a: int, weight_scheme: int = api.ASYMMETRIC) -> "BlockSpecs":
        return BlockSpecs(api.QuantSpec(bits=bits_a, scheme=api.ASYMMETRIC, granularity=api.PER_TOKEN),
                          api.QuantSpec(bits=bits_w, scheme=weight_scheme, granularity=api.PER_CHANNEL))

    def passthrough(self) -> bool:
        return self.act.passthrough() or self.weight.passthrough()


@dataclasses.dataclass
class TraceEvent:
    layer: str
    requant: bool = False
    bitpack: bool = False
    dequant: bool = False


@dataclasses.dataclass
class ForwardTrace:
    """ForwardTrace  toyblock.hpp:128-131."""
    attention: List[np.ndarray] = dataclasses.field(default_factory=list)
    events: List[TraceEvent] = dataclasses.field(default_factory=list)


# ---- real-arithmetic pieces, in the reference's operation order -------------
def _rmsnorm(x: np.ndarray, gain: np.ndarray) -> np.ndarray:
    """detail::rmsnorm  toyblock.hpp:135-144 (sequential sum of squares)."""
    msq = np.zeros(x.shape[0])
    for j in range(x.shape[1]):
        msq = msq + x[:, j] * x[:, j]
    inv = 1.0 / np.sqrt(msq / float(x.shape[1]) + RMS_EPS)
    return (x * inv[:, None]) * gain[None, :]


def _matmul_wt(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """detail::linear_fp = matmul(x, w^T)  core.hpp:72-81: out starts at 0.0 and
    accumulates a(i,k) * b(k,j) for k = 0, 1, ..."""
    out = np.zeros((x.shape[0], w.shape[0]))
    for k in range(x.shape[1]):
        out = out + x[:, k:k + 1] * w[None, :, k]
    return out


_exp = np.vectorize(math.exp, otypes=[np.float64])


def _silu(x: np.ndarray) -> np.ndarray:
    """detail::silu  toyblock.hpp:150-155."""
    return x / (1.0 + _exp(-x))


def _attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, heads: int) -> Tuple[List[np.ndarray], np.ndarray]:
    """detail::attention  toyblock.hpp:158-189."""
    tokens, dim = q.shape
    dh = dim // heads
    ctx = np.zeros((tokens, dim))
    probs = []
    for h in range(heads):
        sl = slice(h * dh, (h + 1) * dh)
        s = np.zeros((tokens, tokens))
        for d in range(dh):
            s = s + q[:, sl][:, d:d + 1] * k[:, sl][None, :, d]
        p = s / math.sqrt(float(dh))
        mx = np.maximum.reduce(np.concatenate([np.full((tokens, 1), -1e300), p], axis=1), axis=1)
        p = _exp(p - mx[:, None])
        tot = np.zeros(tokens)
        for j in range(tokens):
            tot = tot + p[:, j]
        p = p / tot[:, None]
        c = np.zeros((tokens, dh))
        for j in range(tokens):
            c = c + p[:, j:j + 1] * v[j:j + 1, sl]
        ctx[:, sl] = c
        probs.append(p)
    return probs, ctx


# ---- engine-path projection --------------------------------------------------
def quant_linear(x: np.ndarray, w: np.ndarray, specs: BlockSpecs, lp: LayerParams,
                 comp: Optional[Tuple[np.ndarray, np.ndarray]], name: str, trace: ForwardTrace) -> np.ndarray:
    """detail::quant_linear  toyblock.hpp:196-223 with quantize / quantized_linear
    on the device."""
    if specs.passthrough():
        return _matmul_wt(x, w)
    xs, ws = x, w
    if lp.s is not None and len(lp.s):
        if len(lp.s) != w.shape[1]:
            raise api.ShapeError("quant_linear: balance vector length")
        xs = x / lp.s[None, :]
        ws = w * lp.s[None, :]
    wspec = dataclasses.replace(specs.weight, alpha=lp.alpha, beta=lp.beta)
    qa = api.quantize(np.ascontiguousarray(xs), dataclasses.replace(specs.act))
    qw = api.quantize(np.ascontiguousarray(ws), wspec, comp)
    y = api.quantized_linear(qa, qw).cpu().numpy()
    trace.events.append(TraceEvent(name, True, True, True))
    return y


def forward_fp(block: ToyBlock, x: np.ndarray) -> Tuple[np.ndarray, ForwardTrace]:
    """forward_fp  toyblock.hpp:191-214 (no engine)."""
    if x.shape[1] != block.dim:
        raise api.ShapeError("forward_fp: input width must equal block dim")
    trace = ForwardTrace()
    h1 = _rmsnorm(x, block.norm1_gain)
    q, k, v = (_matmul_wt(h1, w) for w in (block.wq, block.wk, block.wv))
    trace.attention, ctx = _attention(q, k, v, block.heads)
    x2 = x + _matmul_wt(ctx, block.wo)
    h2 = _rmsnorm(x2, block.norm2_gain)
    act = _silu(_matmul_wt(h2, block.wgate)) * _matmul_wt(h2, block.wup)
    return x2 + _matmul_wt(act, block.wdown), trace


def forward_quant(block: ToyBlock, x: np.ndarray, specs: BlockSpecs,
                  params: BlockQuantParams) -> Tuple[np.ndarray, ForwardTrace]:
    """forward_quant  toyblock.hpp:245-282: every projection through the engine."""
    if x.shape[1] != block.dim:
        raise api.ShapeError("forward_quant: input width must equal block dim")
    trace = ForwardTrace()
    comp = (params.comp_a, params.comp_b) if params.gamma else None
    lp = params.layers
    h1 = _rmsnorm(x, block.norm1_gain)
    q = quant_linear(h1, block.wq, specs, lp["q_proj"], None, "q_proj", trace)
    k = quant_linear(h1, block.wk, specs, lp["k_proj"], None, "k_proj", trace)
    v = quant_linear(h1, block.wv, specs, lp["v_proj"], None, "v_proj", trace)
    trace.attention, ctx = _attention(q, k, v, block.heads)
    x2 = x + quant_linear(ctx, block.wo, specs, lp["o_proj"], None, "o_proj", trace)
    h2 = _rmsnorm(x2, block.norm2_gain)
    gate = quant_linear(h2, block.wgate, specs, lp["gate_proj"], None, "gate_proj", trace)
    up = quant_linear(h2, block.wup, specs, lp["up_proj"], None, "up_proj", trace)
    act = _silu(gate) * up
    down = quant_linear(act, block.wdown, specs, lp["down_proj"], comp, "down_proj", trace)
    return x2 + down, trace


def first_token_attention_share(trace: ForwardTrace) -> float:
    """first_token_attention_share  toyblock.hpp:285-295."""
    if not trace.attention:
        raise api.ValueError("first_token_attention_share: no attention maps")
    total, count = 0.0, 0
    for p in trace.attention:
        for i in range(p.shape[0]):
            total += p[i, 0]
            count += 1
    return total / float(count)


__all__ = ["ToyBlock", "LayerParams", "BlockQuantParams", "BlockSpecs", "TraceEvent", "ForwardTrace",
           "LAYERS", "quant_linear", "forward_fp", "forward_quant", "first_token_attention_share"]
