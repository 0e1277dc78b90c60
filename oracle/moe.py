"""MoE block of the oracle: route preparation, per-scheme linear blocks, expert FFN, block sum.

The block is computed the paper's "straightforward" way: "sequential
execution, where the summation in Eq. 2 is expanded, and each expert is processed
individually before aggregating the results". Expert e computes
W_down^e( σ(W_gate^e X_e) ⊙ W_up^e X_e ) (Eq. 1) with σ = SiLU (reading R15)
and the block output is F = Σ_e (...) ⊙ w_e (Eq. 2). Each linear block
applies its own scheme (per-linear-block allocation): weight-only schemes
multiply by the dequantized weights rounded once to bf16 (R5); weight-activation schemes quantize the
block input dynamically and accumulate exact integer products per group.
Intermediate h is rounded to bf16 (reading R16).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .bf16 import bf16_round_f64, bits_to_f64
from .fp8 import linear_block_fp8, quantize_weight_fp8
from .quant import dequantize_weight, quantize_act, quantize_weight


# ----------------------------------------------------------------------------- S1
def route_prep(topk_ids: np.ndarray, E: int):
    """Histogram, exclusive scan and stable (t, j)-ordered placement of the T·k routes.

    Returns counts[E], offsets[E+1], perm_src[R] (flat route index t*k+j at each sorted
    position), inv[T*k] (sorted position of route (t, j), −1 for id −1). Raises ValueError
    for ids outside [−1, E) (the GPU raises MXM_E_DATA and skips the route).
    """
    ids = np.asarray(topk_ids).reshape(-1)
    if np.any((ids < -1) | (ids >= E)):
        raise ValueError("expert id out of range")
    counts = np.zeros(E, dtype=np.int64)
    for e in ids:
        if e >= 0:
            counts[e] += 1
    offsets = np.zeros(E + 1, dtype=np.int64)
    for e in range(E):
        offsets[e + 1] = offsets[e] + counts[e]
    fill = offsets[:-1].copy()
    perm = np.zeros(int(offsets[-1]), dtype=np.int64)
    inv = np.full(ids.size, -1, dtype=np.int64)
    for r, e in enumerate(ids):  # (t, j) lexicographic order
        if e >= 0:
            perm[fill[e]] = r
            inv[r] = fill[e]
            fill[e] += 1
    return counts, offsets, perm, inv


# ----------------------------------------------------------------------------- blocks
@dataclass
class QBlock:
    """One quantized linear block W[N, K] in canonical form."""

    w_bits: int
    a_bits: int
    w_group: int
    a_group: int
    symmetric: bool
    codes: np.ndarray  # int64 [N,K]; w16: uint16 bf16 bits; FP8: e4m3 code bytes
    scale: Optional[np.ndarray]
    zero: Optional[np.ndarray]
    fmt: int = 0  # 1: FP8 e4m3 (oracle/fp8.py, readings R25/R26)

    @property
    def N(self):
        return self.codes.shape[0]

    @property
    def K(self):
        return self.codes.shape[1]


def quantize_block(w_bits_u16: np.ndarray, sch) -> QBlock:
    if sch.w_bits == 16:
        return QBlock(16, 16, -1, -1, True, np.asarray(w_bits_u16, dtype=np.uint16), None, None)
    if getattr(sch, "fmt", 0) == 1:
        codes, s = quantize_weight_fp8(w_bits_u16, sch.w_group)
        return QBlock(8, 8, sch.w_group, sch.a_group, True, codes.astype(np.int64), s, None, 1)
    codes, s, z = quantize_weight(w_bits_u16, sch.w_bits, sch.w_group, sch.symmetric)
    return QBlock(sch.w_bits, sch.a_bits, sch.w_group, sch.a_group, sch.symmetric, codes, s, z)


def dequantize_weight_bf16(blk: "QBlock") -> np.ndarray:
    """Weight-only dequantized operand: ŵ = bf16_rne(q·s + z), the exact value rounded once (reading R5).

    The north star fixes parity "on identical dequantized weights"; a bf16 tensor-core path
    multiplies bf16 operands, so the dequantized weight of a weight-only block is this bf16 value.
    """
    return bf16_round_f64(dequantize_weight(blk.codes, blk.scale, blk.zero, blk.w_group))


def wa_int_accumulators(qa: np.ndarray, qw: np.ndarray, group: int) -> np.ndarray:
    """acc[g, m, n] = Σ_{k ∈ group g} qa[m,k]·qw[n,k], exact integers (reading G).

    Computed with fp64 BLAS; exact because every partial sum is an integer < 2^53.
    """
    M, K = qa.shape
    g = K if group == -1 else group
    out = np.zeros((K // g, M, qw.shape[0]), dtype=np.float64)
    for gi in range(K // g):
        sl = slice(gi * g, gi * g + g)
        out[gi] = qa[:, sl].astype(np.float64) @ qw[:, sl].astype(np.float64).T
    return out


def linear_block(xin: np.ndarray, blk: QBlock, exact_weights: bool = False) -> np.ndarray:
    """y[m, n] for block input xin[m, K] (bf16-valued float64). fp64 result.

    exact_weights: weight-only blocks multiply by the exact dequantized ŵ = q·s + z of P:53 instead of its
    bf16 rounding (reading R5); used to check the GPU against the paper's exact dequantization too.
    """
    xin = np.asarray(xin, dtype=np.float64)
    if blk.w_bits == 16:
        return xin @ bits_to_f64(blk.codes).T
    if blk.a_bits == 16:  # weight-only: dequantized weights rounded once to bf16 (reading R5)
        if exact_weights:
            return xin @ dequantize_weight(blk.codes, blk.scale, blk.zero, blk.w_group).T
        return xin @ dequantize_weight_bf16(blk).T
    if blk.fmt == 1:
        return linear_block_fp8(xin, blk.codes, blk.scale, blk.w_group, blk.a_group)
    qa, sa, _ = quantize_act(xin.astype(np.float32), blk.a_bits, blk.a_group)
    acc = wa_int_accumulators(qa, blk.codes, blk.w_group)
    y = np.zeros((xin.shape[0], blk.N))
    for gi in range(acc.shape[0]):
        y += sa[:, gi].astype(np.float64)[:, None] * blk.scale[:, gi][None, :] * acc[gi]
    return y


def silu(v):
    return v / (1.0 + np.exp(-v))


def expert_ffn(xe: np.ndarray, gate: QBlock, up: QBlock, down: QBlock, return_h: bool = False,
               exact_weights: bool = False):
    """Eq. 1: W_down(σ(W_gate X) ⊙ W_up X), h rounded to bf16 (R16)."""
    g = linear_block(xe, gate, exact_weights)
    u = linear_block(xe, up, exact_weights)
    with np.errstate(over="ignore"):
        h = bf16_round_f64(silu(g) * u)
    o = linear_block(h, down, exact_weights)
    return (o, h) if return_h else o


@dataclass
class QuantizedLayer:
    n_routed: int
    n_shared: int
    hidden: int
    inter: int
    shared_inter: int
    blocks: List[List[QBlock]]  # [(n_routed + n_shared)][gate, up, down]


def quantize_layer(weights, table, n_routed: int, n_shared: int) -> QuantizedLayer:
    """weights[e][j] bf16 bits (gate/up [f, d], down [d, f]); table[e][j] Scheme."""
    blocks = []
    for e in range(n_routed + n_shared):
        blocks.append([quantize_block(weights[e][j], table[e][j]) for j in range(3)])
    d = blocks[0][0].K
    f = blocks[0][0].N
    fs = blocks[n_routed][0].N if n_shared else 0
    return QuantizedLayer(n_routed, n_shared, d, f, fs, blocks)


def moe_block(x_bits: np.ndarray, layer: QuantizedLayer, topk_ids: np.ndarray, topk_w: np.ndarray,
              shared_w: Optional[np.ndarray] = None, exact_weights: bool = False) -> np.ndarray:
    """F = Σ_e w_e ⊙ expert_e(X_e) (Eq. 2) + Σ_s shared_w[:, s] ⊙ shared_s(X); fp64 [T, d].

    Routes with id −1 are skipped; duplicate ids in a token are legal and each
    contributes (linearity in w_e).
    """
    x = bits_to_f64(x_bits)
    T = x.shape[0]
    ids = np.asarray(topk_ids)
    w = np.asarray(topk_w, dtype=np.float64)
    y = np.zeros((T, layer.hidden))
    for e in range(layer.n_routed):
        tt, jj = np.nonzero(ids == e)  # row-major: (t, j) order
        if tt.size == 0:
            continue
        o = expert_ffn(x[tt], *layer.blocks[e], exact_weights=exact_weights)
        for r in range(tt.size):
            y[tt[r]] += w[tt[r], jj[r]] * o[r]
    for s in range(layer.n_shared):
        o = expert_ffn(x, *layer.blocks[layer.n_routed + s], exact_weights=exact_weights)
        ws = np.ones(T) if shared_w is None else np.asarray(shared_w, dtype=np.float64)[:, s]
        y += ws[:, None] * o
    return y
