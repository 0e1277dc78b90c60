"""Quantizers of the oracle.

Q  — weight quantizer: uniform min-max quantization x̂ = round((x − x_min)/Δ)·Δ + x_min
     (§2.1), group-wise along K ("to support group-size=128 ...
     tile_k=256 infeasible" — groups run along the reduction dim), scale and zero-point
     stored in 16 bits. Readings: round = half-to-even (R1);
     zero-point = x_min stored as bf16 (R2, R3); the stored scale is the SMALLEST bf16
     s with (2^b − 1)·s ≥ x_max − x_min (R4, "round-up"); codes are computed against
     the stored scale; symmetric: Δ = max|x| / (2^(b−1) − 1), codes ±(2^(b−1) − 1) (R6);
     degenerate (constant / all-zero) groups: s = 1, q = 0 (R7).
     Arithmetic: fp64 IEEE (x − z and division), then rint (half-to-even).
A  — activation quantizer, dynamic and symmetric ("Activations are dynamically
     quantized at runtime", "per-channel symmetric"), per token (a_group = −1) or
     per 128-group along K. fp32 arithmetic fixed by reading R9:
     r = fl32(qmax / amax), s_a = fl32(amax / qmax), q = clamp(rint(fl32(v·r)), ±qmax).
"""
from __future__ import annotations

import numpy as np

from .bf16 import bf16_next_down, bf16_next_up, bf16_round_f64, bits_to_f64


def _groups(K: int, g: int) -> int:
    g = K if g == -1 else g
    if g <= 0 or K % g != 0:
        raise ValueError(f"group size {g} does not divide K={K}")
    return g


def smallest_bf16_at_least(D: np.ndarray, c: int) -> np.ndarray:
    """Smallest bf16 value s > 0 with c·s >= D (D > 0), both sides exact in fp64 (R4)."""
    D = np.asarray(D, dtype=np.float64)
    s = bf16_round_f64(D / c)
    # step down while the predecessor still satisfies the inequality, then up while s fails it
    while True:
        p = bf16_next_down(s)
        m = c * p >= D
        if not m.any():
            break
        s = np.where(m, p, s)
    while True:
        m = c * s < D
        if not m.any():
            break
        s = np.where(m, bf16_next_up(s), s)
    return s


def quantize_weight(w_bits: np.ndarray, w_bits_width: int, group: int, symmetric: bool):
    """Q on a linear block W[N, K] (bf16 bit patterns).

    Returns (codes int64 [N, K], scale float64 [N, K/g] (bf16 values),
             zero float64 [N, K/g] (bf16 values) or None when symmetric).
    asym codes in [0, 2^b − 1]; sym codes in [−(2^(b−1) − 1), 2^(b−1) − 1].
    """
    x = bits_to_f64(w_bits)
    if not np.all(np.isfinite(x)):
        raise ValueError("non-finite weight")
    N, K = x.shape
    g = _groups(K, group)
    xg = x.reshape(N, K // g, g)
    b = w_bits_width
    if not symmetric:
        xmin = xg.min(axis=2)
        xmax = xg.max(axis=2)
        D = xmax - xmin  # exact: both bf16
        c = 2 ** b - 1
        degenerate = D == 0
        s = np.where(degenerate, 1.0, smallest_bf16_at_least(np.where(degenerate, 1.0, D), c))
        z = xmin
        q = np.rint((xg - z[:, :, None]) / s[:, :, None])
        q = np.clip(q, 0, c)
        return q.reshape(N, K).astype(np.int64), s, z
    qmax = 2 ** (b - 1) - 1
    a = np.abs(xg).max(axis=2)
    degenerate = a == 0
    s = np.where(degenerate, 1.0, smallest_bf16_at_least(np.where(degenerate, 1.0, a), qmax))
    q = np.rint(xg / s[:, :, None])
    q = np.clip(q, -qmax, qmax)
    return q.reshape(N, K).astype(np.int64), s, None


def dequantize_weight(codes: np.ndarray, scale: np.ndarray, zero, group: int) -> np.ndarray:
    """ŵ = q·s + z (asym) or q·s (sym), exact in fp64 (reading R5)."""
    N, K = codes.shape
    g = _groups(K, group)
    qg = codes.reshape(N, K // g, g).astype(np.float64)
    w = qg * scale[:, :, None]
    if zero is not None:
        w = w + zero[:, :, None]
    return w.reshape(N, K)


def storage_bits_per_weight(w_bits: int, group: int, symmetric: bool, K: int, meta_bits: int = 16) -> float:
    """w + (1 sym | 2 asym)·16/g, g = K for per-channel (3.25 / 2.25 for g128 asym)."""
    if w_bits == 16:
        return 16.0
    g = K if group == -1 else group
    return w_bits + (1 if symmetric else 2) * meta_bits / g


def quantize_act(v: np.ndarray, a_bits: int, a_group: int):
    """A on activations v[M, K] (bf16-valued floats). fp32 IEEE arithmetic (R9).

    Returns (codes int64 [M, K], scale float32 [M, K/ga], qsum int64 [M, K/ga]).
    """
    v = np.asarray(v, dtype=np.float32)
    M, K = v.shape
    g = _groups(K, a_group)
    vg = v.reshape(M, K // g, g)
    qmax = np.float32(2 ** (a_bits - 1) - 1)
    amax = np.abs(vg).max(axis=2)  # exact (max of bf16 magnitudes)
    zero = amax == 0
    safe = np.where(zero, np.float32(1), amax).astype(np.float32)
    r = (qmax / safe).astype(np.float32)  # fl32(qmax / amax)
    s = (safe / qmax).astype(np.float32)  # fl32(amax / qmax)
    prod = (vg * r[:, :, None]).astype(np.float32)  # fl32(v * r)
    q = np.clip(np.rint(prod), -qmax, qmax)
    q = np.where(zero[:, :, None], 0, q)
    s = np.where(zero, np.float32(1), s).astype(np.float32)
    q = q.reshape(M, K).astype(np.int64)
    return q, s, q.reshape(M, K // g, g).sum(axis=2)
