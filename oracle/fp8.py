"""FP8 (e4m3) scheme of the oracle (NEXT-4 "FP8 ... as extra hardware-supported schemes S"; the
paper's scheme set S is "hardware-supported" quantization schemes, and B200 multiplies e4m3 natively).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module.

Readings (R25, R26):
 R25 e4m3 = OCP FP8 E4M3 (bias 7, no infinities, S.1111.111 = NaN, max finite 448, subnormals m 2^-9). Weights:
     per (row, group) scale s = the smallest bf16 with 448 s >= max|w| (the R4 round-up rule, so no code
     saturates); code = w / s (fp64) rounded to the nearest e4m3 value, ties to the even mantissa; max|w| = 0 ->
     s = 1, codes 0.
 R26 activations, dynamic per token (or per 128-group), R9's arithmetic with qmax = 448: amax = max|v| (fp32),
     r = fl32(448 / amax), s_a = fl32(amax / 448), code = e4m3_rn(min(max(fl32(v r), -448), 448)); amax = 0 ->
     s_a = 1, codes 0. The block output is s_w s_a sum_k q_w q_a over the e4m3 values (exact in fp64).
"""
from __future__ import annotations

import numpy as np

from .bf16 import bits_to_f64
from .quant import _groups, smallest_bf16_at_least

E4M3_MAX = 448.0


def e4m3_value(code: int) -> float:
    """The real value of an e4m3 byte by definition (R25): (-1)^s 2^(e-7) (1 + m/8), e = 0: (-1)^s 2^-6 m/8."""
    s, e, m = (code >> 7) & 1, (code >> 3) & 0xF, code & 7
    if e == 0xF and m == 7:
        return float("nan")
    v = (m / 8.0) * 2.0 ** -6 if e == 0 else (1.0 + m / 8.0) * 2.0 ** (e - 7)
    return -v if s else v


_POS = np.array([e4m3_value(c) for c in range(0x7F)])  # codes 0x00..0x7E: increasing non-negative values


def e4m3_round(x: np.ndarray) -> np.ndarray:
    """Nearest e4m3 value (ties to the even code, i.e. even mantissa), |x| <= 448 (callers clamp / pre-scale).

    Returns the e4m3 byte codes (uint8)."""
    x = np.asarray(x, dtype=np.float64)
    a = np.abs(x)
    if (a > E4M3_MAX).any():
        raise ValueError("value outside the e4m3 range")
    hi = np.searchsorted(_POS, a, side="left")  # first value >= a
    hi = np.minimum(hi, len(_POS) - 1)
    lo = np.maximum(hi - 1, 0)
    dlo, dhi = a - _POS[lo], _POS[hi] - a
    pick_hi = (dhi < dlo) | ((dhi == dlo) & (hi % 2 == 0))
    code = np.where(pick_hi, hi, lo)
    code = np.where(a == _POS[hi], hi, code)
    sign = np.signbit(x).astype(np.int64) << 7  # the sign survives rounding to zero (-0 = 0x80), as in hardware
    return (code | sign).astype(np.uint8)


def e4m3_decode(codes: np.ndarray) -> np.ndarray:
    c = np.asarray(codes, dtype=np.int64)
    v = _POS[np.minimum(c & 0x7F, 0x7E)]
    return np.where(c & 0x80, -v, v)


def quantize_weight_fp8(w_bits: np.ndarray, group: int):
    """R25 on W[N, K] (bf16 bits): (codes uint8 [N, K], scale float64 [N, K/g] (bf16 values))."""
    x = bits_to_f64(w_bits)
    N, K = x.shape
    g = _groups(K, group)
    xg = x.reshape(N, K // g, g)
    a = np.abs(xg).max(axis=2)
    deg = a == 0
    s = np.where(deg, 1.0, smallest_bf16_at_least(np.where(deg, 1.0, a), 448))
    codes = e4m3_round(xg / s[:, :, None]).reshape(N, K)
    return codes, s


def quantize_act_fp8(v: np.ndarray, a_group: int):
    """R26 on v[M, K] (fp32-representable): (codes uint8 [M, K], s_a float32 [M, K/g])."""
    v = np.asarray(v, dtype=np.float32)
    M, K = v.shape
    g = _groups(K, a_group)
    vg = v.reshape(M, K // g, g)
    amax = np.abs(vg).max(axis=2)
    deg = amax == 0
    with np.errstate(divide="ignore"):
        r = np.where(deg, np.float32(0), np.float32(E4M3_MAX) / amax).astype(np.float32)
        s = np.where(deg, np.float32(1), amax / np.float32(E4M3_MAX)).astype(np.float32)
    p = (vg * r[:, :, None]).astype(np.float32)
    p = np.clip(p, -E4M3_MAX, E4M3_MAX)
    return e4m3_round(p.astype(np.float64)).reshape(M, K), s


def linear_block_fp8(xin: np.ndarray, codes_w: np.ndarray, scale_w: np.ndarray, w_group: int, a_group: int):
    """y[m, n] = sum_g s_a[m, g] s_w[n, g] sum_{k in g} q_a q_w (e4m3 values; fp64, exact products and sums)."""
    qa, sa = quantize_act_fp8(np.asarray(xin, dtype=np.float32), a_group)
    va, vw = e4m3_decode(qa), e4m3_decode(codes_w)
    K = va.shape[1]
    g = _groups(K, w_group)
    y = np.zeros((va.shape[0], vw.shape[0]))
    for gi in range(K // g):
        sl = slice(gi * g, gi * g + g)
        acc = va[:, sl] @ vw[:, sl].T
        sa_g = sa[:, 0 if sa.shape[1] == 1 else gi].astype(np.float64)
        y += sa_g[:, None] * scale_w[:, gi][None, :] * acc
    return y
