"""bf16 helpers for the oracle (independent of synth/ and of the CUDA path).

bf16 = 1 sign, 8 exponent, 7 stored fraction bits: 8 significant bits.
Only normal, finite values are handled (DESIGN.md §2 reading R12).
"""
import numpy as np


def bits_to_f64(bits):
    """uint16 bf16 bit patterns -> float64 (exact)."""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)


def f64_to_bits(x):
    """float64 values that ARE bf16-representable -> uint16 bit patterns (asserts exactness)."""
    x = np.asarray(x, dtype=np.float64)
    f = x.astype(np.float32)
    assert np.array_equal(f.astype(np.float64), x), "value not representable in fp32"
    u = f.view(np.uint32)
    assert np.all((u & np.uint32(0xFFFF)) == 0), "value not representable in bf16"
    return (u >> np.uint32(16)).astype(np.uint16)


def bf16_round_f64(x):
    """Round float64 -> nearest bf16 value (ties to even), returned as float64.

    x = m * 2**e with 0.5 <= |m| < 1 (frexp); bf16 keeps 8 significant bits, so the
    result is rint(m * 2**8) * 2**(e - 8). A single rounding from fp64.
    """
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    return np.ldexp(np.rint(m * 256.0), e - 8)


def _sig_exp(s):
    """Positive bf16 value s = M * 2**E with integer M in [128, 256)."""
    m, e = np.frexp(s)
    return (m * 256.0), e - 8


def bf16_next_up(s):
    """Smallest bf16 strictly greater than positive bf16 value s."""
    M, E = _sig_exp(np.asarray(s, dtype=np.float64))
    return np.ldexp(M + 1.0, E)


def bf16_next_down(s):
    """Largest bf16 strictly smaller than positive bf16 value s."""
    M, E = _sig_exp(np.asarray(s, dtype=np.float64))
    return np.where(M == 128.0, np.ldexp(255.0, E - 1), np.ldexp(M - 1.0, E))
