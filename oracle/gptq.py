"""Offline weight preparation of the paper's method: randomized Hadamard incoherence processing + GPTQ.

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module; the
product path (libmxmoe.so: mxm_hadamard_rotate, mxm_gptq_*) never calls it.

PAPER.md P:206 (§4.2.3): "we apply randomized Hadamard transformations to model weights using the incoherence
processing used in QuaRot, then perform GPTQ-based quantization"; P:335 (§5.1, Calibration): "We disabled
online rotations"; "For weight quantization, MxMoE employs GPTQ". The paper restates neither algorithm, so the
readings below (R22-R24) fix them:

 R22 randomized Hadamard: Q = blockdiag_b(diag(sigma_b) H_128) / sqrt(128) over the hidden dimension d
     (128 = the quantization group; H_128 the Sylvester Hadamard matrix; sigma in {-1, +1}^d a random sign
     vector passed in as an input). Offline only (no online rotation): the residual stream is rotated,
     so a block's weights become W_gate Q, W_up Q (input side, K = d) and Q^T W_down (output side, N = d); the
     block then maps x Q to y Q. A rotation is exactly orthogonal (Q Q^T = I), so it changes no output.
 R23 GPTQ = Frantar et al. 2022, Algorithm 1, as its reference implementation runs it without act-order:
     H = 2 X^T X / n over n calibration rows X [n, K]; dead columns (H_jj = 0) get H_jj = 1 and W[:, j] = 0;
     damping H += lambda I with lambda = 0.01 mean(diag H); U = upper Cholesky factor of H^-1; columns
     quantized left to right in blocks of B = 128: inside a block each column's error (w - q) / U_jj is
     propagated to the block's later columns through row j of U, and after the block to all later columns
     (lazy batch update W[:, i2:] -= Err U[i1:i2, i2:]).
 R24 group parameters during GPTQ come from the current (error-updated) weights at each group's first column
     (per channel: from the initial weights), with the S0a quantizer (oracle.quant.quantize_weight, R2/R4/R6/R7)
     generalised to non-bf16 inputs: asymmetric zero = the largest bf16 <= x_min, scale = the smallest bf16 s
     with (2^b - 1) s >= x_max - zero; symmetric scale = the smallest bf16 s with (2^(b-1) - 1) s >= max|x|;
     codes clip(rint((x - zero) / s)) / clip(rint(x / s)). On bf16 inputs this is quantize_weight exactly.
All arithmetic fp64.
"""
from __future__ import annotations

import numpy as np

from .bf16 import bf16_next_down, bf16_round_f64
from .quant import smallest_bf16_at_least


def hadamard(n: int) -> np.ndarray:
    """Sylvester Hadamard matrix H_n (n a power of two): H_1 = [1], H_2m = [[H, H], [H, -H]]."""
    if n < 1 or n & (n - 1):
        raise ValueError("n must be a power of two")
    h = np.ones((1, 1))
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h


def random_rotation(signs: np.ndarray, block: int = 128) -> np.ndarray:
    """R22: Q = blockdiag_b(diag(sigma_b) H_block) / sqrt(block), sigma = signs (+-1) of length d."""
    d = signs.shape[0]
    if d % block:
        raise ValueError("d must be a multiple of the block")
    hb = hadamard(block) / np.sqrt(block)
    q = np.zeros((d, d))
    for b0 in range(0, d, block):
        q[b0:b0 + block, b0:b0 + block] = np.diag(signs[b0:b0 + block].astype(np.float64)) @ hb
    return q


def rotate_rows(x: np.ndarray, signs: np.ndarray, block: int = 128) -> np.ndarray:
    """x Q for Q = random_rotation(signs): per 128-block (x_b diag(sigma_b)) H_128, then one division by sqrt(128).

    Same product as x @ random_rotation(signs); the +-1 sums are exact in fp64 for bf16 inputs, so each output is
    the exact value rounded once (the matrix form rounds every product by the irrational 1/sqrt(128) first)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    h = hadamard(block)
    out = np.empty_like(x)
    for b0 in range(0, d, block):
        out[..., b0:b0 + block] = (x[..., b0:b0 + block] * signs[b0:b0 + block]) @ h
    return out / np.sqrt(block)


def rotate_expert(w_gate: np.ndarray, w_up: np.ndarray, w_down: np.ndarray, signs: np.ndarray):
    """R22: the rotated block maps x Q to y Q: W_gate Q, W_up Q (K = d side), Q^T W_down (N = d side)."""
    return rotate_rows(w_gate, signs), rotate_rows(w_up, signs), rotate_rows(w_down.T, signs).T


def gptq_hessian(x: np.ndarray) -> np.ndarray:
    """R23: H = 2 X^T X / n (X [n, K] calibration rows)."""
    x = np.asarray(x, dtype=np.float64)
    return 2.0 * (x.T @ x) / x.shape[0]


def _bf16_at_most(v: np.ndarray) -> np.ndarray:
    """Largest bf16 value <= v (elementwise)."""
    r = bf16_round_f64(v)
    return np.where(r > v, bf16_next_down(r), r)


def group_params(xg: np.ndarray, w_bits: int, symmetric: bool):
    """R24 on the columns of one group: xg [N, g] -> (scale [N], zero [N] or None)."""
    if symmetric:
        qmax = 2 ** (w_bits - 1) - 1
        a = np.abs(xg).max(axis=1)
        deg = a == 0
        s = np.where(deg, 1.0, smallest_bf16_at_least(np.where(deg, 1.0, a), qmax))
        return s, None
    c = 2 ** w_bits - 1
    z = _bf16_at_most(xg.min(axis=1))
    D = xg.max(axis=1) - z
    deg = D == 0
    s = np.where(deg, 1.0, smallest_bf16_at_least(np.where(deg, 1.0, D), c))
    return s, z


def quant_column(w: np.ndarray, s: np.ndarray, z, w_bits: int):
    """Codes of one column under its group's (s, z) and the dequantized value q s + z (fp64, R5's exact form)."""
    if z is None:
        qmax = 2 ** (w_bits - 1) - 1
        q = np.clip(np.rint(w / s), -qmax, qmax)
        return q, q * s
    c = 2 ** w_bits - 1
    q = np.clip(np.rint((w - z) / s), 0, c)
    return q, q * s + z


def gptq_prepare(h: np.ndarray, w: np.ndarray, percdamp: float = 0.01):
    """R23 set-up: dead columns, damping, U = upper Cholesky factor of H^-1. Returns (U, W with dead cols 0)."""
    h = np.array(h, dtype=np.float64)
    w = np.array(w, dtype=np.float64)
    dead = np.diag(h) == 0
    h[dead, dead] = 1.0
    w[:, dead] = 0.0
    h += percdamp * np.mean(np.diag(h)) * np.eye(h.shape[0])
    hinv = np.linalg.inv(h)
    u = np.linalg.cholesky(hinv).T  # upper: U^T U = H^-1
    return u, w


def gptq_quantize(w: np.ndarray, h: np.ndarray, w_bits: int, group: int, symmetric: bool, block: int = 128,
                  percdamp: float = 0.01):
    """R23/R24: GPTQ of W [N, K] (fp64 values, e.g. a rotated bf16 block) against the Hessian H [K, K].

    Returns (codes int64 [N, K], scale [N, K/g], zero [N, K/g] or None): the S0a canonical format.
    """
    u, w = gptq_prepare(h, w, percdamp)
    N, K = w.shape
    g = K if group == -1 else group
    if K % g:
        raise ValueError("group must divide K")
    codes = np.zeros((N, K), dtype=np.int64)
    scale = np.zeros((N, K // g))
    zero = None if symmetric else np.zeros((N, K // g))
    s = z = None
    for i1 in range(0, K, block):
        i2 = min(i1 + block, K)
        w1 = w[:, i1:i2].copy()
        err = np.zeros((N, i2 - i1))
        for i in range(i2 - i1):
            j = i1 + i
            if j % g == 0:  # group start: parameters from the current weights of the group's columns
                cur = np.concatenate([w1[:, i:], w[:, i2:]], axis=1)[:, :g]
                s, z = group_params(cur, w_bits, symmetric)
                scale[:, j // g] = s
                if zero is not None:
                    zero[:, j // g] = z
            q, deq = quant_column(w1[:, i], s, z, w_bits)
            codes[:, j] = q.astype(np.int64)
            e = (w1[:, i] - deq) / u[j, j]
            w1[:, i:] -= e[:, None] * u[j, j:i2][None, :]
            err[:, i] = e
        w[:, i2:] -= err @ u[i1:i2, i2:]
    return codes, scale, zero


def layer_loss(w: np.ndarray, w_hat: np.ndarray, h: np.ndarray) -> float:
    """tr((W - W_hat) H (W - W_hat)^T): the layer-output squared error GPTQ minimises (H = 2 X^T X / n)."""
    d = np.asarray(w, dtype=np.float64) - np.asarray(w_hat, dtype=np.float64)
    return float(np.einsum("ij,jk,ik->", d, h, d))
