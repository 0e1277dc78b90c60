"""Pins of oracle/gptq.py (randomized Hadamard incoherence processing + GPTQ; DESIGN R22-R24)
against things other than itself: Hadamard algebra, exact orthogonality, the rotated block's equivalence computed by
an independent torch fp64 SwiGLU MLP, the S0a quantizer (already pinned) on bf16 inputs, RTN on a diagonal Hessian,
and an independent fixed-order OBQ (inverse-Hessian downdating, no Cholesky) that GPTQ must reproduce code for code.
"""
import numpy as np
import pytest
import torch

from oracle.bf16 import bf16_next_down, bf16_next_up, bf16_round_f64, bits_to_f64, f64_to_bits
from oracle.gptq import (gptq_hessian, gptq_prepare, gptq_quantize, group_params, hadamard, layer_loss,
                         quant_column, random_rotation, rotate_expert)
from oracle.quant import dequantize_weight, quantize_weight


def test_hadamard_small_and_orthogonal():
    assert np.array_equal(hadamard(2), np.array([[1, 1], [1, -1]]))
    assert np.array_equal(hadamard(4), np.array([[1, 1, 1, 1], [1, -1, 1, -1], [1, 1, -1, -1], [1, -1, -1, 1]]))
    h = hadamard(128)
    assert set(np.unique(h)) == {-1.0, 1.0}
    assert np.array_equal(h @ h.T, 128 * np.eye(128))  # exact in fp64 (integer entries)
    with pytest.raises(ValueError):
        hadamard(96)


def test_random_rotation_orthogonal_blockdiag():
    rng = np.random.default_rng(0)
    d = 384
    sig = rng.choice([-1, 1], size=d)
    q = random_rotation(sig)
    assert np.abs(q @ q.T - np.eye(d)).max() < 1e-14
    for b0 in range(0, d, 128):
        blk = q[b0:b0 + 128, b0:b0 + 128]
        assert np.allclose(np.abs(blk), 1 / np.sqrt(128), atol=1e-15)
        off = q[b0:b0 + 128, :].copy()
        off[:, b0:b0 + 128] = 0
        assert not off.any()
    # row r of block b is sigma_r times row r of H / sqrt(128)
    assert np.allclose(q[5, :128], sig[5] * hadamard(128)[5] / np.sqrt(128))


def test_rotated_block_equivalence_torch_mlp():
    """x Q through the rotated weights equals (the original block on x) Q: an independent torch fp64 SwiGLU MLP."""
    rng = np.random.default_rng(1)
    d, f, T = 256, 192, 7
    wg, wu, wd = rng.standard_normal((f, d)), rng.standard_normal((f, d)), rng.standard_normal((d, f))
    x = rng.standard_normal((T, d))
    q = random_rotation(rng.choice([-1, 1], size=d))
    assert np.all(np.abs(q[np.arange(d), np.arange(d) // 128 * 128]) > 0)

    def mlp(xx, g, u, dn):
        xt = torch.tensor(xx, dtype=torch.float64)
        h = torch.nn.functional.silu(xt @ torch.tensor(g).T) * (xt @ torch.tensor(u).T)
        return (h @ torch.tensor(dn).T).numpy()

    y = mlp(x, wg, wu, wd)
    sig = np.sign(q[np.arange(d), np.arange(d) // 128 * 128])  # sigma_r = sign of row r's first block entry
    rg, ru, rd = rotate_expert(wg, wu, wd, sig)
    assert np.abs(rg - wg @ q).max() < 1e-13 and np.abs(rd - q.T @ wd).max() < 1e-13  # = the matrix form
    yr = mlp(x @ q, rg, ru, rd)
    assert np.abs(yr - y @ q).max() < 1e-10 * np.abs(y).max()


def _bf16_weights(rng, N, K, scale=0.05):
    return f64_to_bits(bf16_round_f64(rng.standard_normal((N, K)) * scale))


@pytest.mark.parametrize("bits,sym", [(2, False), (3, False), (4, False), (4, True), (8, True)])
def test_group_params_equal_s0a_on_bf16(bits, sym):
    """R24 on bf16 inputs is the S0a quantizer (pinned in test_oracle_quant.py)."""
    rng = np.random.default_rng(bits + 10 * sym)
    wb = _bf16_weights(rng, 16, 128)
    codes, s, z = quantize_weight(wb, bits, 128, sym)
    s2, z2 = group_params(bits_to_f64(wb), bits, sym)
    assert np.array_equal(s2, s[:, 0])
    if not sym:
        assert np.array_equal(z2, z[:, 0])
    for j in range(128):
        q, _ = quant_column(bits_to_f64(wb)[:, j], s2, z2, bits)
        assert np.array_equal(q.astype(np.int64), codes[:, j])


@pytest.mark.parametrize("bits,sym", [(2, False), (4, False), (4, True)])
def test_group_params_non_bf16_bounds(bits, sym):
    """Non-bf16 inputs: bf16 zero <= x_min with no bf16 in between, minimal bf16 scale, no clamping,
    |x - (q s + z)| <= s / 2 exactly."""
    rng = np.random.default_rng(3 + bits)
    x = rng.standard_normal((32, 64)) * 0.03 + 0.001
    s, z = group_params(x, bits, sym)
    assert np.array_equal(bf16_round_f64(s), s)
    if sym:
        qmax = 2 ** (bits - 1) - 1
        a = np.abs(x).max(axis=1)
        assert (qmax * s >= a).all() and (qmax * bf16_next_down(s) < a).all()
        q = np.rint(x / s[:, None])
        assert (np.abs(q) <= qmax).all()
    else:
        c = 2 ** bits - 1
        assert np.array_equal(bf16_round_f64(z), z)
        assert (z <= x.min(axis=1)).all() and (bf16_next_up(z) > x.min(axis=1)).all()
        D = x.max(axis=1) - z
        assert (c * s >= D).all() and (c * bf16_next_down(s) < D).all()
        q = np.rint((x - z[:, None]) / s[:, None])
        assert (q >= 0).all() and (q <= c).all()
    for j in range(64):
        _, deq = quant_column(x[:, j], s, z, bits)
        assert (np.abs(x[:, j] - deq) <= s / 2 + 1e-18).all()


@pytest.mark.parametrize("bits,group,sym", [(4, 128, False), (3, -1, False), (4, -1, True), (2, 128, False)])
def test_gptq_diagonal_hessian_is_rtn(bits, group, sym):
    """H diagonal -> U diagonal -> no error propagation: GPTQ = round-to-nearest S0a on the same bf16 weights."""
    rng = np.random.default_rng(bits)
    N, K = 24, 256
    wb = _bf16_weights(rng, N, K)
    h = np.diag(rng.uniform(0.5, 2.0, K))
    codes, s, z = gptq_quantize(bits_to_f64(wb), h, bits, group, sym)
    c0, s0, z0 = quantize_weight(wb, bits, group, sym)
    assert np.array_equal(codes, c0) and np.array_equal(s, s0)
    if not sym:
        assert np.array_equal(z, z0)


def _obq_fixed_order(w, h, bits, group, sym, percdamp=0.01):
    """Independent reference: optimal brain quantization in fixed column order with explicit inverse-Hessian
    downdating (Frantar & Alistarh 2022), which GPTQ's Cholesky form reproduces. Group parameters at each group
    start from the current weights (R24, via the pinned group_params)."""
    w = np.array(w, dtype=np.float64)
    h = np.array(h, dtype=np.float64)
    dead = np.diag(h) == 0
    h[dead, dead] = 1
    w[:, dead] = 0
    h += percdamp * np.mean(np.diag(h)) * np.eye(h.shape[0])
    hinv = np.linalg.inv(h)
    N, K = w.shape
    g = K if group == -1 else group
    codes = np.zeros((N, K), dtype=np.int64)
    for j in range(K):
        if j % g == 0:
            s, z = group_params(w[:, j:j + g], bits, sym)
        q, deq = quant_column(w[:, j], s, z, bits)
        codes[:, j] = q
        e = w[:, j] - deq
        w[:, j:] -= np.outer(e / hinv[j, j], hinv[j, j:])
        hinv[j:, j:] -= np.outer(hinv[j:, j], hinv[j, j:]) / hinv[j, j]
    return codes


@pytest.mark.parametrize("bits,group,sym,block", [(4, 8, False, 4), (3, -1, False, 8), (4, 16, True, 16),
                                                   (2, 8, False, 32)])
def test_gptq_equals_fixed_order_obq(bits, group, sym, block):
    rng = np.random.default_rng(7 * bits + block)
    N, K, n = 12, 32, 200
    mix = rng.standard_normal((K, K)) * 0.4 + np.eye(K)  # correlated calibration features
    x = rng.standard_normal((n, K)) @ mix
    h = gptq_hessian(x)
    w = bits_to_f64(_bf16_weights(rng, N, K, 0.1))
    codes, _, _ = gptq_quantize(w, h, bits, group, sym, block=block)
    assert np.array_equal(codes, _obq_fixed_order(w, h, bits, group, sym))


def test_gptq_hessian_and_dead_columns():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((50, 16))
    x[:, 3] = 0
    h = gptq_hessian(x)
    assert np.allclose(h, 2 * sum(np.outer(r, r) for r in x) / 50)
    u, w = gptq_prepare(h, np.ones((4, 16)))
    assert not w[:, 3].any() and w[:, 2].all()
    hd = h.copy()
    hd[3, 3] = 1
    hd += 0.01 * np.mean(np.diag(hd)) * np.eye(16)
    assert np.allclose(u.T @ u, np.linalg.inv(hd)) and np.allclose(u, np.triu(u))


def test_gptq_lowers_layer_loss_vs_rtn():
    """Seeded correlated calibration data: GPTQ's layer-output error below round-to-nearest's (P:206's reason)."""
    rng = np.random.default_rng(11)
    N, K, n = 64, 256, 1024
    mix = rng.standard_normal((K, K)) * 0.3 + np.eye(K)
    x = rng.standard_normal((n, K)) @ mix
    h = gptq_hessian(x)
    wb = _bf16_weights(rng, N, K)
    w = bits_to_f64(wb)
    for bits, group in ((3, 128), (4, 128), (2, -1)):
        c, s, z = gptq_quantize(w, h, bits, group, False)
        c0, s0, z0 = quantize_weight(wb, bits, group, False)
        lg = layer_loss(w, dequantize_weight(c, s, z, group), h)
        lr = layer_loss(w, dequantize_weight(c0, s0, z0, group), h)
        assert lg < 0.8 * lr, (bits, group, lg, lr)
