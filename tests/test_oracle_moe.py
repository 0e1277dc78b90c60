"""Pins for the oracle GEMMs and MoE block (not gpu).

Brute force on tiny shapes in exact rationals / int64 loops, library special cases
(all-16-bit block == torch fp64 SwiGLU MLP; silu == torch), and block properties
from SPEC S:147-172: linearity in w_e, duplicates 0.5/0.5 == one at 1.0, dead expert,
conservation Σ counts = T·k, top_k = E.
"""
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import bf16 as ob
from oracle.moe import (QBlock, expert_ffn, linear_block, moe_block, quantize_block, quantize_layer, route_prep,
                        silu, wa_int_accumulators)
from oracle.quant import quantize_act
from synth import configs as C
from synth.gen import bf16_bits_from_f32, gen_activations, gen_routing, gen_weight, weight_seed


def _rand_bf16(rng, shape, scale=1.0):
    return bf16_bits_from_f32((rng.standard_normal(shape) * scale).astype(np.float32))


def test_route_prep_bruteforce():
    rng = np.random.default_rng(0)
    T, k, E = 37, 3, 5
    ids = rng.integers(-1, E, (T, k))
    counts, offsets, perm, inv = route_prep(ids, E)
    assert counts.sum() == (ids >= 0).sum()
    # independent: sort routes by (expert, t, j) with Python's stable sort
    routes = sorted([(int(ids[t, j]), t, j) for t in range(T) for j in range(k) if ids[t, j] >= 0])
    assert perm.tolist() == [t * k + j for (_, t, j) in routes]
    for p, r in enumerate(perm):
        assert inv[r] == p
    assert np.all(inv[ids.reshape(-1) < 0] == -1)
    assert offsets.tolist() == [sum(counts[:e]) for e in range(E + 1)]


def test_route_prep_conservation_and_topk_e():
    T, E, k = 512, 8, 4
    ids, w = gen_routing(T, E, k, seed=3)
    counts, *_ = route_prep(ids, E)
    assert counts.sum() == T * k  # SPEC S:128 (conservation; "each token activating 4 experts")
    ids, _ = gen_routing(T, E, E, seed=4)
    counts, *_ = route_prep(ids, E)
    assert np.all(counts == T)  # top_k = E -> every expert sees every token
    with pytest.raises(ValueError):
        route_prep(np.array([[0, E]]), E)


def _bf16_round_exact(v: Fraction) -> Fraction:
    """Round a rational to the nearest bf16 value (8 significant bits), ties to even — exact arithmetic."""
    if v == 0:
        return v
    sgn = 1 if v > 0 else -1
    a = abs(v)
    e = 0
    while a >= 2:
        a /= 2
        e += 1
    while a < 1:
        a *= 2
        e -= 1
    m = a * 128  # in [128, 256)
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sgn * Fraction(fl) * Fraction(2) ** (e - 7)


def test_bf16_round_exact_helper():
    assert _bf16_round_exact(Fraction(257)) == 256 and _bf16_round_exact(Fraction(259)) == 260
    assert _bf16_round_exact(Fraction(-1, 3)) == Fraction(-171, 512)


@pytest.mark.parametrize("sch", [C.WO(4, 64), C.WO(2, 128), C.WO(3, -1, True), C.WO(8, 64)])
def test_wo_linear_bruteforce(sch):
    rng = np.random.default_rng(1)
    N, K, M = 3, 128, 2
    W = _rand_bf16(rng, (N, K), 0.1)
    X = ob.bits_to_f64(_rand_bf16(rng, (M, K)))
    blk = quantize_block(W, sch)
    y = linear_block(X, blk)
    y_exact = linear_block(X, blk, exact_weights=True)
    g = K if sch.w_group == -1 else sch.w_group
    for m in range(M):
        for n in range(N):
            acc, acc_x = Fraction(0), Fraction(0)
            for k in range(K):
                wq = int(blk.codes[n, k]) * Fraction(blk.scale[n, k // g])
                if blk.zero is not None:
                    wq += Fraction(blk.zero[n, k // g])
                acc += Fraction(X[m, k]) * _bf16_round_exact(wq)  # reading R5: bf16 dequantized weight
                acc_x += Fraction(X[m, k]) * wq                   # the exact dequantized weight
            assert abs(float(acc) - y[m, n]) <= 1e-12 * max(1.0, abs(float(acc)))
            assert abs(float(acc_x) - y_exact[m, n]) <= 1e-12 * max(1.0, abs(float(acc_x)))


@pytest.mark.parametrize("sch", [C.WA(8, -1), C.WA(4, 128), C.WA(5, 128), C.WA(4, -1)])
def test_wa_linear_bruteforce(sch):
    rng = np.random.default_rng(2)
    N, K, M = 3, 256, 2
    W = _rand_bf16(rng, (N, K), 0.1)
    Xb = _rand_bf16(rng, (M, K))
    X = ob.bits_to_f64(Xb)
    blk = quantize_block(W, sch)
    qa, sa, _ = quantize_act(X.astype(np.float32), sch.a_bits, sch.a_group)
    acc = wa_int_accumulators(qa, blk.codes, sch.w_group)
    g = K if sch.w_group == -1 else sch.w_group
    y = linear_block(X, blk)
    for m in range(M):
        for n in range(N):
            tot = Fraction(0)
            for gi in range(K // g):
                a = 0
                for k in range(gi * g, gi * g + g):
                    a += int(qa[m, k]) * int(blk.codes[n, k])  # int64 loop
                assert acc[gi, m, n] == a
                tot += Fraction(float(sa[m, gi])) * Fraction(blk.scale[n, gi]) * a
            assert abs(float(tot) - y[m, n]) <= 1e-12 * max(1.0, abs(float(tot)))


def test_int_acc_matches_torch_int_mm():
    """Independent library pin: torch._int_mm-style int32 GEMM (CPU int64 matmul) == fp64-BLAS acc."""
    rng = np.random.default_rng(9)
    qa = rng.integers(-127, 128, (16, 512))
    qw = rng.integers(-127, 128, (24, 512))
    acc = wa_int_accumulators(qa, qw, -1)[0]
    ref = (torch.from_numpy(qa) @ torch.from_numpy(qw).T).numpy()
    assert np.array_equal(acc.astype(np.int64), ref)


def test_silu_matches_torch():
    v = np.linspace(-30, 30, 1001)
    assert np.allclose(silu(v), torch.nn.functional.silu(torch.from_numpy(v)).numpy(), rtol=1e-14, atol=1e-300)


def test_w16_expert_is_dense_swiglu_mlp():
    """All-16-bit scheme (identity) == plain SwiGLU MLP with torch fp64."""
    rng = np.random.default_rng(4)
    d, f, T = 64, 128, 9
    Wg, Wu, Wd = _rand_bf16(rng, (f, d), 0.2), _rand_bf16(rng, (f, d), 0.2), _rand_bf16(rng, (d, f), 0.2)
    X = _rand_bf16(rng, (T, d))
    blks = [quantize_block(W, C.W16) for W in (Wg, Wu, Wd)]
    o = expert_ffn(ob.bits_to_f64(X), *blks)
    t = lambda b: torch.from_numpy(ob.bits_to_f64(b))
    x = t(X)
    h = torch.nn.functional.silu(x @ t(Wg).T) * (x @ t(Wu).T)
    h = h.to(torch.float32).to(torch.bfloat16).to(torch.float64)  # via fp32 (may double-round)
    ref = (h @ t(Wd).T).numpy()
    # bf16 rounding via fp32 can double-round; accept rare 1-ulp h differences through a tolerance
    assert np.max(np.abs(o - ref)) <= 1e-2 * np.max(np.abs(ref))


def _tiny_layer(table=None, cfg=C.get_config("tiny")):
    E, S = cfg.n_routed, cfg.n_shared
    W = []
    for e in range(E + S):
        f = cfg.inter if e < E else cfg.shared_inter
        W.append([gen_weight(f, cfg.hidden, weight_seed(e, 0)), gen_weight(f, cfg.hidden, weight_seed(e, 1)),
                  gen_weight(cfg.hidden, f, weight_seed(e, 2))])
    table = table or C.precision_table(cfg)
    return quantize_layer(W, table, E, S)


def test_block_properties():
    cfg = C.get_config("tiny")
    layer = _tiny_layer()
    T = 24
    x = gen_activations(T, cfg.hidden)
    ids, w = gen_routing(T, cfg.n_routed, cfg.top_k)
    y = moe_block(x, layer, ids, w)
    # linearity in w_e
    assert np.allclose(moe_block(x, layer, ids, 2 * w), 2 * y, rtol=1e-13, atol=1e-13)
    # duplicate expert with 0.5/0.5 == single route with weight 1.0
    ids1 = np.stack([ids[:, 0], ids[:, 0]], 1)
    y_dup = moe_block(x, layer, ids1, np.full((T, 2), 0.5, np.float32))
    y_one = moe_block(x, layer, np.stack([ids[:, 0], -np.ones(T, np.int32)], 1),
                      np.stack([np.ones(T, np.float32), np.zeros(T, np.float32)], 1))
    assert np.array_equal(y_dup, y_one)
    # dead expert: replace expert 3's weights; no token routes to 3 -> unchanged
    ids_no3 = np.where(ids == 3, -1, ids)
    y_a = moe_block(x, layer, ids_no3, w)
    layer.blocks[3] = _tiny_layer(C.uniform_table(cfg, C.WO(2, 64))).blocks[3]
    assert np.array_equal(moe_block(x, layer, ids_no3, w), y_a)
    # per-token independence: a subset of tokens gives the same rows
    sub = np.array([3, 7, 11])
    assert np.allclose(moe_block(x[sub], layer, ids[sub], w[sub]), moe_block(x, layer, ids, w)[sub], rtol=0, atol=0)


def test_quantized_close_to_unquantized_w8():
    """w8 weight-only output is near the bf16 output (quantization error small; sanity of scale/zero use)."""
    cfg = C.get_config("tiny")
    T = 16
    x = gen_activations(T, cfg.hidden)
    ids, w = gen_routing(T, cfg.n_routed, cfg.top_k)
    y16 = moe_block(x, _tiny_layer(C.uniform_table(cfg, C.W16)), ids, w)
    y8 = moe_block(x, _tiny_layer(C.uniform_table(cfg, C.WO(8, 64))), ids, w)
    y2 = moe_block(x, _tiny_layer(C.uniform_table(cfg, C.WO(2, 64))), ids, w)
    e8 = np.abs(y8 - y16).max() / np.abs(y16).max()
    e2 = np.abs(y2 - y16).max() / np.abs(y16).max()
    assert e8 < 0.02 and e2 > e8  # 2-bit weights perturb more


def test_table6_counts():
    """PAPER.md Table tab:w5a5-scheme: 61 rows, gate == up, a_gsize == w_gsize."""
    rows = C.parse_table6()
    assert len(rows) == 61
    flat = [b for r in rows for b in r]
    assert sum(1 for b in flat if (b.w_bits, b.w_group) == (4, 128)) == 128
    assert sum(1 for b in flat if (b.w_bits, b.w_group) == (8, -1)) == 37
    assert sum(1 for b in flat if (b.w_bits, b.w_group) == (4, -1)) == 18
    assert all(r[0] == r[1] for r in rows)
    assert all(b.a_group == b.w_group and b.a_bits == b.w_bits for b in flat)


def test_shared_experts_pin():
    """Shared-expert branch of moe_block pinned to an independent torch fp64 computation (reading R13): every token
    gets sum_j w[t,j] MLP_ids[t,j](x_t) + sum_s shared_w[t,s] MLP_shared_s(x_t), with S = 2 shared experts of their own
    width, non-uniform per-token shared weights, dead routes (-1) and a token with no routed expert at all."""
    rng = np.random.default_rng(11)
    E, S, d, f, fs, T, k = 3, 2, 64, 128, 192, 11, 2
    W = [[_rand_bf16(rng, (ff, d), 0.2), _rand_bf16(rng, (ff, d), 0.2), _rand_bf16(rng, (d, ff), 0.2)]
         for ff in [f] * E + [fs] * S]
    layer = quantize_layer(W, [[C.W16] * 3] * (E + S), E, S)
    assert layer.shared_inter == fs
    X = _rand_bf16(rng, (T, d))
    ids = rng.integers(-1, E, (T, k))
    ids[4] = -1
    w = rng.uniform(0.1, 1.0, (T, k)).astype(np.float32)
    sw = rng.uniform(-0.5, 1.5, (T, S)).astype(np.float32)
    y = moe_block(X, layer, ids, w, sw)

    t = lambda b: torch.from_numpy(ob.bits_to_f64(b))
    x = t(X)

    def mlp(v, xs):
        h = torch.nn.functional.silu(xs @ t(W[v][0]).T) * (xs @ t(W[v][1]).T)
        h = h.to(torch.float32).to(torch.bfloat16).to(torch.float64)
        return h @ t(W[v][2]).T

    ref = torch.zeros(T, d, dtype=torch.float64)
    for tt in range(T):
        for j in range(k):
            if ids[tt, j] >= 0:
                ref[tt] += float(w[tt, j]) * mlp(int(ids[tt, j]), x[tt:tt + 1])[0]
    for s in range(S):
        ref += torch.from_numpy(sw[:, s].astype(np.float64))[:, None] * mlp(E + s, x)
    ref = ref.numpy()
    assert np.max(np.abs(y - ref)) <= 1e-2 * np.max(np.abs(ref))
    # the token without routed experts is exactly its shared part; shared weights enter linearly per expert
    only_shared = moe_block(X[4:5], layer, ids[4:5], w[4:5], sw[4:5])
    assert np.allclose(only_shared[0], y[4], rtol=0, atol=0)
    sw2 = sw.copy()
    sw2[:, 1] *= 2.0
    y2 = moe_block(X, layer, ids, w, sw2)
    sw0 = sw.copy()
    sw0[:, 1] = 0.0
    y0 = moe_block(X, layer, ids, w, sw0)
    assert np.allclose(y2 - y, y - y0, rtol=1e-12, atol=1e-12)
    assert np.max(np.abs(y - y0)) > 1e-3  # shared expert 1 contributes
