"""Pins for the oracle quantizers (not gpu).

Each test pins the oracle to something other than itself: hand-worked fixtures
(tests/golden/quant_fixtures.json, each cited), the closed-form round-trip bound
|x − ŵ| <= s/2 checked in exact rational arithmetic, brute force over all codes,
minimality of the stored scale, on-grid round trips and the paper's storage bits.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import bf16 as ob
from oracle.quant import quantize_act, quantize_weight, storage_bits_per_weight, dequantize_weight
from synth.gen import bf16_bits_from_f32


def _bits(vals):
    b = bf16_bits_from_f32(np.asarray(vals, dtype=np.float32))
    assert np.array_equal(ob.bits_to_f64(b), np.asarray(vals, dtype=np.float64)), "fixture not bf16-exact"
    return b


def _load(golden_dir):
    with open(os.path.join(golden_dir, "quant_fixtures.json")) as f:
        return json.load(f)


def test_weight_fixtures(golden_dir):
    fx = _load(golden_dir)["weight"]
    assert len(fx) >= 10
    for c in fx:
        x = _bits(c["x"])[None, :]
        q, s, z = quantize_weight(x, c["bits"], c["group"], c["sym"])
        assert q[0].tolist() == c["codes"], c["cite"]
        sc = c["scale"] if isinstance(c["scale"][0], list) else [c["scale"]]
        for gi, (num, den) in enumerate(sc):
            assert Fraction(s[0, gi]) == Fraction(num, den), c["cite"]
        if c["sym"]:
            assert z is None
        else:
            zz = c["zero"] if isinstance(c["zero"], list) else [c["zero"]]
            for gi, zv in enumerate(zz):
                assert z[0, gi] == zv, c["cite"]


def test_act_fixtures(golden_dir):
    for c in _load(golden_dir)["act"]:
        v = ob.bits_to_f64(_bits(c["v"]))[None, :].astype(np.float32)
        q, s, qs = quantize_act(v, c["bits"], -1)
        assert q[0].tolist() == c["codes"], c["cite"]
        num, den = c["scale_f32_of"]
        assert s[0, 0] == np.float32(np.float32(num) / np.float32(den)), c["cite"]
        assert qs[0, 0] == sum(c["codes"])


def _groups(rng, kind, n, g):
    if kind == "gauss":
        x = rng.standard_normal((n, g))
    elif kind == "narrow":
        x = 3.0 + 1e-3 * rng.standard_normal((n, g))
    elif kind == "heavy":
        x = rng.standard_t(2, (n, g))
    elif kind == "tiny":
        x = 1e-30 * rng.standard_normal((n, g))
    else:
        x = np.abs(rng.standard_normal((n, g))) + 5.0
    return bf16_bits_from_f32(x.astype(np.float32))


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("sym", [False, True])
def test_roundtrip_bound_exact(bits, sym):
    """|x − ŵ| <= s/2 in exact rationals, no clamping (DESIGN R4 round-up)."""
    rng = np.random.default_rng(bits * 10 + sym)
    for kind in ["gauss", "narrow", "heavy", "tiny", "offset"]:
        xb = _groups(rng, kind, 24, 16)
        q, s, z = quantize_weight(xb, bits, -1, sym)
        x = ob.bits_to_f64(xb)
        for r in range(x.shape[0]):
            S = Fraction(s[r, 0])
            Z = Fraction(0) if sym else Fraction(z[r, 0])
            for k in range(x.shape[1]):
                err = abs(Fraction(x[r, k]) - (int(q[r, k]) * S + Z))
                assert err <= S / 2, (kind, r, k)
            # minimality of the stored scale (smallest bf16 satisfying the range inequality)
            c = (2 ** bits - 1) if not sym else (2 ** (bits - 1) - 1)
            D = Fraction(x[r].max()) - Fraction(x[r].min()) if not sym else max(abs(Fraction(v)) for v in x[r])
            if D > 0:
                assert c * S >= D
                assert c * Fraction(float(ob.bf16_next_down(s[r, 0]))) < D


@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("sym", [False, True])
def test_bruteforce_codes(bits, sym):
    """Each code is the nearest grid point among ALL codes (ties -> even code)."""
    rng = np.random.default_rng(100 + bits)
    xb = _groups(rng, "gauss", 30, 8)
    q, s, z = quantize_weight(xb, bits, -1, sym)
    x = ob.bits_to_f64(xb)
    lo, hi = (0, 2 ** bits - 1) if not sym else (-(2 ** (bits - 1) - 1), 2 ** (bits - 1) - 1)
    for r in range(x.shape[0]):
        S = Fraction(s[r, 0])
        Z = Fraction(0) if sym else Fraction(z[r, 0])
        for k in range(x.shape[1]):
            X = Fraction(x[r, k])
            dists = {c: abs(X - (c * S + Z)) for c in range(lo, hi + 1)}
            best = min(dists.values())
            cands = sorted(c for c, dv in dists.items() if dv == best)
            exp = cands[0] if len(cands) == 1 else [c for c in cands if c % 2 == 0][0]
            assert int(q[r, k]) == exp


def test_on_grid_roundtrip_and_zero():
    # x = q * 2^-3 + 1 on the grid q = 0..15 (w4 asym): quantizer must recover q and x exactly
    qs = np.arange(16)
    x = qs * 0.125 + 1.0
    xb = _bits(x)[None, :]
    q, s, z = quantize_weight(xb, 4, -1, False)
    assert q[0].tolist() == qs.tolist() and s[0, 0] == 0.125 and z[0, 0] == 1.0
    assert np.array_equal(dequantize_weight(q, s, z, -1)[0], x)
    zb = _bits(np.zeros(8))[None, :]
    for sym in (False, True):
        q, s, z = quantize_weight(zb, 3, -1, sym)
        assert np.all(dequantize_weight(q, s, z, -1) == 0)


def test_groupwise_independent():
    rng = np.random.default_rng(5)
    xb = bf16_bits_from_f32(rng.standard_normal((4, 256)).astype(np.float32))
    q, s, z = quantize_weight(xb, 4, 64, False)
    for gi in range(4):
        q1, s1, z1 = quantize_weight(xb[:, gi * 64:(gi + 1) * 64], 4, -1, False)
        assert np.array_equal(q[:, gi * 64:(gi + 1) * 64], q1)
        assert np.array_equal(s[:, gi], s1[:, 0]) and np.array_equal(z[:, gi], z1[:, 0])


def test_group_must_divide():
    with pytest.raises(ValueError):
        quantize_weight(np.zeros((1, 100), dtype=np.uint16), 4, 64, False)


def test_storage_bits():
    # PAPER.md P:339 / Table 1: g128 asym 16-bit meta -> 3.25 and 2.25 bits; SPEC S:67 w4 pc sym
    assert storage_bits_per_weight(3, 128, False, 2048) == 3.25
    assert storage_bits_per_weight(2, 128, False, 2048) == 2.25
    assert storage_bits_per_weight(4, -1, True, 4096) == 4 + 16 / 4096
    assert storage_bits_per_weight(16, -1, True, 4096) == 16


@pytest.mark.parametrize("bits", [4, 5, 8])
@pytest.mark.parametrize("group", [-1, 128])
def test_act_bound(bits, group):
    """|v − q·s_a| <= s_a·(1/2 + 3·qmax·2^-24): rounding of r, s_a, v·r (derivation DESIGN §4.1)."""
    rng = np.random.default_rng(bits + group)
    vb = bf16_bits_from_f32(rng.standard_t(3, (16, 256)).astype(np.float32))
    v = ob.bits_to_f64(vb).astype(np.float32)
    q, s, qs = quantize_act(v, bits, group)
    g = 256 if group == -1 else group
    qmax = 2 ** (bits - 1) - 1
    assert np.abs(q).max() <= qmax
    for m in range(16):
        for k in range(256):
            sa = float(s[m, k // g])
            assert abs(float(v[m, k]) - int(q[m, k]) * sa) <= sa * (0.5 + 3 * qmax * 2.0 ** -24)
    assert np.array_equal(qs, q.reshape(16, 256 // g, g).sum(axis=2))


def test_act_zero_row():
    q, s, qs = quantize_act(np.zeros((2, 128), np.float32), 8, -1)
    assert np.all(q == 0) and np.all(s == 1) and np.all(qs == 0)


def test_bf16_round_matches_torch():
    """oracle bf16 RNE (from fp64) == torch's float32->bf16 for fp32-exact inputs."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal(10000).astype(np.float32) * np.float32(3.0)
    a[:5] = [1.00390625, 1.01171875, -1.00390625, 3.0, 0.0]  # exact ties
    ref = ob.bits_to_f64(bf16_bits_from_f32(a))
    got = ob.bf16_round_f64(a.astype(np.float64))
    assert np.array_equal(ref, got)
