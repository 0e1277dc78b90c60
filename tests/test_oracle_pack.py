"""Pins for the oracle's packed layout (docs/packed_format.md) (not gpu).

Hand-computed words for known code patterns, the swizzle position of a known
element, invertibility, and size == the paper's storage bits.
"""
import numpy as np
import pytest

from oracle.pack import pack_block, packed_size, unpack_block
from oracle.quant import storage_bits_per_weight
from oracle.bf16 import f64_to_bits


SCHEMES = [  # (w_bits, a_bits, group, sym)
    (2, 16, 128, False), (2, 16, -1, False), (3, 16, 128, False), (3, 16, 64, True), (4, 16, 128, False),
    (4, 16, 64, False), (4, 16, -1, True), (8, 16, 128, False), (8, 16, -1, True),
    (4, 4, 128, True), (4, 4, -1, True), (5, 5, 128, True), (5, 5, -1, True), (8, 8, -1, True), (8, 8, 128, True),
]


def _rand_codes(rng, w, a, g, sym, N, K):
    if sym or a != 16:
        q = 2 ** (w - 1) - 1
        codes = rng.integers(-q, q + 1, (N, K))
    else:
        codes = rng.integers(0, 2 ** w, (N, K))
    G = K // (K if g == -1 else g)
    scale = np.ldexp(rng.integers(128, 256, (N, G)).astype(np.float64), -12)
    zero = None if (sym or a != 16) else np.ldexp(rng.integers(-255, 256, (N, G)).astype(np.float64), -8)
    return codes, scale, zero


@pytest.mark.parametrize("sch", SCHEMES)
def test_roundtrip(sch):
    w, a, g, sym = sch
    rng = np.random.default_rng(w * 100 + a + (g if g > 0 else 7))
    N, K = 256, 256
    codes, scale, zero = _rand_codes(rng, w, a, g, sym, N, K)
    p = pack_block(codes, scale, zero, w, a, g, sym)
    assert p.size == packed_size(w, a, g, sym, N, K)
    c2, s2, z2 = unpack_block(p, w, a, g, sym, N, K)
    assert np.array_equal(c2, codes)
    assert np.array_equal(s2, scale)
    if zero is not None:
        assert np.array_equal(z2, zero)


@pytest.mark.parametrize("sch", SCHEMES)
def test_size_equals_storage_bits(sch):
    """packed bytes * 8 / (N K) == w + meta*16/g (w8a8 image = 8 bits + meta)."""
    w, a, g, sym = sch
    N, K = 256, 1024
    bits = packed_size(w, a, g, sym, N, K) * 8 / (N * K)
    assert bits == storage_bits_per_weight(w, g, sym or a != 16, K)


def test_w4_weight_only_word_hand():
    """Row 0 elements 0..7 = codes 0..7: field f(i)=(i>>1)+4(i&1) -> nibbles 0,2,4,6,1,3,5,7 = 0x75316420."""
    N, K = 128, 64
    codes = np.tile(np.arange(64) % 16, (N, 1))
    scale = np.full((N, 1), 1.0)
    zero = np.zeros((N, 1))
    p = pack_block(codes, scale, zero, 4, 16, -1, False)
    meta = 512
    w0 = int(p[meta:meta + 4].view("<u4")[0])
    assert w0 == 0x75316420
    # word 1 of row 0 (elements 8..15 = codes 8..15) sits at u32 index 1*128 + 0
    w1 = int(p[meta + 128 * 4: meta + 128 * 4 + 4].view("<u4")[0])
    assert w1 == 0xFDB9ECA8
    # scale of row 5 in the meta block
    assert int(p[10:12].view("<u2")[0]) == int(f64_to_bits(np.array([1.0]))[0])


def test_w4a4_word_hand():
    """q = i+1-8 -> u = i+1; I8 nibble order gives nibbles (n7..n0) = 8,4,7,3,6,2,5,1."""
    N, K = 128, 128
    row = (np.arange(128) % 8) + 1 - 8
    codes = np.tile(row, (N, 1))
    p = pack_block(codes, np.ones((N, 1)), None, 4, 4, -1, True)
    assert int(p[0:4].view("<u4")[0]) == 0x84736251


def test_w2_word_hand():
    """w2 asym, codes of row 0 = 0,1,2,3,0,1,2,3,...: evens (0,2,0,2..) in fields 0-7, odds (1,3..) in 8-15."""
    N, K = 128, 64
    codes = np.tile(np.arange(64) % 4, (N, 1))
    p = pack_block(codes, np.ones((N, 1)), np.zeros((N, 1)), 2, 16, -1, False)
    w0 = int(p[512:516].view("<u4")[0])
    evens = sum(((2 * t) % 4) << (2 * t) for t in range(8))
    odds = sum(((2 * t + 1) % 4) << (2 * (8 + t)) for t in range(8))
    assert w0 == evens | odds


def test_image_swizzle_hand():
    """w16 image: element (row 1, k 0) bytes live at 1*128 + ((0 ^ 1) << 4) = 144."""
    N, K = 128, 64
    codes = np.zeros((N, K), dtype=np.uint16)
    codes[1, 0] = 0x3F80  # bf16 1.0
    codes[9, 17] = 0x4000  # row 9 (r&7=1), byte 34 -> chunk 2 -> (2^1)=3 -> 9*128+48+2
    p = pack_block(codes, None, None, 16, 16, -1, True)
    assert int(p[144:146].view("<u2")[0]) == 0x3F80
    assert int(p[9 * 128 + 48 + 2: 9 * 128 + 48 + 4].view("<u2")[0]) == 0x4000
    assert np.count_nonzero(p) == 3  # 0x80,0x3F and 0x40


def test_chunk_offsets_meta_at_group_starts():
    """g128 w4 asym: stages of 64 -> meta (512 B) only at even stages; chunk 1 starts at 512 + 4096."""
    N, K = 128, 256
    rng = np.random.default_rng(0)
    codes, scale, zero = _rand_codes(rng, 4, 16, 128, False, N, K)
    p = pack_block(codes, scale, zero, 4, 16, 128, False)
    CB = 128 * 64 * 4 // 8
    assert p.size == 4 * CB + 2 * 512
    # stage 1 codes immediately follow stage 0 codes (no meta)
    u = codes[0, 64:72]
    nib = [0] * 8
    for i in range(8):
        nib[(i >> 1) + 4 * (i & 1)] = u[i]
    word = sum(int(v) << (4 * k) for k, v in enumerate(nib))
    assert int(p[512 + CB: 512 + CB + 4].view("<u4")[0]) == word
