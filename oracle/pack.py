"""Native packed layout (docs/packed_format.md), written out plainly.

Step S0b of the hot-path table: planes per P:225 ("fused
dequantization with bit manipulation"), 16-bit meta per P:339. The layout itself is
this project's definition; this module follows docs/packed_format.md line by line.
"""
from __future__ import annotations

import numpy as np

from .bf16 import f64_to_bits


def kind_of(w_bits: int, a_bits: int) -> str:
    if w_bits == 16 or a_bits == 16:
        return "F16"
    return "I8"


def stage_elems(kind: str) -> int:
    return 64 if kind == "F16" else 128


def planes_of(w_bits: int) -> list:
    return {2: [2], 3: [2, 1], 4: [4], 5: [4, 1], 8: [8]}[w_bits]


def field_pos(kind: str, pb: int, i: int) -> int:
    """Bit-field index f of local element i' inside a plane word (table in the doc)."""
    if kind == "F16":
        if pb == 2:
            return (i >> 1) + 8 * (i & 1)
        if pb == 1:
            return (i >> 1) + 16 * (i & 1)
        if pb == 4:
            return (i >> 1) + 4 * (i & 1)
        if pb == 8:
            return i
    else:
        if pb == 4:
            return 2 * i if i < 4 else 2 * (i - 4) + 1
        if pb == 1:
            return 8 * (i & 3) + (i >> 2)
    raise ValueError((kind, pb))


def _is_image(w_bits: int, a_bits: int) -> bool:
    return w_bits == 16 or (w_bits == 8 and a_bits == 8)


def _meta_bytes(w_bits, a_bits, symmetric):
    if kind_of(w_bits, a_bits) == "I8" or w_bits == 16:
        return 0
    return 256 if symmetric else 512


def _code_bytes(w_bits, a_bits):
    kind = kind_of(w_bits, a_bits)
    if w_bits == 16:
        return 16384
    return 128 * stage_elems(kind) * w_bits // 8


def packed_size(w_bits, a_bits, group, symmetric, N, K) -> int:
    kind = kind_of(w_bits, a_bits)
    KS = stage_elems(kind)
    g = K if group == -1 else group
    NS, RB, NG = K // KS, N // 128, (K // g if w_bits != 16 else 0)
    total = RB * (NS * _code_bytes(w_bits, a_bits) + NG * _meta_bytes(w_bits, a_bits, symmetric))
    if kind == "I8":
        total += NG * N * 2
    return total


def _swizzle_image(rows_bytes: np.ndarray) -> np.ndarray:
    """rows_bytes uint8[128, 128] -> 16384-byte canonical SW128 image."""
    img = np.zeros(16384, dtype=np.uint8)
    for r in range(128):
        for b in range(128):
            img[r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15)] = rows_bytes[r, b]
    return img


def pack_block(codes, scale, zero, w_bits, a_bits, group, symmetric) -> np.ndarray:
    """codes: int [N,K] canonical codes (w16: uint16 bf16 bits); scale/zero: float64 [N, K/g]."""
    codes = np.asarray(codes)
    N, K = codes.shape
    kind = kind_of(w_bits, a_bits)
    KS = stage_elems(kind)
    g = K if group == -1 else group
    if N % 128 or K % KS or K % g:
        raise ValueError("shape not packable")
    out = np.zeros(packed_size(w_bits, a_bits, group, symmetric, N, K), dtype=np.uint8)
    pos = 0
    if w_bits == 16:
        u = codes.astype(np.uint16)
    elif kind == "F16" and not symmetric:
        u = codes.astype(np.int64)
    elif w_bits == 8 and a_bits == 8:
        u = codes.astype(np.int64) & 0xFF  # two's complement byte
    else:
        u = codes.astype(np.int64) + 2 ** (w_bits - 1)  # offset binary
    for rb in range(N // 128):
        rows = slice(rb * 128, rb * 128 + 128)
        for ks in range(K // KS):
            cols = slice(ks * KS, ks * KS + KS)
            if _is_image(w_bits, a_bits):
                if w_bits == 16:
                    blk = u[rows, cols].astype("<u2").view(np.uint8).reshape(128, 128)
                else:
                    blk = u[rows, cols].astype(np.uint8)
                out[pos:pos + 16384] = _swizzle_image(blk)
                pos += 16384
                continue
            if kind == "F16" and (ks * KS) % g == 0:
                grp = ks * KS // g
                out[pos:pos + 256] = f64_to_bits(scale[rows, grp]).astype("<u2").view(np.uint8)
                pos += 256
                if not symmetric:
                    out[pos:pos + 256] = f64_to_bits(zero[rows, grp]).astype("<u2").view(np.uint8)
                    pos += 256
            ublk = u[rows, cols]  # [128, KS]
            shift = 0
            for pb in planes_of(w_bits):
                plane = (ublk >> shift) & ((1 << pb) - 1)
                shift += pb
                per_word = 32 // pb
                W = KS // per_word
                words = np.zeros((W, 128), dtype=np.uint64)
                for j in range(W):
                    for ii in range(per_word):
                        f = field_pos(kind, pb, ii)
                        words[j] |= plane[:, j * per_word + ii].astype(np.uint64) << np.uint64(f * pb)
                out[pos:pos + W * 128 * 4] = words.astype("<u4").reshape(-1).view(np.uint8)
                pos += W * 128 * 4
    if kind == "I8":
        NG = K // g
        sc = np.ascontiguousarray(scale.T)  # [NG, N]
        out[pos:pos + NG * N * 2] = f64_to_bits(sc).astype("<u2").reshape(-1).view(np.uint8)
        pos += NG * N * 2
    assert pos == out.size
    return out


def unpack_block(packed, w_bits, a_bits, group, symmetric, N, K):
    """Inverse of pack_block: returns (codes, scale, zero) in canonical form (self-test aid)."""
    from .bf16 import bits_to_f64

    kind = kind_of(w_bits, a_bits)
    KS = stage_elems(kind)
    g = K if group == -1 else group
    NG = K // g
    codes = np.zeros((N, K), dtype=np.int64)
    scale = np.zeros((N, NG)) if w_bits != 16 else None
    zero = np.zeros((N, NG)) if (kind == "F16" and not symmetric and w_bits != 16) else None
    pos = 0
    for rb in range(N // 128):
        rows = slice(rb * 128, rb * 128 + 128)
        for ks in range(K // KS):
            cols = slice(ks * KS, ks * KS + KS)
            if _is_image(w_bits, a_bits):
                img = packed[pos:pos + 16384]
                blk = np.zeros((128, 128), dtype=np.uint8)
                for r in range(128):
                    for b in range(128):
                        blk[r, b] = img[r * 128 + (((b >> 4) ^ (r & 7)) << 4) + (b & 15)]
                if w_bits == 16:
                    codes[rows, cols] = blk.reshape(-1).view("<u2").reshape(128, 64)
                else:
                    codes[rows, cols] = blk.astype(np.int8)
                pos += 16384
                continue
            if kind == "F16" and (ks * KS) % g == 0:
                grp = ks * KS // g
                scale[rows, grp] = bits_to_f64(packed[pos:pos + 256].view("<u2"))
                pos += 256
                if not symmetric:
                    zero[rows, grp] = bits_to_f64(packed[pos:pos + 256].view("<u2"))
                    pos += 256
            u = np.zeros((128, KS), dtype=np.int64)
            shift = 0
            for pb in planes_of(w_bits):
                per_word = 32 // pb
                W = KS // per_word
                words = packed[pos:pos + W * 128 * 4].view("<u4").reshape(W, 128).astype(np.int64)
                pos += W * 128 * 4
                for j in range(W):
                    for ii in range(per_word):
                        f = field_pos(kind, pb, ii)
                        u[:, j * per_word + ii] |= ((words[j] >> (f * pb)) & ((1 << pb) - 1)) << shift
                shift += pb
            if kind == "F16" and not symmetric:
                codes[rows, cols] = u
            else:
                codes[rows, cols] = u - 2 ** (w_bits - 1)
    if kind == "I8":
        sc = packed[pos:pos + NG * N * 2].view("<u2").reshape(NG, N)
        scale = bits_to_f64(sc).T.copy()
    return codes, scale, zero
