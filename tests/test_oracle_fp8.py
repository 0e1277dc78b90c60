"""Pins of oracle/fp8.py (NEXT-4 FP8 e4m3 scheme; readings R25, R26) against torch's float8_e4m3fn conversions
(a library routine), exhaustive code tables, exact midpoints, quantizer bounds and a dequantized-operand identity."""
import numpy as np
import pytest
import torch

from oracle.bf16 import bf16_next_down, bf16_round_f64, bits_to_f64, f64_to_bits
from oracle.fp8 import (E4M3_MAX, e4m3_decode, e4m3_round, e4m3_value, linear_block_fp8, quantize_act_fp8,
                        quantize_weight_fp8)


def test_code_table_equals_torch():
    codes = torch.arange(256, dtype=torch.int32).to(torch.uint8)
    ref = codes.view(torch.float8_e4m3fn).to(torch.float64).numpy()
    mine = np.array([e4m3_value(c) for c in range(256)])
    assert np.array_equal(np.isnan(mine), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert np.array_equal(mine[ok], ref[ok])
    assert e4m3_value(0x7E) == 448.0 and e4m3_value(0x01) == 2.0 ** -9 and e4m3_value(0x38) == 1.0


def test_round_equals_torch_including_ties():
    rng = np.random.default_rng(0)
    pos = np.array([e4m3_value(c) for c in range(0x7F)])
    mids = (pos[:-1] + pos[1:]) / 2  # exact ties
    x = np.concatenate([rng.uniform(-448, 448, 20000), rng.uniform(-0.02, 0.02, 20000), mids, -mids, pos, -pos])
    mine = e4m3_round(x)
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(mine, ref)
    assert np.array_equal(e4m3_decode(mine), torch.from_numpy(x).to(torch.float8_e4m3fn).to(torch.float64).numpy())
    with pytest.raises(ValueError):
        e4m3_round(np.array([449.0]))


@pytest.mark.parametrize("group", [-1, 128])
def test_weight_quantizer_bounds(group):
    rng = np.random.default_rng(1)
    w = f64_to_bits(bf16_round_f64(rng.standard_normal((16, 256)) * 0.05))
    w[3, :] = 0  # degenerate row
    codes, s = quantize_weight_fp8(w, group)
    x = bits_to_f64(w).reshape(16, -1, 256 if group == -1 else 128)
    a = np.abs(x).max(axis=2)
    nz = a > 0
    assert (448 * s[nz] >= a[nz]).all() and (448 * bf16_next_down(s[nz]) < a[nz]).all()
    assert (s[~nz] == 1).all() and not (codes[3] & 0x7F).any()
    assert not ((codes & 0x7F) == 0x7F).any()  # never NaN / saturated beyond 448
    v = e4m3_decode(codes).reshape(x.shape) * s[:, :, None]
    # rounding error at most half an e4m3 spacing of |w/s| (relative 2^-4 for normals, absolute 2^-10 s below)
    rel = np.abs(v - x) / np.maximum(np.abs(x), 2.0 ** -6 * s[:, :, None])
    assert (rel <= 2.0 ** -4 + 1e-12).all()


def test_act_quantizer_fixture_and_bounds():
    v = np.array([[1.0, -2.0, 0.5, 0.0], [0, 0, 0, 0], [3.0, 3.0, -3.0, 1e-3]], dtype=np.float32)
    codes, s = quantize_act_fp8(v, -1)
    assert s[0, 0] == np.float32(2.0) / np.float32(448) and s[1, 0] == 1.0
    assert e4m3_decode(codes[0])[1] == -448.0 and e4m3_decode(codes[0])[0] == 224.0
    assert not (codes[1] & 0x7F).any()
    rng = np.random.default_rng(2)
    x = rng.standard_normal((8, 256)).astype(np.float32)
    c, s = quantize_act_fp8(x, 128)
    d = e4m3_decode(c).reshape(8, 2, 128) * s[:, :, None]
    xg = x.reshape(8, 2, 128).astype(np.float64)
    assert (np.abs(d - xg) <= np.maximum(np.abs(xg) * 2.0 ** -4, 2.0 ** -10 * s[:, :, None]) * 1.0001).all()


def test_linear_block_identity():
    """y = (s_a q_a)(s_w q_w)^T per group: the same real numbers through an independent torch fp64 matmul."""
    rng = np.random.default_rng(3)
    w = f64_to_bits(bf16_round_f64(rng.standard_normal((24, 256)) * 0.05))
    x = bf16_round_f64(rng.standard_normal((5, 256)))
    for wg, ag in ((-1, -1), (128, 128)):
        cw, sw = quantize_weight_fp8(w, wg)
        ca, sa = quantize_act_fp8(x.astype(np.float32), ag)
        g = 256 if wg == -1 else 128
        wd = torch.tensor(e4m3_decode(cw).reshape(24, -1, g) * sw[:, :, None]).reshape(24, 256)
        xd = torch.tensor(e4m3_decode(ca).reshape(5, -1, g) * sa.astype(np.float64)[:, :, None]).reshape(5, 256)
        ref = (xd @ wd.T).numpy()
        got = linear_block_fp8(x, cw, sw, wg, ag)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
