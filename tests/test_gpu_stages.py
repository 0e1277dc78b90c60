"""Stage-wise bit-exact GPU parity through the C ABI (quantize, pack, dequantize, act-quant, route-prep)."""
import numpy as np
import pytest
import torch

from oracle.bf16 import bits_to_f64, f64_to_bits
from oracle.moe import route_prep as o_route_prep
from oracle.pack import pack_block
from oracle.quant import dequantize_weight, quantize_act, quantize_weight
from synth.gen import bf16_bits_from_f32, gen_weight
from tests.moe_cases import bf16_tensor

pytestmark = pytest.mark.gpu

WO_SCHEMES = [(b, g, s) for b in (2, 3, 4, 8) for g in (64, 128, -1) for s in (False, True)]
WA_SCHEMES = [(b, g) for b in (4, 5, 8) for g in (128, -1)]


@pytest.fixture(scope="module")
def mx():
    import paper_2505_05799_b200 as mx
    mx.load()
    return mx


def _weights(N, K, seed):
    w = gen_weight(N, K, seed)
    rng = np.random.default_rng(seed)
    # heavy-tailed rows, a constant group and an all-zero group (degenerate cases, DESIGN R7)
    ht = bf16_bits_from_f32((rng.standard_t(2, (8, K)) * 0.05).astype(np.float32))
    w[:8] = ht
    w[8, :64] = bf16_bits_from_f32(np.full(64, 0.25, np.float32))
    w[9, :] = 0
    return w


def _check(mx, sch_tuple, N=256, K=512, seed=3):
    w_bits, a_bits, group, sym = sch_tuple
    sch = mx.Scheme(w_bits, a_bits, group, group if a_bits != 16 else -1, sym)
    W = _weights(N, K, seed + w_bits)
    codes, scale, zero = mx.quantize(sch, bf16_tensor(W))
    q, s, z = quantize_weight(W, w_bits, group, sym)
    torch.cuda.synchronize()
    assert np.array_equal(codes.cpu().numpy().astype(np.int64), q), "codes"
    assert np.array_equal(scale.view(torch.int16).cpu().numpy().view(np.uint16), f64_to_bits(s)), "scale"
    if not sym:
        assert np.array_equal(zero.view(torch.int16).cpu().numpy().view(np.uint16), f64_to_bits(z)), "zero"
    packed = mx.pack(sch, codes, scale, zero, N, K)
    ref = pack_block(q, s, z, w_bits, a_bits, group, sym)
    got = packed.cpu().numpy()
    assert got.size == ref.size
    assert np.array_equal(got, ref), f"packed bytes differ at {np.nonzero(got != ref)[0][:8]}"
    deq = mx.dequantize(sch, packed, N, K).cpu().numpy()
    assert np.array_equal(deq, dequantize_weight(q, s, z, group).astype(np.float32)), "dequant"


@pytest.mark.parametrize("sch", WO_SCHEMES)
def test_weight_only_quant_pack(mx, sch):
    _check(mx, (sch[0], 16, sch[1], sch[2]))


@pytest.mark.parametrize("sch", WA_SCHEMES)
def test_weight_act_quant_pack(mx, sch):
    _check(mx, (sch[0], sch[0], sch[1], True))


def test_w16_pack(mx):
    N, K = 256, 192
    W = gen_weight(N, K, 5)
    sch = mx.Scheme(16, 16, -1, -1, True)
    packed = mx.pack(sch, bf16_tensor(W), None, None, N, K)
    ref = pack_block(W, None, None, 16, 16, -1, True)
    assert np.array_equal(packed.cpu().numpy(), ref)
    assert np.array_equal(mx.dequantize(sch, packed, N, K).cpu().numpy(), bits_to_f64(W).astype(np.float32))


def test_quant_nonfinite_sets_error(mx):
    W = gen_weight(128, 128, 1)
    W[3, 5] = 0x7F80  # +inf
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    mx.quantize(mx.Scheme(4, 16, 128, -1, False), bf16_tensor(W), err=err)
    assert int(err.item()) == 4


def test_scheme_rejections(mx):
    with pytest.raises(mx.MxmError):
        mx.quant_sizes(mx.Scheme(6, 16, 128), 128, 256)  # unsupported bits
    with pytest.raises(mx.MxmError):
        mx.quant_sizes(mx.Scheme(4, 4, 128, -1, True), 128, 256)  # a_group != w_group
    with pytest.raises(mx.MxmError):
        mx.quant_sizes(mx.Scheme(4, 4, 128, 128, False), 128, 256)  # asym W-A
    with pytest.raises(mx.MxmError):
        mx.quant_sizes(mx.Scheme(4, 16, 128), 100, 256)  # N % 128


@pytest.mark.parametrize("bits", [4, 5, 8])
@pytest.mark.parametrize("group", [-1, 128])
def test_act_quant_bitexact(mx, bits, group):
    rng = np.random.default_rng(bits * 3 + group)
    v = bf16_bits_from_f32(rng.standard_t(3, (67, 1024)).astype(np.float32))
    v[5] = 0  # zero row
    v[6, :128] = bf16_bits_from_f32(np.array([1.0, -0.5, 0.25, 0.30078125] * 32, np.float32))  # half-way ties
    codes, scale, qsum = mx.act_quant(bf16_tensor(v), bits, group)
    q, s, qs = quantize_act(bits_to_f64(v).astype(np.float32), bits, group)
    assert np.array_equal(codes.cpu().numpy().astype(np.int64), q)
    assert np.array_equal(scale.cpu().numpy(), s)
    assert np.array_equal(qsum.cpu().numpy().astype(np.int64), qs)


@pytest.mark.parametrize("T,k,E", [(1, 1, 4), (37, 3, 5), (3000, 6, 64), (8192, 8, 64), (100, 2, 256)])
def test_route_prep_bitexact(mx, T, k, E):
    rng = np.random.default_rng(T + E)
    ids = rng.integers(-1, E, (T, k)).astype(np.int32)
    counts, offsets, perm, err = mx.route_prep(torch.from_numpy(ids).cuda(), E)
    c, o, p, _ = o_route_prep(ids, E)
    assert np.array_equal(counts.cpu().numpy(), c)
    assert np.array_equal(offsets.cpu().numpy(), o)
    assert np.array_equal(perm.cpu().numpy()[: o[-1]], p)
    assert int(err.item()) == 0


def test_route_prep_bad_id(mx):
    ids = np.array([[0, 1], [7, 2], [1, -1]], np.int32)
    counts, offsets, perm, err = mx.route_prep(torch.from_numpy(ids).cuda(), 4)
    assert int(err.item()) == 4
    assert counts.cpu().numpy().tolist() == [1, 2, 1, 0]
