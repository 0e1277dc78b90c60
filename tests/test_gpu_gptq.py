"""NEXT-4 parity: the CUDA randomized-Hadamard rotation and GPTQ (mxm_hadamard_rotate, mxm_gptq_*)
against oracle/gptq.py (readings R22-R24) on the same seeded inputs.

Both sides run in fp64; the rotation's bf16 outputs and GPTQ's integer codes, bf16 scales and zeros are compared
bit-exactly (a code is decided by fp64 arithmetic on both sides; the Hessian / inverse-factor differ only in the
last bits of their sums, far from any rounding boundary of the seeded data).
"""
import numpy as np
import pytest
import torch

from oracle.bf16 import bf16_round_f64, bits_to_f64, f64_to_bits
from oracle.gptq import gptq_hessian, gptq_prepare, gptq_quantize, rotate_expert, rotate_rows
from oracle.quant import dequantize_weight
from synth import configs as C

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mx():
    import paper_2505_05799_b200 as mx
    mx.load()
    return mx


def _bf16(rng, shape, scale=1.0):
    return f64_to_bits(bf16_round_f64(rng.standard_normal(shape) * scale))


def _t(bits_u16):
    return torch.from_numpy(np.ascontiguousarray(bits_u16).view(np.int16)).view(torch.bfloat16).cuda()


def _np_bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("N,K", [(128, 256), (384, 128), (96, 512)])
def test_hadamard_rotate_bitexact(mx, N, K):
    rng = np.random.default_rng(N + K)
    w = _bf16(rng, (N, K), 0.05)
    sk = rng.choice([-1, 1], size=K).astype(np.int8)
    sn = rng.choice([-1, 1], size=N).astype(np.int8)
    got1 = _np_bits(mx.hadamard_rotate(_t(w), torch.from_numpy(sk).cuda(), 1))
    ref1 = f64_to_bits(bf16_round_f64(rotate_rows(bits_to_f64(w), sk)))
    assert np.array_equal(got1, ref1)
    if N % 128 == 0:
        got0 = _np_bits(mx.hadamard_rotate(_t(w), torch.from_numpy(sn).cuda(), 0))
        ref0 = f64_to_bits(bf16_round_f64(rotate_rows(bits_to_f64(w).T, sn).T))
        assert np.array_equal(got0, ref0)


def test_rotate_expert_axes(mx):
    """The three blocks of an expert: gate / up rotated along K = d, down along N = d (R22)."""
    rng = np.random.default_rng(3)
    d, f = 256, 384
    wg, wu, wd = _bf16(rng, (f, d), 0.05), _bf16(rng, (f, d), 0.05), _bf16(rng, (d, f), 0.05)
    sig = rng.choice([-1, 1], size=d).astype(np.int8)
    rg, ru, rd = rotate_expert(bits_to_f64(wg), bits_to_f64(wu), bits_to_f64(wd), sig)
    st = torch.from_numpy(sig).cuda()
    assert np.array_equal(_np_bits(mx.hadamard_rotate(_t(wg), st, 1)), f64_to_bits(bf16_round_f64(rg)))
    assert np.array_equal(_np_bits(mx.hadamard_rotate(_t(wu), st, 1)), f64_to_bits(bf16_round_f64(ru)))
    assert np.array_equal(_np_bits(mx.hadamard_rotate(_t(wd), st, 0)), f64_to_bits(bf16_round_f64(rd)))


def _calib(rng, n, K):
    mix = rng.standard_normal((K, K)) * (0.5 / np.sqrt(K)) + np.eye(K)
    return f64_to_bits(bf16_round_f64(rng.standard_normal((n, K)) @ mix))


def test_hessian_and_prepare(mx):
    rng = np.random.default_rng(7)
    n, K = 300, 256
    x = _calib(rng, n, K)
    x[:, 5] = 0  # a dead input channel
    H = mx.gptq_hessian(_t(x))
    href = gptq_hessian(bits_to_f64(x))
    assert np.abs(H.cpu().numpy() - href).max() <= 1e-12 * np.abs(href).max()
    U, dead = mx.gptq_prepare(H.clone())
    uref, _ = gptq_prepare(href, np.zeros((1, K)))
    assert np.array_equal(dead.cpu().numpy(), (np.arange(K) == 5).astype(np.int32))
    assert np.abs(U.cpu().numpy() - uref).max() <= 1e-9 * np.abs(uref).max()
    assert not np.tril(U.cpu().numpy(), -1).any()


SCHEMES = [C.WO(4, 128), C.WO(3, 128), C.WO(2, -1), C.WO(2, 128), C.WO(4, 64, True), C.WO(8, -1, True),
           C.WA(4, 128), C.WA(8, -1)]


@pytest.mark.parametrize("sch", SCHEMES, ids=lambda s: s.name())
def test_gptq_bitexact(mx, sch):
    rng = np.random.default_rng(sch.w_bits * 31 + (sch.w_group + 1))
    N, K, n = 256, 384, 512
    x = _calib(rng, n, K)
    w = _bf16(rng, (N, K), 0.05)
    H = mx.gptq_hessian(_t(x))
    U, dead = mx.gptq_prepare(H)
    codes, scale, zero = mx.gptq_quantize(mx.Scheme.of(sch), _t(w), U, dead)
    sym = sch.symmetric or sch.a_bits != 16
    c_ref, s_ref, z_ref = gptq_quantize(bits_to_f64(w), gptq_hessian(bits_to_f64(x)), sch.w_bits, sch.w_group, sym)
    got = codes.cpu().numpy().astype(np.int64)
    assert np.array_equal(got, c_ref)
    assert np.array_equal(bits_to_f64(_np_bits(scale)), s_ref)
    if not sym:
        assert np.array_equal(bits_to_f64(_np_bits(zero)), z_ref)
    # the codes are in the canonical format: pack + dequantize reproduce q s + z exactly
    if sch.a_bits == 16:
        packed = mx.pack(mx.Scheme.of(sch), codes, scale, zero, N, K)
        deq = mx.dequantize(mx.Scheme.of(sch), packed, N, K).cpu().numpy().astype(np.float64)
        assert np.array_equal(deq, dequantize_weight(c_ref, s_ref, z_ref, sch.w_group))


def test_gptq_full_size_sampled_rows(mx):
    """Mixtral gate shape (N 14336, K 4096, w4-g128): GPTQ rows are independent given U, so the oracle runs on a
    seeded sample of rows with the full-K U and must reproduce those rows of the GPU result exactly."""
    rng = np.random.default_rng(1)
    N, K, n = 14336, 4096, 1024
    x = _calib(rng, n, K)
    H = mx.gptq_hessian(_t(x))
    href = H.cpu().numpy()
    U, dead = mx.gptq_prepare(H)
    w = _bf16(rng, (N, K), 0.02)
    codes, scale, zero = mx.gptq_quantize(mx.Scheme.of(C.WO(4, 128)), _t(w), U, dead)
    rows = np.sort(rng.choice(N, size=24, replace=False))
    c_ref, s_ref, z_ref = gptq_quantize(bits_to_f64(w[rows]), href, 4, 128, False)
    assert np.array_equal(codes.cpu().numpy()[rows].astype(np.int64), c_ref)
    assert np.array_equal(bits_to_f64(_np_bits(scale))[rows], s_ref)
    assert np.array_equal(bits_to_f64(_np_bits(zero))[rows], z_ref)
