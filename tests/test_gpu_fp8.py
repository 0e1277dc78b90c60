"""NEXT-4 FP8 e4m3 scheme on the GPU (readings R25/R26) against oracle/fp8.py through the C ABI:
  - weight quantizer: e4m3 code bytes and bf16 scales bit-exact; packed bytes = the oracle's image packing;
  - the hot path's activation quantizer: FP8 codes / scales of every route row read back from a real call
    (token-major gather), bit-exact;
  - whole block at the 1e-2 gate (R19): uniform FP8 per-channel and g128 tables, FP8 mixed with integer schemes
    (heterogeneous gate/up, FP8 g128 / per-token downs, a shared expert), ragged token counts.
The f32 tensor-core sums over e4m3 products are not exact (unlike the integer kinds), so accumulators are
checked through the block output only.
"""
import numpy as np
import pytest
import torch

from oracle.fp8 import quantize_act_fp8, quantize_weight_fp8
from oracle.pack import pack_block
from synth import configs as C
from synth.gen import bf16_bits_to_f64, gen_weight
from tests.moe_cases import bf16_tensor, gpu_layer, gpu_run, make_case, oracle_layer, oracle_run, row_rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-2


@pytest.fixture(scope="module")
def mx():
    import paper_2505_05799_b200 as mx
    mx.load()
    return mx


@pytest.mark.parametrize("group", [-1, 128])
def test_fp8_weight_quant_pack(mx, group):
    N, K = 256, 512
    W = gen_weight(N, K, 17)
    W[5, :] = 0
    sch = mx.Scheme.of(C.FP8(group))
    codes, scale, zero = mx.quantize(sch, bf16_tensor(W))
    q, s = quantize_weight_fp8(W, group)
    assert np.array_equal(codes.cpu().numpy().view(np.uint8), q), "e4m3 codes"
    assert np.array_equal(bf16_bits_to_f64(scale.view(torch.int16).cpu().numpy().view(np.uint16)), s), "scales"
    packed = mx.pack(sch, codes, scale, zero, N, K)
    ref = pack_block(q.astype(np.int64), s, None, 8, 8, group, True)
    assert np.array_equal(packed.cpu().numpy(), ref)
    deq = mx.dequantize(sch, packed, N, K).cpu().numpy().astype(np.float64)
    from oracle.fp8 import e4m3_decode
    g = K if group == -1 else group
    assert np.array_equal(deq, (e4m3_decode(q).reshape(N, -1, g) * s[:, :, None]).reshape(N, K).astype(np.float32))


@pytest.mark.parametrize("group", [-1, 128])
def test_fp8_gather_codes_bitexact(mx, group):
    """Codes / scales of every route row written by the hot path's gather (one call, workspace read back)."""
    cfg = C.LayerConfig("f8g", 4, 1, 256, 384, 256, 2, 40)
    sch = C.FP8(group)
    case = make_case(cfg, C.uniform_table(cfg, sch), 40, seed=group + 5)
    layer = gpu_layer(case)
    T, k = case["T"], case["k"]
    y, ws, _, _ = layer.call_dump(bf16_tensor(case["x"]), torch.from_numpy(case["ids"].astype(np.int32)).cuda(),
                                  torch.from_numpy(case["w"].astype(np.float32)).cuda(),
                                  None if case["shared_w"] is None else torch.from_numpy(case["shared_w"]).cuda())
    torch.cuda.synchronize()
    lay = layer.workspace_layout(T, k)
    wsn = ws.cpu().numpy()
    R, d = lay["R"], cfg.hidden
    row_src = np.frombuffer(wsn[lay["row_src"]: lay["row_src"] + 4 * R].tobytes(), np.int32)
    v_off = np.frombuffer(wsn[lay["v_off"]: lay["v_off"] + 4 * (cfg.n_routed + 2)].tobytes(), np.int32)
    rows = np.arange(0, int(v_off[cfg.n_routed + cfg.n_shared]))  # shared rows then routed rows
    xq = wsn[lay["xqa"]: lay["xqa"] + R * d].reshape(R, d)[rows]
    G = d // 128 if group == 128 else 1
    xs = np.frombuffer(wsn[lay["xsa"]: lay["xsa"] + 4 * R * (d // 128)].tobytes(), np.float32)
    xs = xs.reshape(d // 128, R)[:G, rows].T
    q_ref, s_ref = quantize_act_fp8(bf16_bits_to_f64(case["x"][row_src[rows]]).astype(np.float32), group)
    assert np.array_equal(xq, q_ref), "FP8 activation codes"
    assert np.array_equal(xs, s_ref), "FP8 activation scales"


def _parity(case):
    layer = gpu_layer(case)
    y = gpu_run(layer, case)
    ref = oracle_run(oracle_layer(case), case)
    n, ex = layer.task_stats(case["T"], case["k"])
    assert n > 0 and ex == n and layer.poll_error() == 0
    return row_rel_err(y, ref)


@pytest.mark.parametrize("group", [-1, 128])
@pytest.mark.parametrize("T", [1, 17, 64, 300])
def test_fp8_uniform_block(mx, group, T):
    cfg = C.get_config("tiny")
    case = make_case(cfg, C.uniform_table(cfg, C.FP8(group)), T, seed=T + group)
    e = _parity(case)
    assert e <= TOL, e


def test_fp8_mixed_with_integer_schemes(mx):
    """FP8 next to the integer schemes in one launch: heterogeneous gate/up pairs (FP8 + w4a4 / weight-only), FP8
    g128 and per-token downs (fused and one-pass h quantization), a shared expert with FP8 gate/up."""
    cfg = C.LayerConfig("f8m", 5, 1, 256, 384, 512, 2, 96)
    f8c, f8g = C.FP8(-1), C.FP8(128)
    table = [[f8c, f8c, f8g], [f8g, C.WA(4, 128), f8c], [C.WO(4, 128), f8c, C.WA(8, -1)],
             [C.WA(8, -1), C.WA(8, -1), f8g], [f8g, f8g, C.WO(2, 128)], [f8c, f8c, f8c]]
    for T in (37, 96):
        case = make_case(cfg, table, T, seed=T)
        e = _parity(case)
        assert e <= TOL, (T, e)
