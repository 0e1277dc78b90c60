"""Bit-exact parity of the hot path's integer stages, read back from a real mxm_moe_group_gemm call.

North star: "Packed codes, scales and int32 accumulations must match the oracle bit-exactly". After one call
through the C ABI (the accumulator-dump instantiation of the persistent kernel, mxm_debug_moe_group_gemm_dump)
the workspace holds the hot path's own intermediates; each is compared with the oracle on the same inputs:
  - gather (S2): bf16 rows and the activation quantizer's codes / scales / code sums of every route row vs
    oracle.quant.quantize_act of x[token] (reading R9);
  - h quantization (S5): the fused g128 and per-token quantizers' codes / scales / sums vs quantize_act of the
    GPU's own bf16 h (the bf16 rounding of h itself is floating point and checked by the 1e-2 gate);
  - accumulators (S4/S6): every weight-activation block's per-group integer accumulator vs
    oracle.moe.wa_int_accumulators(q_a, q_w, group) (reading G). kind::i8 blocks (w5a5, w8a8) dump the int32;
    kind::f8f6f4 blocks (w4a4) dump the f32 2^-18 * sum (q_w + 8) q_a, which must be an exact integer
    multiple of 2^-18.
"""
import numpy as np
import pytest
import torch

from oracle.moe import wa_int_accumulators
from oracle.quant import quantize_act, quantize_weight
from synth import configs as C
from synth.gen import bf16_bits_to_f64
from tests.moe_cases import bf16_tensor, gpu_layer, make_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mx():
    import paper_2505_05799_b200 as mx
    mx.load()
    return mx


def _view(ws_np, off, dtype, count):
    return np.frombuffer(ws_np[off: off + np.dtype(dtype).itemsize * count].tobytes(), dtype=dtype)


def decode_codes(raw_u8: np.ndarray, a_bits: int) -> np.ndarray:
    """Integer codes from the hot path's code bytes: two's complement (a5, a8) or e4m3 (q<0)<<7 | |q| (a4)."""
    raw = raw_u8.astype(np.int64)
    if a_bits == 4:
        mag = raw & 0x7F
        assert (mag <= 7).all(), "a4 e4m3 code magnitude out of range"
        return np.where(raw & 0x80, -mag, mag)
    return raw_u8.view(np.int8).astype(np.int64)


def _slots(table_row):
    """Input slot of gate / up (0 bf16, 1 slot A, 2 slot B): the layer's rule (api.cu mxm_layer_init)."""
    g, u = table_row[0], table_row[1]
    gwa, uwa = g.a_bits != 16, u.a_bits != 16
    sg = 1 if gwa else 0
    if not uwa:
        su = 0
    elif gwa and g.a_bits == u.a_bits and g.a_group == u.a_group:
        su = 1
    else:
        su = 2 if gwa else 1
    return sg, su


def _run(mx, case):
    layer = gpu_layer(case)
    T, k = case["T"], case["k"]
    x = bf16_tensor(case["x"])
    ids = torch.from_numpy(np.ascontiguousarray(case["ids"], dtype=np.int32)).cuda()
    w = torch.from_numpy(np.ascontiguousarray(case["w"], dtype=np.float32)).cuda()
    sw = None if case["shared_w"] is None else torch.from_numpy(case["shared_w"]).cuda()
    y, ws, acc_gu, acc_dn = layer.call_dump(x, ids, w, sw)
    torch.cuda.synchronize()
    assert layer.poll_error(ws) == 0
    lay = layer.workspace_layout(T, k)
    return layer, lay, ws.cpu().numpy(), acc_gu.cpu().numpy().view(np.uint32), acc_dn.cpu().numpy().view(np.uint32)


def _acc_as_int(raw_u32: np.ndarray, f8: bool, qsum: np.ndarray) -> np.ndarray:
    """int32 accumulator words (i8 kinds), or the exact integer sum (q_w + 8) q_a - 8 sum q_a from f32 words."""
    if not f8:
        return raw_u32.view(np.int32).astype(np.int64)
    v = raw_u32.view(np.float32).astype(np.float64) * 262144.0
    assert np.array_equal(v, np.rint(v)), "f8 accumulator is not an integer multiple of 2^-18"
    return v.astype(np.int64) - 8 * qsum[:, None]


def _h_rows(ws, off, dtype, case, rows, v):
    """h / h-code rows of expert v from the two-region layout (include/mxmoe.h MXM_WS_H): the T*S shared rows at
    the shared width first, then the routed rows at the routed width."""
    cfg, T, k = case["cfg"], case["T"], case["k"]
    srows, fs, f = T * cfg.n_shared, cfg.shared_inter if cfg.n_shared else 0, cfg.inter
    if v >= cfg.n_routed:
        return _view(ws, off, dtype, srows * fs).reshape(srows, fs)[rows]
    base = off + srows * fs * np.dtype(dtype).itemsize
    return _view(ws, base, dtype, T * k * f).reshape(T * k, f)[rows - srows]


def check_case(mx, case, min_rows=1):
    cfg, table = case["cfg"], case["table"]
    E, S, d = cfg.n_routed, cfg.n_shared, cfg.hidden
    layer, lay, ws, acc_gu, acc_dn = _run(mx, case)
    R, F = lay["R"], lay["f_max"]
    row_src = _view(ws, lay["row_src"], np.int32, R)
    v_off = _view(ws, lay["v_off"], np.int32, E + S + 1)
    x64 = bf16_bits_to_f64(case["x"])
    checked = 0
    for v in range(E + S):
        # routed expert v: rows [v_off[v], v_off[v+1]) (the last one ends at v_off[E+S]); shared: T rows
        r0 = int(v_off[v])
        r1 = r0 + case["T"] if v >= E else int(v_off[v + 1] if v + 1 < E else v_off[E + S])
        rows = np.arange(r0, r1)
        if rows.size == 0:
            continue
        f = cfg.inter if v < E else cfg.shared_inter
        xin = x64[row_src[rows]]
        slots = _slots(table[v])
        # ---- gate / up input codes and accumulators
        for j in (0, 1):
            sch = table[v][j]
            if sch.a_bits == 16:
                if slots[j] == 0:  # gathered bf16 rows
                    xb = _view(ws, lay["xb"], np.uint16, R * d).reshape(R, d)
                    assert np.array_equal(xb[rows], case["x"][row_src[rows]]), "gathered bf16 rows"
                continue
            name = "a" if slots[j] == 1 else "b"
            G = d // 128 if sch.a_group == 128 else 1
            q_ref, s_ref, qs_ref = quantize_act(xin.astype(np.float32), sch.a_bits, sch.a_group)
            codes = decode_codes(_view(ws, lay["xq" + name], np.uint8, R * d).reshape(R, d)[rows], sch.a_bits)
            scales = _view(ws, lay["xs" + name], np.float32, G * R).reshape(G, R)[:, rows].T
            assert np.array_equal(codes, q_ref), f"expert {v} block {j}: activation codes"
            assert np.array_equal(scales, s_ref), f"expert {v} block {j}: activation scales"
            f8 = sch.w_bits == 4
            if f8:
                qs = _view(ws, lay["xc" + name], np.int32, G * R).reshape(G, R)[:, rows].T
                assert np.array_equal(qs.astype(np.int64), qs_ref), f"expert {v} block {j}: code sums"
            qw, _, _ = quantize_weight(case["weights"][v][j], sch.w_bits, sch.w_group, True)
            ref = wa_int_accumulators(q_ref, qw, sch.w_group)  # [G, m, f]
            for g in range(ref.shape[0]):
                got = _acc_as_int(acc_gu[j, g][rows][:, :f], f8, qs_ref[:, g] if f8 else None)
                assert np.array_equal(got, ref[g].astype(np.int64)), f"expert {v} block {j} group {g}: accumulators"
            checked += rows.size
        # ---- down input (h) quantization and accumulators
        sch = table[v][2]
        if sch.a_bits != 16:
            G = f // 128 if sch.a_group == 128 else 1
            h_bits = _h_rows(ws, lay["h"], np.uint16, case, rows, v)
            hin = bf16_bits_to_f64(h_bits).astype(np.float32)
            q_ref, s_ref, qs_ref = quantize_act(hin, sch.a_bits, sch.a_group)
            codes = decode_codes(_h_rows(ws, lay["hq"], np.uint8, case, rows, v), sch.a_bits)
            scales = _view(ws, lay["hs"], np.float32, (F // 128) * R).reshape(F // 128, R)[:G, rows].T
            assert np.array_equal(codes, q_ref), f"expert {v} down: h codes"
            assert np.array_equal(scales, s_ref), f"expert {v} down: h scales"
            f8 = sch.w_bits == 4
            if f8:
                qs = _view(ws, lay["hc"], np.int32, (F // 128) * R).reshape(F // 128, R)[:G, rows].T
                assert np.array_equal(qs.astype(np.int64), qs_ref), f"expert {v} down: h code sums"
            qw, _, _ = quantize_weight(case["weights"][v][2], sch.w_bits, sch.w_group, True)
            ref = wa_int_accumulators(q_ref, qw, sch.w_group)
            for g in range(ref.shape[0]):
                got = _acc_as_int(acc_dn[g][rows][:, :d], f8, qs_ref[:, g] if f8 else None)
                assert np.array_equal(got, ref[g].astype(np.int64)), f"expert {v} down group {g}: accumulators"
            checked += rows.size
    assert checked >= min_rows


WA = [C.WA(b, g) for b in (4, 5, 8) for g in (128, -1)]


@pytest.mark.parametrize("sch", WA, ids=lambda s: s.name())
@pytest.mark.parametrize("T", [1, 17, 64, 96, 300])
def test_uniform_wa_bitexact(mx, sch, T):
    """Every W-A scheme x per-channel / g128, m spanning 1 .. 300 tokens per expert (ragged tiles, pairs)."""
    cfg = C.LayerConfig("bx", 2, 0, 256, 512, 0, 2, T)
    case = make_case(cfg, C.uniform_table(cfg, sch), T, seed=T)
    check_case(mx, case)


def test_mixed_hetero_and_shared_bitexact(mx):
    """Heterogeneous gate/up pairs (two sub-loops, two input slots), a shared expert and every W-A kind."""
    cfg = C.LayerConfig("bx2", 4, 1, 256, 384, 512, 2, 80)
    a4g, a4c, a5g, a8c = C.WA(4, 128), C.WA(4, -1), C.WA(5, 128), C.WA(8, -1)
    table = [[a4g, a8c, a5g], [a8c, a4g, a4c], [a5g, a5g, a8c], [C.WO(4, 128), a4c, a4g], [a4c, a4c, a8c]]
    case = make_case(cfg, table, 80, seed=3)
    check_case(mx, case)


@pytest.mark.parametrize("sch", [C.WA(4, 128), C.WA(8, -1), C.WA(4, -1)], ids=lambda s: s.name())
def test_long_k_bitexact(mx, sch):
    """Down K = 14336 (Mixtral inter): whole-K int32 / exact f32 sums at the largest reduction length."""
    cfg = C.LayerConfig("bxk", 2, 0, 256, 14336, 0, 1, 24)
    case = make_case(cfg, C.uniform_table(cfg, sch), 24, seed=5)
    check_case(mx, case)


def test_token_major_gather_equals_row_major(mx, monkeypatch):
    """S2: the token-major gather (each token quantized once per input format, stored to all its route rows)
    writes the same bytes as the row-major one (one warp per route row), here with a bf16 slot, three quantized
    formats (e4m3 per-token and g128, int8 per-token), two input slots and a shared expert."""
    cfg = C.LayerConfig("bx3", 4, 1, 256, 384, 512, 3, 70)
    a4g, a4c, a8c = C.WA(4, 128), C.WA(4, -1), C.WA(8, -1)
    table = [[a4g, a8c, a4g], [a8c, a4g, a4c], [C.WO(4, 128), a4c, a4g], [C.WO(2, 128), C.W16, a8c],
             [a4c, a4c, a8c]]
    case = make_case(cfg, table, 70, seed=11)
    check_case(mx, case)
    _, lay, ws_tok, _, _ = _run(mx, case)
    monkeypatch.setenv("MXM_GATHER_ROWS", "1")
    _, _, ws_row, _, _ = _run(mx, case)
    R, d = lay["R"], cfg.hidden
    for key, n in (("xb", 2 * R * d), ("xqa", R * d), ("xqb", R * d), ("xsa", 4 * R * (d // 128)),
                   ("xsb", 4 * R * (d // 128)), ("xca", 4 * R * (d // 128)), ("xcb", 4 * R * (d // 128))):
        off = lay[key]
        if off < 0:
            continue
        # only rows that hold a route are defined (rows past the last valid route are never written)
        assert np.array_equal(ws_tok[off: off + n], ws_row[off: off + n]), key
