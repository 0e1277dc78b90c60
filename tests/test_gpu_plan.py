"""Scheduler structure, read back from the workspace of a real call:
  - the queue holds every phase-0 task before every h-quant task before every down task (the order that makes
    the dynamic queue deadlock-free);
  - the m-tile groups of each expert partition its route rows, with token tiles 16 / 32 / 64 / cap;
  - every (group, gate/up 128-channel tile), every (group, 32-row h-quant chunk) of a per-token W-A down and
    every (group, down tile or tile pair, K slice) appears exactly once (a per-task visit count);
  - the kernel executed every task exactly once;
  - ten repeated calls give bit-identical outputs.
"""
import numpy as np
import pytest
import torch

from synth import configs as C
from tests.moe_cases import bf16_tensor, gpu_layer, make_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mx():
    import paper_2505_05799_b200 as mx
    mx.load()
    return mx


def _call(layer, case):
    T, k = case["T"], case["k"]
    x = bf16_tensor(case["x"])
    ids = torch.from_numpy(np.ascontiguousarray(case["ids"], dtype=np.int32)).cuda()
    w = torch.from_numpy(np.ascontiguousarray(case["w"], dtype=np.float32)).cuda()
    sw = None if case["shared_w"] is None else torch.from_numpy(case["shared_w"]).cuda()
    ws = layer.workspace(T, k)
    y = layer(x, ids, w, sw, workspace=ws)
    torch.cuda.synchronize()
    return y, ws


def check_plan(mx, cfg, table, T, seed=1):
    case = make_case(cfg, table, T, seed=seed)
    layer = gpu_layer(case)
    _, ws = _call(layer, case)
    k = case["k"]
    lay = layer.workspace_layout(T, k)
    wsn = ws.cpu().numpy()
    gmax = lay["g_max"]
    meta = np.frombuffer(wsn[lay["meta"]: lay["meta"] + 4 * (8 + 4 * gmax)].tobytes(), np.int32)
    n_tasks, n1, nq, n2, G, _, executed, S = (int(v) for v in meta[:8])
    assert n_tasks == n1 + nq + n2 and executed == n_tasks
    gv, grow0, grows, gnt = (meta[8 + i * gmax: 8 + i * gmax + G] for i in range(4))
    rec = np.frombuffer(wsn[lay["tasks"]: lay["tasks"] + 16 * n_tasks].tobytes(),
                        dtype=np.dtype([("expert", "<u2"), ("phase", "u1"), ("nt", "u1"), ("row0", "<i4"),
                                        ("rows", "<u2"), ("ntile", "<u2"), ("gid", "<i4")]))
    # phase order of the queue
    ph = rec["phase"].astype(np.int64)
    assert np.all(np.diff(ph) >= 0), "a later-phase task precedes an earlier-phase one"
    assert (ph == 0).sum() == n1 and (ph == 1).sum() == nq and (ph == 2).sum() == n2
    # groups partition each expert's route rows
    E, Sh = cfg.n_routed, cfg.n_shared
    v_off = np.frombuffer(wsn[lay["v_off"]: lay["v_off"] + 4 * (E + Sh + 1)].tobytes(), np.int32)
    for v in range(E + Sh):
        lo = int(v_off[v])
        hi = lo + T if v >= E else int(v_off[v + 1] if v + 1 < E else v_off[E + Sh])
        mine = np.nonzero(gv == v)[0]
        spans = sorted((int(grow0[g]), int(grow0[g]) + int(grows[g])) for g in mine)
        cover = lo
        for a, b in spans:
            assert a == cover, (v, spans)
            cover = b
        assert cover == hi, (v, cover, hi)
        for g in mine:
            assert gnt[g] in (16, 32, 64, 96) and grows[g] <= gnt[g] and grows[g] > 0
    # visit counts
    nd = cfg.hidden // 128
    for g in range(G):
        v = int(gv[g])
        sch = table[v]
        f = cfg.inter if v < E else cfg.shared_inter
        t0 = rec[(rec["gid"] == g) & (rec["phase"] == 0)]
        assert sorted(t0["ntile"].tolist()) == list(range(f // 128)), ("gate/up tiles", g)
        wa_down = sch[2].a_bits != 16
        g128_down = wa_down and sch[2].a_group == 128
        tq = rec[(rec["gid"] == g) & (rec["phase"] == 1)]
        want_q = (int(grows[g]) + 31) // 32 if wa_down and not g128_down else 0
        assert sorted(tq["ntile"].tolist()) == list(range(want_q)), ("h-quant chunks", g)
        t2 = rec[(rec["gid"] == g) & (rec["phase"] == 2)]
        pair = nd >= 2 and not (g128_down and gnt[g] > 64)
        n_down = (nd + 1) // 2 if pair else nd
        slices = S if (S > 1 and not g128_down) else 1
        got = sorted(((int(t) & 0x3FF), (int(t) >> 10)) for t in t2["ntile"])
        assert got == sorted((j, s) for j in range(n_down) for s in range(slices)), ("down tasks", g)
    return case, layer


def test_plan_tiny_mixed(mx):
    cfg = C.get_config("tiny")
    check_plan(mx, cfg, C.precision_table(cfg), 80)


def test_plan_mixed_wa_with_shared(mx):
    cfg = C.LayerConfig("pl2", 6, 1, 256, 384, 512, 3, 300)
    a4g, a8c, a5g = C.WA(4, 128), C.WA(8, -1), C.WA(5, 128)
    table = [[a4g, a4g, a8c], [a8c, a8c, a4g], [C.WO(4, 128)] * 3, [a5g, a8c, a5g], [C.FP8(-1)] * 3,
             [a4g, a4g, a4g], [a8c, a8c, a8c]]
    check_plan(mx, cfg, table, 300, seed=2)


def test_plan_dsv2_and_split_k(mx):
    cfg = C.get_config("dsv2")
    check_plan(mx, cfg, C.precision_table(cfg), 512, seed=3)
    mxc = C.get_config("mx")
    for T in (1, 8):  # split-K of the downs: every (tile pair, slice) once
        check_plan(mx, mxc, C.precision_table(mxc, T), T, seed=T)


def test_ten_repeats_bit_identical(mx):
    cfg = C.LayerConfig("pl3", 6, 1, 256, 384, 512, 3, 200)
    table = [[C.WA(4, 128)] * 3, [C.WA(8, -1)] * 3, [C.WO(2, -1)] * 3, [C.FP8(128)] * 3, [C.WA(4, -1)] * 3,
             [C.WO(3, 128)] * 3, [C.WA(8, -1), C.WA(8, -1), C.WA(4, 128)]]
    case = make_case(cfg, table, 200, seed=9)
    layer = gpu_layer(case)
    y0, _ = _call(layer, case)
    y0 = y0.clone()
    for _ in range(10):
        y, _ = _call(layer, case)
        assert torch.equal(y, y0)
