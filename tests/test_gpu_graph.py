"""mxm_moe_group_gemm inside a CUDA graph (serving: launch-bound small-T steps are replayed):
one call is captured on a side stream, and its replays with NEW inputs copied into the captured buffers equal
eager calls on those inputs bitwise, including split-K (tiny T) and a layer with shared experts."""
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


def _inputs(case):
    x = bf16_tensor(case["x"])
    ids = torch.from_numpy(np.ascontiguousarray(case["ids"], dtype=np.int32)).cuda()
    w = torch.from_numpy(np.ascontiguousarray(case["w"], dtype=np.float32)).cuda()
    sw = None if case["shared_w"] is None else torch.from_numpy(case["shared_w"]).cuda()
    return x, ids, w, sw


@pytest.mark.parametrize("name,T", [("tiny", 5), ("tiny", 80), ("pl", 300)])
def test_graph_replay_equals_eager(mx, name, T):
    if name == "tiny":
        cfg = C.get_config("tiny")
        table = C.precision_table(cfg)
    else:
        cfg = C.LayerConfig("pl", 6, 1, 256, 384, 512, 3, T)
        a4g, a8c = C.WA(4, 128), C.WA(8, -1)
        table = [[a4g, a4g, a8c], [a8c, a8c, a4g], [C.WO(4, 128)] * 3, [C.FP8(-1)] * 3, [a4g] * 3,
                 [C.WO(2, -1)] * 3, [a8c] * 3]
    case0, case1 = make_case(cfg, table, T, seed=1), make_case(cfg, table, T, seed=2)
    layer = gpu_layer(case0)
    x, ids, w, sw = _inputs(case0)
    ws = layer.workspace(T, case0["k"])
    out = torch.empty(T, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):  # warm-up outside capture (tensor-map cache, smem attribute)
            layer(x, ids, w, sw, workspace=ws, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        layer(x, ids, w, sw, workspace=ws, out=out)
    for case in (case1, case0):
        x2, ids2, w2, sw2 = _inputs(case)
        x.copy_(x2)
        ids.copy_(ids2)
        w.copy_(w2)
        if sw is not None:
            sw.copy_(sw2)
        g.replay()
        torch.cuda.synchronize()
        got = out.clone()
        ref = layer(x2, ids2, w2, sw2)
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
