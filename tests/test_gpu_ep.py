"""Expert-parallel kernels on one GPU: index semantics vs the torch reference, and a loopback emulation of
G ranks (all-to-all = tensor slicing) through the real mxm_ep_* kernels and per-rank layers, compared to
the unsharded layer and to the oracle."""
import numpy as np
import pytest
import torch

from synth import configs as C
from tests.moe_cases import bf16_tensor, make_case, oracle_layer, oracle_run, row_rel_err
from tests.test_ep_gloo import TorchRefEpOps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mx():
    import paper_2505_05799_b200 as mx
    mx.load()
    return mx


@pytest.mark.parametrize("G", [1, 2, 4])
def test_ep_kernels_match_reference(mx, G):
    from paper_2505_05799_b200.ep import CudaEpOps
    rng = np.random.default_rng(G)
    T, k, E, d = 300, 4, 8, 256
    ids = rng.integers(-1, E, (T, k)).astype(np.int32)
    w = rng.random((T, k)).astype(np.float32)
    x = torch.randn(T, d).to(torch.bfloat16)
    ops, ref = CudaEpOps(), TorchRefEpOps()
    c_g, p_g = ops.route(torch.from_numpy(ids).cuda(), E, G)
    c_r, p_r = ref.route(torch.from_numpy(ids), E, G)
    assert c_g.cpu().tolist() == c_r.tolist() and torch.equal(p_g.cpu(), p_r)
    off = [0]
    for c in c_r.tolist():
        off.append(off[-1] + c)
    off_t = torch.tensor(off, dtype=torch.int32)
    sg = ops.pack(x.cuda(), torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda(), p_g, off_t.cuda(), E, G, off[-1])
    sr = ref.pack(x, torch.from_numpy(ids), torch.from_numpy(w), p_r, off_t, E, G, off[-1])
    for a, b in zip(sg, sr):
        assert torch.equal(a.cpu(), b)
    back = torch.randn(off[-1], d).to(torch.bfloat16)
    ysh = torch.randn(T, d).to(torch.bfloat16)
    yg = ops.combine(back.cuda(), p_g, off_t.cuda(), G, ysh.cuda(), T, d)
    yr = ref.combine(back, p_r, off_t, G, ysh, T, d)
    assert torch.equal(yg.cpu(), yr)


@pytest.mark.parametrize("G", [2, 4])
def test_ep_loopback_equals_unsharded(mx, G):
    """G virtual ranks in one process: same kernels and layers as the NCCL path, all-to-all by slicing."""
    from paper_2505_05799_b200.ep import CudaEpOps
    cfg = C.get_config("dsv2")
    table = C.precision_table(cfg)
    T = 256
    case = make_case(cfg, table, T, seed=5)
    W = [[bf16_tensor(b) for b in blk] for blk in case["weights"]]
    tab = [[mx.Scheme.of(s) for s in row] for row in table]
    E, S, d = cfg.n_routed, cfg.n_shared, cfg.hidden
    epr = E // G
    locals_ = [mx.MoELayer.from_weights(epr, 0, d, cfg.inter, 0, W[r * epr:(r + 1) * epr], tab[r * epr:(r + 1) * epr])
               for r in range(G)]
    shared = mx.MoELayer.from_weights(S, 0, d, cfg.shared_inter, 0, W[E:], tab[E:])
    ops = CudaEpOps()
    Tr = T // G
    xs = [bf16_tensor(case["x"][r * Tr:(r + 1) * Tr]) for r in range(G)]
    ids = [torch.from_numpy(case["ids"][r * Tr:(r + 1) * Tr]).cuda() for r in range(G)]
    ws = [torch.from_numpy(case["w"][r * Tr:(r + 1) * Tr]).cuda() for r in range(G)]
    sws = [torch.from_numpy(case["shared_w"][r * Tr:(r + 1) * Tr]).cuda() for r in range(G)]
    route = [ops.route(ids[r], E, G) for r in range(G)]
    offs = []
    packs = []
    for r in range(G):
        c = route[r][0].cpu().tolist()
        off = [0]
        for v in c:
            off.append(off[-1] + v)
        offs.append(off)
        packs.append(ops.pack(xs[r], ids[r], ws[r], route[r][1], torch.tensor(off, dtype=torch.int32).cuda(), E, G,
                              off[-1]))
    # all-to-all: destination q receives the block for q from every source r (in source order)
    outs = {}
    for q in range(G):
        parts = [(r, offs[r][q], offs[r][q + 1]) for r in range(G)]
        rx = torch.cat([packs[r][0][a:b] for r, a, b in parts])
        rid = torch.cat([packs[r][1][a:b] for r, a, b in parts])
        rw = torch.cat([packs[r][2][a:b] for r, a, b in parts])
        ry = locals_[q](rx.contiguous(), rid.contiguous(), rw.contiguous())
        n = 0
        for r, a, b in parts:
            outs[(r, q)] = ry[n:n + (b - a)]
            n += b - a
    ys = []
    for r in range(G):
        back = torch.cat([outs[(r, q)] for q in range(G)])
        sid = torch.arange(S, dtype=torch.int32, device="cuda").repeat(Tr, 1)
        ysh = shared(xs[r], sid, sws[r])
        ys.append(ops.combine(back.contiguous(), route[r][1], torch.tensor(offs[r], dtype=torch.int32).cuda(), G, ysh,
                              Tr, d))
    y = torch.cat(ys).float().cpu().numpy().astype(np.float64)
    # sync-free exchange (ep.py): fixed capacity Tr rows per destination, padding rows with expert id -1;
    # destination q receives G * Tr rows, the valid ones in the same relative order -> the same bits
    cap = Tr
    doff = torch.arange(G + 1, dtype=torch.int32, device="cuda") * cap
    cpacks = [ops.pack(xs[r], ids[r], ws[r], route[r][1], doff, E, G, G * cap) for r in range(G)]
    couts = {}
    for q in range(G):
        rx = torch.cat([cpacks[r][0][q * cap:(q + 1) * cap] for r in range(G)])
        rid = torch.cat([cpacks[r][1][q * cap:(q + 1) * cap] for r in range(G)])
        rw = torch.cat([cpacks[r][2][q * cap:(q + 1) * cap] for r in range(G)])
        ry = locals_[q](rx.contiguous(), rid.contiguous(), rw.contiguous())
        for r in range(G):
            couts[(r, q)] = ry[r * cap:(r + 1) * cap]
    ys2 = []
    for r in range(G):
        back = torch.cat([couts[(r, q)] for q in range(G)])
        sid = torch.arange(S, dtype=torch.int32, device="cuda").repeat(Tr, 1)
        ysh = shared(xs[r], sid, sws[r])
        ys2.append(ops.combine(back.contiguous(), route[r][1], doff, G, ysh, Tr, d))
    assert torch.equal(torch.cat(ys), torch.cat(ys2))
    rows = np.arange(0, T, 4)
    ref = oracle_run(oracle_layer(case), case, rows=rows)
    assert row_rel_err(y[rows], ref) <= 1e-2


def test_ep_c_abi_nccl_world1(mx):
    """mxm_ep_init / mxm_ep_moe_group_gemm on a real NCCL communicator (torch ProcessGroupNCCL, world size 1 on the
    one reachable GPU): the library's own NCCL dispatch / combine path equals the torch-orchestrated EP path bitwise
    (same kernels, same order), matches the oracle, and reports bad expert ids through its error word."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2505_05799_b200.ep import CAbiExpertParallelMoE, ExpertParallelMoE
    if not dist.is_initialized():
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    cfg = C.LayerConfig("ep1", 8, 1, 256, 512, 384, 2, 96)
    table = ([[C.WA(4, 128)] * 3] * 3 + [[C.WO(4, 128)] * 3] * 3 + [[C.WA(8, -1)] * 3] * 2 + [[C.WO(2, -1)] * 3])
    case = make_case(cfg, table, 96, seed=12)
    W = [[bf16_tensor(b) for b in blk] for blk in case["weights"]]
    py = ExpertParallelMoE.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, W, table)
    cab = CAbiExpertParallelMoE(py.local, py.shared, cfg.n_routed)
    x = bf16_tensor(case["x"])
    ids = torch.from_numpy(case["ids"]).cuda()
    w = torch.from_numpy(case["w"]).cuda()
    sw = torch.from_numpy(case["shared_w"]).cuda()
    y_py = py(x, ids, w, sw)  # torch orchestration, sync-free
    py.sync_free = False
    y_v1 = py(x, ids, w, sw)  # torch orchestration, v1
    y_c = cab(x, ids, w, sw)  # C ABI, sync-free (default)
    cab.set_sync_free(False)
    y_c1 = cab(x, ids, w, sw)  # C ABI, v1
    cab.set_sync_free(True)
    torch.cuda.synchronize()
    assert torch.equal(y_py, y_c) and torch.equal(y_v1, y_c) and torch.equal(y_c1, y_c)
    ref = oracle_run(oracle_layer(case), case)
    assert row_rel_err(y_c.float().cpu().numpy().astype(np.float64), ref) <= 1e-2
    assert cab.poll_error() == 0
    bad = ids.clone()
    bad[3, 0] = 99
    cab(x, bad, w, sw)
    assert cab.poll_error() == 4
    del cab, py
    dist.destroy_process_group()
