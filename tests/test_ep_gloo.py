"""Expert-parallel orchestration over 2 ranks with the gloo backend on CPU (not gpu).

The host logic of paper_2505_05799_b200/ep.py (count exchange, split sizes, all-to-all-v of rows and
metadata, reverse exchange, fixed-order combine, replicated shared experts) is run for real across two
processes. The device kernels are replaced by a plain torch reference of their documented index
semantics (include/mxmoe.h, mxm_ep_*) and the per-rank layers by the oracle, so the test checks that
the sharded block equals the unsharded oracle block (Eq. 2 is a sum over experts).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import configs as C


class TorchRefEpOps:
    """Plain-torch reference of mxm_ep_route / mxm_ep_pack / mxm_ep_combine (CPU tensors)."""

    def route(self, ids, E, G):
        T, k = ids.shape
        epr = E // G
        has = torch.zeros(T, G, dtype=torch.bool)
        for r in range(G):
            has[:, r] = ((ids >= 0) & (ids // epr == r)).any(1)
        pos = torch.full((T, G), -1, dtype=torch.int32)
        counts = torch.zeros(G, dtype=torch.int32)
        for r in range(G):
            n = 0
            for t in range(T):
                if has[t, r]:
                    pos[t, r] = n
                    n += 1
            counts[r] = n
        return counts, pos

    def pack(self, x, ids, w, pos, dest_off, E, G, S_total):
        T, k = ids.shape
        epr = E // G
        sx = torch.zeros(S_total, x.shape[1], dtype=x.dtype)
        sids = torch.full((S_total, k), -1, dtype=torch.int32)
        sw = torch.zeros(S_total, k, dtype=torch.float32)
        ssrc = torch.zeros(S_total, dtype=torch.int32)
        for t in range(T):
            for r in range(G):
                p = int(pos[t, r])
                if p < 0:
                    continue
                row = int(dest_off[r]) + p
                sx[row] = x[t]
                for j in range(k):
                    e = int(ids[t, j])
                    if e >= 0 and e // epr == r:
                        sids[row, j] = e - r * epr
                        sw[row, j] = w[t, j]
                ssrc[row] = t
        return sx, sids, sw, ssrc

    def combine(self, back, pos, dest_off, G, ysh, T, d):
        y = torch.zeros(T, d, dtype=torch.float32)
        for t in range(T):
            for r in range(G):
                p = int(pos[t, r])
                if p >= 0:
                    y[t] += back[int(dest_off[r]) + p].float()
        if ysh is not None:
            y += ysh.float()
        return y.to(torch.bfloat16)


def _bits(t):
    return t.view(torch.int16).numpy().view(np.uint16)


class OracleLayer:
    """Per-rank layer backed by the oracle (fp64), returning bf16 like the device layer."""

    def __init__(self, qlayer):
        self.q = qlayer

    def __call__(self, x, ids, w):
        from oracle.moe import moe_block
        y = moe_block(_bits(x), self.q, ids.numpy(), w.numpy())
        return torch.from_numpy(y.astype(np.float32)).to(torch.bfloat16)


def _case():
    from tests.moe_cases import make_case
    cfg = C.LayerConfig("tiny_s", 4, 1, 128, 256, 384, 2, 24)
    table = C.precision_table(C.get_config("tiny")) + [[C.WO(4, 64), C.WA(8, -1), C.WO(8, -1)]]
    return cfg, table, make_case(cfg, table, 24, seed=3)


def _placed_case(case, table, cfg, world):
    """The same block with an LPT expert placement (placement.py): experts re-indexed, ids mapped."""
    from paper_2505_05799_b200.placement import apply_placement, inverse, lpt_placement
    ids = case["ids"]
    loads = np.bincount(ids[ids >= 0], minlength=cfg.n_routed).astype(float)
    perm = lpt_placement(loads, world)
    w2, t2 = apply_placement(case["weights"], table, perm, cfg.n_routed)
    inv = inverse(perm)
    c2 = dict(case, weights=w2, ids=np.where(ids >= 0, inv[np.maximum(ids, 0)], -1).astype(np.int32))
    return c2, t2


def _worker(rank, world, port, out_path, placed=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.moe import QuantizedLayer, quantize_layer
    from paper_2505_05799_b200.ep import ExpertParallelMoE

    cfg, table, case = _case()
    if placed:
        case, table = _placed_case(case, table, cfg, world)
    full = quantize_layer(case["weights"], table, cfg.n_routed, cfg.n_shared)
    epr = cfg.n_routed // world
    lo = rank * epr
    local = QuantizedLayer(epr, 0, cfg.hidden, cfg.inter, 0, full.blocks[lo:lo + epr])
    shared = QuantizedLayer(cfg.n_shared, 0, cfg.hidden, cfg.shared_inter, 0, full.blocks[cfg.n_routed:])
    eps = {mode: ExpertParallelMoE(cfg.n_routed, cfg.hidden, OracleLayer(local), OracleLayer(shared), cfg.n_shared,
                                   ops=TorchRefEpOps(), sync_free=mode == "sync_free")
           for mode in ("v1", "sync_free")}
    # each rank owns a different slice of the tokens (data parallel), routing is global
    T = case["T"]
    sl = slice(rank * T // world, (rank + 1) * T // world)
    x = torch.from_numpy(case["x"][sl].view(np.int16)).view(torch.bfloat16)
    ids = torch.from_numpy(case["ids"][sl].astype(np.int32))
    w = torch.from_numpy(case["w"][sl])
    sw = torch.from_numpy(case["shared_w"][sl])
    for mode, ep in eps.items():
        y = ep(x, ids, w, sw)
        np.save(f"{out_path}_{mode}_{rank}.npy", y.float().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_ep_two_ranks_equals_unsharded_oracle(tmp_path, world):
    out = str(tmp_path / "y")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    y = np.concatenate([np.load(f"{out}_v1_{r}.npy") for r in range(world)])
    # the sync-free exchange (fixed capacity, padding rows without routes) gives the same bits as v1
    y_sf = np.concatenate([np.load(f"{out}_sync_free_{r}.npy") for r in range(world)])
    assert np.array_equal(y, y_sf)
    from oracle.moe import moe_block, quantize_layer
    from tests.moe_cases import row_rel_err
    cfg, table, case = _case()
    ref = moe_block(case["x"], quantize_layer(case["weights"], table, cfg.n_routed, cfg.n_shared), case["ids"],
                    case["w"], case["shared_w"])
    assert row_rel_err(y.astype(np.float64), ref) <= 1e-2


def test_ep_two_ranks_lpt_placement(tmp_path):
    """LPT-placed experts over 2 gloo ranks (sync-free exchange) = the unsharded block with the original order."""
    world = 2
    out = str(tmp_path / "yp")
    mp.spawn(_worker, args=(world, _free_port(), out, True), nprocs=world, join=True)
    y = np.concatenate([np.load(f"{out}_sync_free_{r}.npy") for r in range(world)])
    from oracle.moe import moe_block, quantize_layer
    from tests.moe_cases import row_rel_err
    cfg, table, case = _case()
    ref = moe_block(case["x"], quantize_layer(case["weights"], table, cfg.n_routed, cfg.n_shared), case["ids"],
                    case["w"], case["shared_w"])
    assert row_rel_err(y.astype(np.float64), ref) <= 1e-2


def test_ref_ops_route_semantics():
    ops = TorchRefEpOps()
    ids = torch.tensor([[0, 3], [1, 1], [2, -1], [3, 0]], dtype=torch.int32)
    counts, pos = ops.route(ids, 4, 2)
    assert counts.tolist() == [3, 3]  # rank 0 (experts 0,1): tokens 0,1,3; rank 1 (2,3): tokens 0,2,3
    assert pos.tolist() == [[0, 0], [1, -1], [-1, 1], [2, 2]]
