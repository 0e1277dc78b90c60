"""Seeded MoE test cases shared by the GPU parity tests (inputs from synth/, nothing computed here)."""
from __future__ import annotations

import numpy as np
import torch

from synth import configs as C
from synth.gen import gen_activations, gen_routing, gen_shared_weights, gen_weight, weight_seed


def bf16_tensor(bits: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(device)


def make_case(cfg: C.LayerConfig, table, T: int, seed: int = 0, heavy: bool = False, k: int = None,
              routing_s: float = 0.8):
    E, S = cfg.n_routed, cfg.n_shared
    k = cfg.top_k if k is None else k
    weights = []
    for v in range(E + S):
        f = cfg.inter if v < E else cfg.shared_inter
        weights.append([gen_weight(f, cfg.hidden, weight_seed(v, 0)), gen_weight(f, cfg.hidden, weight_seed(v, 1)),
                        gen_weight(cfg.hidden, f, weight_seed(v, 2))])
    x = gen_activations(T, cfg.hidden, seed=1 + seed, heavy_tailed=heavy)
    ids, w = gen_routing(T, E, k, s=routing_s, seed=seed)
    sw = gen_shared_weights(T, S) if S else None
    return dict(cfg=cfg, table=table, weights=weights, x=x, ids=ids, w=w, shared_w=sw, T=T, k=k)


def gpu_layer(case):
    import paper_2505_05799_b200 as mx
    cfg = case["cfg"]
    W = [[bf16_tensor(b) for b in blk] for blk in case["weights"]]
    tab = [[mx.Scheme.of(s) for s in row] for row in case["table"]]
    return mx.MoELayer.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, W, tab)


def gpu_run(layer, case, ids=None, w=None):
    ids = case["ids"] if ids is None else ids
    w = case["w"] if w is None else w
    x = bf16_tensor(case["x"])
    sw = None if case["shared_w"] is None else torch.from_numpy(case["shared_w"]).cuda()
    y = layer(x, torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)).cuda(),
              torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32)).cuda(), sw)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


def oracle_layer(case):
    from oracle.moe import quantize_layer
    cfg = case["cfg"]
    return quantize_layer(case["weights"], case["table"], cfg.n_routed, cfg.n_shared)


def oracle_run(olayer, case, rows=None, ids=None, w=None):
    from oracle.moe import moe_block
    ids = case["ids"] if ids is None else ids
    w = case["w"] if w is None else w
    x, sw = case["x"], case["shared_w"]
    if rows is not None:
        x, ids, w = x[rows], ids[rows], w[rows]
        sw = None if sw is None else sw[rows]
    return moe_block(x, olayer, ids, w, sw)


def row_rel_err(y, ref):
    """max_t max_i |y - ref| / max_i |ref|  (R19 gate metric)."""
    den = np.maximum(np.abs(ref).max(axis=1), 1e-30)
    return float((np.abs(y - ref).max(axis=1) / den).max())
