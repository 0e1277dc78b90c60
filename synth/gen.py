"""Seeded generators (inputs only; see synth/__init__.py)."""
from __future__ import annotations

import numpy as np
import torch


def bf16_bits_from_f32(a: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 (via torch's conversion) and return uint16 bit patterns."""
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16).copy()


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """Decode uint16 bf16 bit patterns to float64 (exact)."""
    u = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def gen_activations(T: int, d: int, seed: int = 1, heavy_tailed: bool = False) -> np.ndarray:
    """x[T, d] as bf16 bits. N(0,1); heavy_tailed: Student-t(3) with 1% channels x20."""
    g = torch.Generator().manual_seed(seed)
    if not heavy_tailed:
        x = torch.randn(T, d, generator=g, dtype=torch.float32)
    else:
        n = torch.randn(T, d, generator=g, dtype=torch.float32)
        chi = torch.zeros(T, d)
        for _ in range(3):
            chi += torch.randn(T, d, generator=g) ** 2
        x = n / torch.sqrt(chi / 3.0)
        n_out = max(1, d // 100)
        ch = torch.randperm(d, generator=g)[:n_out]
        x[:, ch] *= 20.0
    return x.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16).copy()


def gen_weight(N: int, K: int, seed: int) -> np.ndarray:
    """W[N, K] ~ N(0, 1/K) as bf16 bits."""
    g = torch.Generator().manual_seed(seed)
    w = torch.randn(N, K, generator=g, dtype=torch.float32) * (1.0 / np.sqrt(K))
    return w.to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16).copy()


def weight_seed(expert: int, block: int) -> int:
    return 1000 + 3 * expert + block


def gen_routing(T: int, E: int, k: int, s: float = 0.8, seed: int = 0):
    """Zipf-skewed Gumbel-top-k routing.

    Returns (topk_ids int32[T,k], topk_w float32[T,k]). Experts within a token are
    distinct; weights are the softmax over the k selected perturbed logits.
    """
    rng = np.random.default_rng(seed)
    perm = rng.permutation(E)
    ranks = np.empty(E, dtype=np.float64)
    ranks[perm] = np.arange(1, E + 1, dtype=np.float64)
    logp = -s * np.log(ranks)  # log p_e up to a constant
    gumbel = -np.log(-np.log(rng.random((T, E)).clip(1e-300, 1.0)))
    logits = logp[None, :] + gumbel
    # top-k with ties -> lower id: stable argsort on -logits
    order = np.argsort(-logits, axis=1, kind="stable")[:, :k]
    sel = np.take_along_axis(logits, order, axis=1)
    sel = sel - sel.max(axis=1, keepdims=True)
    w = np.exp(sel)
    w = w / w.sum(axis=1, keepdims=True)
    return order.astype(np.int32), w.astype(np.float32)


def gen_shared_weights(T: int, S: int, seed: int = 2) -> np.ndarray:
    """Per-token shared-expert weights in (0, 1] (the caller's sigmoid gate); float32[T, S]."""
    rng = np.random.default_rng(seed)
    return (1.0 / (1.0 + np.exp(-rng.standard_normal((T, S))))).astype(np.float32)
