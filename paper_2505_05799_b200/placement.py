"""LPT expert placement for expert parallelism ("LPT expert placement").

Rank r of G owns the routed experts at positions [r·E/G, (r+1)·E/G) of the layer's expert order (ep.py). With
Zipf-skewed routing (">10x" activation-frequency spread) the contiguous default puts hot experts together;
a placement is a permutation of the expert order chosen so that every rank's expected load is balanced. It is
applied offline, like the bit allocation: the experts' weights / precision table are reordered and the caller's
router emits ids in the new order (its gate columns permuted the same way), so the hot path is unchanged and
the block output is identical (Eq. 2 is a sum over experts). Host-side planning code, no device work.

lpt_placement: longest-processing-time list scheduling with a cardinality constraint (each rank exactly E/G
experts): experts by expected load, descending, each to the least-loaded rank that still has room.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def lpt_placement(loads: Sequence[float], G: int) -> np.ndarray:
    """perm[new_position] = old expert id; rank r owns new positions [r·E/G, (r+1)·E/G)."""
    loads = np.asarray(loads, dtype=np.float64)
    E = loads.shape[0]
    if G <= 0 or E % G:
        raise ValueError("the number of experts must be divisible by the number of ranks")
    per = E // G
    order = sorted(range(E), key=lambda e: (-loads[e], e))
    rank_load = np.zeros(G)
    members: List[List[int]] = [[] for _ in range(G)]
    for e in order:
        open_ranks = [r for r in range(G) if len(members[r]) < per]
        r = min(open_ranks, key=lambda q: (rank_load[q], q))
        members[r].append(e)
        rank_load[r] += loads[e]
    return np.array([e for r in range(G) for e in sorted(members[r])], dtype=np.int64)


def rank_loads(loads: Sequence[float], perm: Sequence[int], G: int) -> np.ndarray:
    """Expected load of each rank under a placement (perm[new] = old)."""
    loads = np.asarray(loads, dtype=np.float64)
    per = len(perm) // G
    return np.array([loads[np.asarray(perm[r * per:(r + 1) * per])].sum() for r in range(G)])


def inverse(perm: Sequence[int]) -> np.ndarray:
    """new_id[old] for remapping router ids (the caller's router permutes its gate columns by perm)."""
    perm = np.asarray(perm, dtype=np.int64)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    return inv


def apply_placement(weights: Sequence, table: Sequence, perm: Sequence[int], n_routed: int) -> Tuple[list, list]:
    """Reorder the routed experts' weights / precision rows (shared experts, after n_routed, stay in place)."""
    perm = list(perm)
    w = [weights[p] for p in perm] + list(weights[n_routed:])
    t = [table[p] for p in perm] + list(table[n_routed:])
    return w, t
