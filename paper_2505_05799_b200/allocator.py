"""Host-side bit allocation of MxMoE (§4.2, Eq. 7).

Chooses one quantization scheme per linear block (expert i, block j) to minimise L^r · T^(1-r) under a memory
budget (Eq. 7):
    L = Σ Δ[i,j,k] x[i,j,k]                    quantization loss (Δ = ||Ô − O||_2, Eq. 6)
    T = (1/P) Σ c[i,j,k] x[i,j,k]              serial tile time over P SMs, c from the measured
                                                single-tile costs of THIS GPU (mxm_profile_tile_costs)
    Σ_k x[i,j,k] = 1,  Σ W[i,j,k] x[i,j,k] <= M  (bytes)
The product objective is handled exactly on a grid of time budgets: for each budget T_b the mixed-integer
program min L s.t. T <= T_b, memory <= M (a multiple-choice knapsack) is solved with scipy's HiGHS MILP, and
the candidate with the smallest L^r T^(1-r) wins (the optimum lies on the L-vs-T Pareto front, which the
budget grid samples). The allocation is a host input of the hot path (north star); nothing here runs on the
GPU except the measurements that produce Δ and c (`measure_costs`, `measure_deltas`).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np


@dataclass
class Problem:
    delta: np.ndarray   # [B, K] loss of block b under scheme k (B = experts * 3 linear blocks)
    cost: np.ndarray    # [B, K] serial tile time (any unit) of block b under scheme k
    weight: np.ndarray  # [B, K] bytes of block b under scheme k
    budget: float       # memory budget M (bytes)
    n_sm: int = 148     # P


@dataclass
class Allocation:
    choice: np.ndarray  # [B] scheme index per block
    L: float
    T: float
    M: float


def _evaluate(p: Problem, choice: np.ndarray) -> Allocation:
    b = np.arange(len(choice))
    return Allocation(choice, float(p.delta[b, choice].sum()), float(p.cost[b, choice].sum() / p.n_sm),
                      float(p.weight[b, choice].sum()))


def _milp_min_loss(p: Problem, t_budget: float) -> Optional[np.ndarray]:
    """min Σ Δ x  s.t. one scheme per block, Σ c x / P <= t_budget, Σ W x <= M, x binary (HiGHS)."""
    from scipy.optimize import Bounds, LinearConstraint, milp
    from scipy.sparse import csr_matrix
    B, K = p.delta.shape
    n = B * K
    rows = np.repeat(np.arange(B), K)
    one = csr_matrix((np.ones(n), (rows, np.arange(n))), shape=(B, n))
    cons = [LinearConstraint(one, 1, 1),
            LinearConstraint(p.cost.reshape(1, n) / p.n_sm, -np.inf, t_budget),
            LinearConstraint(p.weight.reshape(1, n), -np.inf, p.budget)]
    res = milp(c=p.delta.reshape(n), constraints=cons, integrality=np.ones(n), bounds=Bounds(0, 1))
    if res.status != 0 or res.x is None:
        return None
    return np.argmax(res.x.reshape(B, K), axis=1)


def allocate(p: Problem, r: float, n_budgets: int = 24) -> Allocation:
    """Eq. 7: the allocation minimising L^r · T^(1-r) subject to the memory budget."""
    B, K = p.delta.shape
    b = np.arange(B)
    # time range of feasible allocations: fastest-per-block (ignoring memory) up to slowest
    t_lo = p.cost.min(axis=1).sum() / p.n_sm
    t_hi = p.cost.max(axis=1).sum() / p.n_sm
    best: Optional[Allocation] = None
    for tb in np.linspace(t_lo, t_hi, n_budgets):
        ch = _milp_min_loss(p, float(tb) * (1 + 1e-9))
        if ch is None:
            continue
        a = _evaluate(p, ch)
        obj = (a.L ** r) * (a.T ** (1 - r))
        if best is None or obj < (best.L ** r) * (best.T ** (1 - r)) - 1e-15:
            best = a
    if best is None:
        raise ValueError("no allocation fits the memory budget")
    return best


def brute_force(p: Problem, r: float) -> Allocation:
    """Exhaustive search (tests / tiny problems only)."""
    import itertools
    B, K = p.delta.shape
    best = None
    for ch in itertools.product(range(K), repeat=B):
        a = _evaluate(p, np.array(ch))
        if a.M > p.budget:
            continue
        obj = (a.L ** r) * (a.T ** (1 - r))
        if best is None or obj < (best.L ** r) * (best.T ** (1 - r)) - 1e-15:
            best = a
    return best


# ---------------------------------------------------------------- measurements on the GPU (inputs of Eq. 7)
def measure_costs(mx, hidden: int, inter: int, schemes: Sequence, expert_tokens: Sequence[int]) -> np.ndarray:
    """c[i, k]: serial time (ms) of one linear block of expert i under scheme k, from measured m-tile group
    costs of THIS GPU (mxm_profile_tile_costs on a one-expert probe layer per scheme): the expert's
    m-tiles at its expected token count times the group cost at the matching token tile, / 3 blocks."""
    import torch
    from synth.gen import gen_weight
    W = [[torch.from_numpy(gen_weight(inter, hidden, 7000 + j).view(np.int16)).view(torch.bfloat16).cuda()
          if j < 2 else torch.from_numpy(gen_weight(hidden, inter, 7002).view(np.int16)).view(torch.bfloat16).cuda()
          for j in range(3)]]
    tiles = [16, 32, 64, 96]
    per_scheme = []
    for s in schemes:
        lay = mx.MoELayer.from_weights(1, 0, hidden, inter, 0, W, [[mx.Scheme.of(s)] * 3])
        per_scheme.append(lay.profile_tile_costs()[0])  # [4] ms per m-tile group of the whole expert
        del lay
    out = np.zeros((len(expert_tokens), len(schemes)))
    for i, m in enumerate(expert_tokens):
        for k, s in enumerate(schemes):
            if m <= 0:
                continue
            cap = 96 if (s.a_bits == 16 or s.w_group == -1) else 64
            full, rem = divmod(int(m), cap)
            c = full * per_scheme[k][3 if cap == 96 else 2]
            if rem:
                ti = next(t for t in range(4) if tiles[t] >= rem)
                c += per_scheme[k][ti]
            out[i, k] = c / 3.0
    return out


def measure_deltas(mx, weights, schemes: Sequence, x_cal, freq: Sequence[float]) -> np.ndarray:
    """Δ[b, k] = p_i · ||Ô − O||_2 for linear block b = (i, j) quantized alone with scheme k (Eq. 6),
    on calibration inputs: gate/up see x_cal, down sees the full-precision expert's h. The weights are
    quantized / dequantized by the library (mxm_quantize / mxm_pack / mxm_dequantize); weight-activation schemes
    also quantize the block input with the hot path's activation quantizer (mxm_act_quant)."""
    import torch
    out = []
    for i, blk in enumerate(weights):
        wg, wu, wd = [w.float() for w in blk]
        g, u = x_cal.float() @ wg.T, x_cal.float() @ wu.T
        h = (torch.nn.functional.silu(g) * u).to(torch.bfloat16)
        for j, (w, xin) in enumerate(((blk[0], x_cal), (blk[1], x_cal), (blk[2], h))):
            ref = xin.float() @ w.float().T
            row = []
            for s in schemes:
                N, K = w.shape
                if s.w_bits == 16:
                    row.append(0.0)
                    continue
                packed = mx.quantize_pack(s, w.contiguous())
                wq = mx.dequantize(s, packed, N, K)
                xq = xin.float()
                if s.a_bits != 16:
                    codes, sc, _ = mx.act_quant(xin.contiguous(), s.a_bits, s.a_group)
                    g_ = K if s.a_group == -1 else s.a_group
                    xq = (codes.float().view(-1, K // g_, g_) * sc.view(-1, K // g_, 1)).view(-1, K)
                row.append(float(freq[i]) * float(torch.linalg.norm(xq @ wq.T - ref)))
            out.append(row)
    return np.array(out)
