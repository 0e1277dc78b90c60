"""Eq. 7 allocator (NEXT-2), host side: exact against brute force on small instances,
constraints, and the direction of the r trade-off (P:384 fig:ablation-r: larger r favours accuracy)."""
import numpy as np
import pytest

from paper_2505_05799_b200.allocator import Problem, allocate, brute_force


def _rand_problem(seed, B=5, K=4, slack=0.6):
    rng = np.random.default_rng(seed)
    bits = np.array([2.25, 4.25, 8.0, 16.0])[:K]
    delta = np.outer(rng.uniform(0.5, 2.0, B), 2.0 ** (-bits)) * rng.uniform(0.8, 1.2, (B, K))
    cost = np.outer(rng.uniform(0.5, 2.0, B), np.array([1.0, 1.3, 0.7, 1.6])[:K]) * rng.uniform(0.9, 1.1, (B, K))
    weight = np.outer(rng.uniform(1, 3, B), bits)
    budget = weight.min(axis=1).sum() + slack * (weight.max(axis=1).sum() - weight.min(axis=1).sum())
    return Problem(delta, cost, weight, budget, n_sm=2)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("r", [0.0, 0.5, 0.75, 1.0])
def test_matches_brute_force(seed, r):
    p = _rand_problem(seed)
    a, b = allocate(p, r, n_budgets=64), brute_force(p, r)
    assert a.M <= p.budget + 1e-9
    obj = lambda x: (x.L ** r) * (x.T ** (1 - r))
    assert obj(a) <= obj(b) * (1 + 1e-6) + 1e-12, (obj(a), obj(b))


def test_extremes_and_direction():
    p = _rand_problem(11, B=6)
    fast, acc = allocate(p, 0.0), allocate(p, 1.0)
    # r = 0: the fastest allocation that fits; r = 1: the most accurate one
    assert fast.T <= min(allocate(p, r).T for r in (0.25, 0.5, 0.75, 1.0)) + 1e-12
    assert acc.L <= min(allocate(p, r).L for r in (0.0, 0.25, 0.5, 0.75)) + 1e-12
    Ls = [allocate(p, r).L for r in (0.0, 0.5, 0.75, 1.0)]
    assert all(Ls[i + 1] <= Ls[i] + 1e-12 for i in range(len(Ls) - 1))


def test_memory_budget_binds():
    p = _rand_problem(3, slack=0.0)  # only the smallest scheme of every block fits
    a = allocate(p, 1.0)
    assert np.array_equal(a.choice, p.weight.argmin(axis=1))
