"""LPT expert placement (NEXT-1 part; paper_2505_05799_b200/placement.py): a valid permutation with E/G experts per
rank, better balance than the contiguous default on the synthetic Zipf loads, within 4/3 of the brute-force
optimum on small cases, and an exact re-indexing of the block (the oracle gives bit-identical outputs)."""
import itertools

import numpy as np
import pytest

from paper_2505_05799_b200.placement import apply_placement, inverse, lpt_placement, rank_loads
from synth import configs as C


@pytest.mark.parametrize("name,G", [("dsv2", 8), ("q2", 8), ("q15", 4), ("mx", 2)])
def test_lpt_valid_and_better_than_contiguous(name, G):
    cfg = C.get_config(name)
    loads = C.zipf_popularity(cfg.n_routed, 0.8, seed=0)
    perm = lpt_placement(loads, G)
    assert sorted(perm.tolist()) == list(range(cfg.n_routed))
    rl = rank_loads(loads, perm, G)
    rc = rank_loads(loads, np.arange(cfg.n_routed), G)
    assert rl.max() <= rc.max() + 1e-12
    assert rl.max() <= loads.sum() / G + loads.max() + 1e-12  # list-scheduling bound
    # within 10 % of a lower bound on the optimum: the mean, or the hottest expert plus the E/G - 1 coldest
    per = cfg.n_routed // G
    lb = max(loads.sum() / G, loads.max() + np.sort(loads)[:per - 1].sum())
    assert rl.max() <= 1.10 * lb


def test_lpt_within_four_thirds_of_optimum():
    rng = np.random.default_rng(0)
    for _ in range(30):
        E, G = 6, 2 if rng.random() < 0.5 else 3
        loads = rng.pareto(1.2, E) + 0.05
        perm = lpt_placement(loads, G)
        got = rank_loads(loads, perm, G).max()
        per = E // G
        best = np.inf
        for p in itertools.permutations(range(E)):
            if any(list(p[r * per:(r + 1) * per]) != sorted(p[r * per:(r + 1) * per]) for r in range(G)):
                continue
            best = min(best, rank_loads(loads, p, G).max())
        assert got <= 4 / 3 * best + 1e-12


def test_placement_is_an_exact_reindexing():
    """moe_block on the placed layer with ids remapped through inverse(perm) = the original block, bitwise."""
    from oracle.moe import moe_block, quantize_layer
    from tests.moe_cases import make_case
    cfg = C.LayerConfig("plc", 8, 1, 128, 256, 256, 2, 24)
    table = [[C.WO(4, 64)] * 3, [C.WA(8, -1)] * 3, [C.WO(2, 128)] * 3, [C.WA(4, 128)] * 3, [C.W16] * 3,
             [C.WO(3, 128)] * 3, [C.FP8(-1)] * 3, [C.WA(4, -1)] * 3, [C.WO(8, -1, True)] * 3]
    case = make_case(cfg, table, 24, seed=4)
    loads = np.bincount(case["ids"].reshape(-1)[case["ids"].reshape(-1) >= 0], minlength=8).astype(float)
    perm = lpt_placement(loads, 2)
    w2, t2 = apply_placement(case["weights"], table, perm, 8)
    inv = inverse(perm)
    ids2 = np.where(case["ids"] >= 0, inv[np.maximum(case["ids"], 0)], -1).astype(np.int32)
    y = moe_block(case["x"], quantize_layer(case["weights"], table, 8, 1), case["ids"], case["w"], case["shared_w"])
    y2 = moe_block(case["x"], quantize_layer(w2, t2, 8, 1), ids2, case["w"], case["shared_w"])
    assert np.array_equal(y, y2)
