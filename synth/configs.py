"""Layer configs of BASELINE.json and their per-(expert, block) precision tables.

Shapes: PAPER.md Table `tab:exp-model` + public model configs as
restated in SURVEY.md §8(d). Precision tables: SURVEY.md §8(d) "Configs";
Qwen1.5 uses PAPER.md Table `tab:w5a5-scheme` verbatim.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


@dataclass(frozen=True)
class Scheme:
    """`wxay_gz_{sym,asym}`. a_bits=16 -> weight-only; w_bits=16 -> bf16."""

    w_bits: int
    a_bits: int = 16
    w_group: int = -1
    a_group: int = -1
    symmetric: bool = False
    fmt: int = 0  # 0: integer codes (the paper's quantizer); 1: FP8 e4m3 weights and activations (NEXT-4, R25/R26)

    @property
    def weight_only(self) -> bool:
        return self.a_bits == 16

    def name(self) -> str:
        if self.w_bits == 16:
            return "w16a16"
        g = self.w_group
        s = "sym" if self.symmetric else "asym"
        if self.weight_only:
            return f"w{self.w_bits}a16_g{g}_{s}"
        if self.fmt == 1:
            return f"fp8_e4m3_g{g}"
        return f"w{self.w_bits}a{self.a_bits}_g{g}_{s}"


W16 = Scheme(16, 16, -1, -1, True)


def WO(bits: int, group: int = 128, sym: bool = False) -> Scheme:
    return Scheme(bits, 16, group, -1, sym)


def WA(bits: int, group: int = -1) -> Scheme:
    return Scheme(bits, bits, group, group, True)


def FP8(group: int = -1) -> Scheme:
    """FP8 e4m3 weights and activations (NEXT-4 extra hardware-supported scheme; DESIGN R25/R26)."""
    return Scheme(8, 8, group, group, True, 1)


@dataclass
class LayerConfig:
    name: str
    n_routed: int
    n_shared: int
    hidden: int
    inter: int
    shared_inter: int
    top_k: int
    tokens: int
    sweep: List[int] = field(default_factory=list)
    desc: str = ""


CONFIGS = {
    "tiny": LayerConfig("tiny", 4, 0, 128, 256, 0, 2, 64, desc="tiny MoE layer, mixed w4a16-g64/w8a8"),
    "dsv2": LayerConfig("dsv2", 64, 2, 2048, 1408, 1408, 6, 4096, [512, 4096],
                        desc="DeepSeek-V2-Lite MoE layer, mixed w2/w3/w4 weight-only (2.25-bit avg)"),
    "q15": LayerConfig("q15", 60, 1, 2048, 1408, 5632, 4, 8192, [512, 8192],
                       desc="Qwen1.5-MoE-A2.7B layer, Table-6 w4a4/w8a8 (5-bit avg W-A)"),
    "mx": LayerConfig("mx", 8, 0, 4096, 14336, 0, 2, 512,
                      [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384],
                      desc="Mixtral-8x7B layer, w4a16/w8a8 by expected load"),
    "q2": LayerConfig("q2", 64, 1, 3584, 2560, 20480, 8, 16384, [16384],
                      desc="Qwen2-57B-A14B layer, W-A mix, expert parallel"),
}


def get_config(name: str) -> LayerConfig:
    return CONFIGS[name]


# PAPER.md Table `tab:w5a5-scheme`, Qwen1.5-MoE layer 5, verbatim.
# Columns: expert | gate w-act, w_gsize, a_gsize | up ... | down ...
TABLE6 = """
0 4-4 128 128 4-4 128 128 4-4 128 128
1 4-4 128 128 4-4 128 128 8-8 -1 -1
2 4-4 128 128 4-4 128 128 8-8 -1 -1
3 4-4 128 128 4-4 128 128 8-8 -1 -1
4 4-4 -1 -1 4-4 -1 -1 4-4 128 128
5 4-4 128 128 4-4 128 128 4-4 128 128
6 4-4 128 128 4-4 128 128 8-8 -1 -1
7 4-4 -1 -1 4-4 -1 -1 4-4 128 128
8 4-4 128 128 4-4 128 128 8-8 -1 -1
9 4-4 128 128 4-4 128 128 8-8 -1 -1
10 4-4 128 128 4-4 128 128 8-8 -1 -1
11 4-4 128 128 4-4 128 128 8-8 -1 -1
12 4-4 128 128 4-4 128 128 8-8 -1 -1
13 4-4 128 128 4-4 128 128 4-4 128 128
14 4-4 -1 -1 4-4 -1 -1 4-4 128 128
15 4-4 128 128 4-4 128 128 8-8 -1 -1
16 4-4 128 128 4-4 128 128 8-8 -1 -1
17 4-4 128 128 4-4 128 128 8-8 -1 -1
18 4-4 128 128 4-4 128 128 8-8 -1 -1
19 4-4 128 128 4-4 128 128 8-8 -1 -1
20 4-4 128 128 4-4 128 128 4-4 128 128
21 4-4 128 128 4-4 128 128 8-8 -1 -1
22 8-8 -1 -1 8-8 -1 -1 8-8 -1 -1
23 4-4 128 128 4-4 128 128 4-4 128 128
24 4-4 128 128 4-4 128 128 8-8 -1 -1
25 4-4 128 128 4-4 128 128 4-4 128 128
26 4-4 128 128 4-4 128 128 8-8 -1 -1
27 4-4 128 128 4-4 128 128 4-4 128 128
28 4-4 128 128 4-4 128 128 8-8 -1 -1
29 4-4 128 128 4-4 128 128 4-4 128 128
30 4-4 128 128 4-4 128 128 4-4 128 128
31 4-4 128 128 4-4 128 128 8-8 -1 -1
32 4-4 128 128 4-4 128 128 4-4 128 128
33 4-4 128 128 4-4 128 128 4-4 128 128
34 4-4 128 128 4-4 128 128 8-8 -1 -1
35 4-4 128 128 4-4 128 128 8-8 -1 -1
36 4-4 128 128 4-4 128 128 8-8 -1 -1
37 4-4 128 128 4-4 128 128 8-8 -1 -1
38 4-4 128 128 4-4 128 128 8-8 -1 -1
39 4-4 128 128 4-4 128 128 4-4 128 128
40 4-4 128 128 4-4 128 128 4-4 128 128
41 4-4 128 128 4-4 128 128 8-8 -1 -1
42 4-4 128 128 4-4 128 128 8-8 -1 -1
43 4-4 128 128 4-4 128 128 8-8 -1 -1
44 4-4 -1 -1 4-4 -1 -1 4-4 128 128
45 4-4 128 128 4-4 128 128 8-8 -1 -1
46 4-4 128 128 4-4 128 128 8-8 -1 -1
47 4-4 128 128 4-4 128 128 4-4 128 128
48 4-4 128 128 4-4 128 128 8-8 -1 -1
49 4-4 128 128 4-4 128 128 8-8 -1 -1
50 4-4 128 128 4-4 128 128 4-4 128 128
51 4-4 128 128 4-4 128 128 4-4 128 128
52 4-4 128 128 4-4 128 128 8-8 -1 -1
53 4-4 128 128 4-4 128 128 4-4 128 128
54 4-4 -1 -1 4-4 -1 -1 4-4 128 128
55 4-4 -1 -1 4-4 -1 -1 4-4 128 128
56 4-4 -1 -1 4-4 -1 -1 4-4 128 128
57 4-4 128 128 4-4 128 128 4-4 128 128
58 4-4 -1 -1 4-4 -1 -1 4-4 128 128
59 4-4 128 128 4-4 128 128 8-8 -1 -1
60 4-4 -1 -1 4-4 -1 -1 8-8 -1 -1
"""


def parse_table6() -> List[List[Scheme]]:
    rows = []
    for line in TABLE6.strip().splitlines():
        f = line.split()
        blocks = []
        for j in range(3):
            wa, wg, ag = f[1 + 3 * j], int(f[2 + 3 * j]), int(f[3 + 3 * j])
            wb, ab = (int(v) for v in wa.split("-"))
            blocks.append(Scheme(wb, ab, wg, ag, True))
        rows.append(blocks)
    return rows


def zipf_popularity(E: int, s: float = 0.8, seed: int = 0) -> np.ndarray:
    """Expected routing popularity p_e used by gen_routing (same seeded permutation)."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(E)
    ranks = np.empty(E, dtype=np.float64)
    ranks[perm] = np.arange(1, E + 1, dtype=np.float64)
    p = ranks ** (-s)
    return p / p.sum()


def uniform_table(cfg: LayerConfig, scheme: Scheme) -> List[List[Scheme]]:
    return [[scheme, scheme, scheme] for _ in range(cfg.n_routed + cfg.n_shared)]


MIXTRAL_CROSSOVER = 124  # B200 roofline crossover W4A16 vs W8A8 (SURVEY.md §6, App. derivation)


def precision_table(cfg: LayerConfig, tokens: Optional[int] = None) -> List[List[Scheme]]:
    """Per-(expert, block) schemes, rows = routed experts then shared experts; cols gate, up, down."""
    T = cfg.tokens if tokens is None else tokens
    if cfg.name == "tiny":
        a, b = WO(4, 64, False), WA(8, -1)
        return [[a, a, b], [b, b, a], [a, b, a], [b, a, b]]
    if cfg.name == "dsv2":
        nblk = 3 * (cfg.n_routed + cfg.n_shared)
        pool = [WO(4, 128)] * 8 + [WO(3, 128)] * 16 + [WO(2, 128)] * 36
        pool += [WO(2, -1)] * (nblk - len(pool))
        rng = np.random.default_rng(7)
        order = rng.permutation(nblk)
        flat = [pool[i] for i in order]
        return [flat[3 * e: 3 * e + 3] for e in range(cfg.n_routed + cfg.n_shared)]
    if cfg.name == "q15":
        return parse_table6()
    if cfg.name == "mx":
        p = zipf_popularity(cfg.n_routed)
        rows = []
        for e in range(cfg.n_routed):
            sch = WA(8, -1) if T * cfg.top_k * p[e] >= MIXTRAL_CROSSOVER else WO(4, 128)
            rows.append([sch, sch, sch])
        return rows
    if cfg.name == "q2":
        rng = np.random.default_rng(11)
        n8 = int(round(cfg.n_routed * 35 / 61))
        pc_down = set(rng.permutation(cfg.n_routed)[:n8].tolist())
        rows = []
        for e in range(cfg.n_routed):
            down = WA(8, -1) if e in pc_down else WA(4, 128)
            rows.append([WA(4, 128), WA(4, 128), down])
        rows.append([WA(4, -1), WA(4, -1), WA(8, -1)])
        return rows
    raise KeyError(cfg.name)
