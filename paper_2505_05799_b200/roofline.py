"""Roofline bookkeeping for bench.py (host-side, §3.2).

Per-expert roofline of one MoE block: for every (expert e, block j) with m_e > 0
    t_roof(e, j) = max(2 m n k / P(kind), bytes(e, j) / BW)
    bytes = n k w/8 + meta + m k (a/8 or 2) [+ act scales] + m n 2
The paper's arithmetic-intensity argument (A = m for n, k >> m) gives the
crossover token counts between schemes, e.g. W4A16 vs W8A8.
"""
from __future__ import annotations

import json
import os
from typing import Dict, Optional

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_peaks() -> Dict[str, float]:
    """Measured peaks (MEASURED_PEAKS.json, driver-written) + our own i8 measurement if present."""
    out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            m = json.load(f)
        out.update({k: float(m[k]) for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        out["source"] = "measured"
    q = os.path.join(ROOT, "profiles", "i8_peak.json")
    m8 = {}
    if os.path.exists(q):
        with open(q) as f:
            m8 = json.load(f)
    if m8.get("i8_tops"):
        out["i8_tops"] = float(m8["i8_tops"])
        out["i8_source"] = "measured (profiles/i8_peak.json, torch._int_mm 8192^3)"
    else:
        out["i8_tops"] = 2.0 * out["bf16_tflops"]
        out["i8_source"] = "assumed 2 x bf16 (B200 nominal ratio 4.5/2.25)"
    # w4a4 runs on kind::f8f6f4 (e4m3): its own measured peak, else the i8 figure (same nominal 4.5 PF dense)
    if m8.get("f8_tflops"):
        out["f8_tflops"] = float(m8["f8_tflops"])
        out["f8_source"] = "measured (profiles/i8_peak.json, torch._scaled_mm e4m3 8192^3)"
    else:
        out["f8_tflops"] = out["i8_tops"]
        out["f8_source"] = "assumed = i8 (B200 nominal fp8 = int8 = 4.5 PF dense)"
    return out


def kind_peak(kind: str, peaks) -> float:
    """Tensor peak (FLOP/s) of an MMA kind: bf16 (kind::f16), i8 (w5a5 / w8a8), f8 (w4a4 on kind::f8f6f4)."""
    return {"bf16": peaks["bf16_tflops"], "i8": peaks["i8_tops"], "f8": peaks.get("f8_tflops", peaks["i8_tops"])}[kind] * 1e12


def crossover_m(peak_a: float, bytes_per_w_b: float, bw: float) -> float:
    """Arithmetic intensity (tokens per expert) where scheme a (fewer weight bytes, slower math, e.g.
    W4A16) stops beating scheme b (more bytes, faster math, e.g. W8A8): per weight element
    t(m) = max(2m / P, b / BW); a turns compute-bound while b is still memory-bound, so the two
    times meet at 2m / P_a = b_b / BW  ->  m* = P_a * b_b / (2 BW)   (n, k >> m).
    """
    return peak_a * bytes_per_w_b / (2.0 * bw)


def block_roofline(m: int, n: int, k: int, w_bits: int, a_bits: int, w_group: int, sym: bool, peaks) -> Dict:
    flops = 2.0 * m * n * k
    if w_bits == 16:
        wbytes, meta, kind = n * k * 2.0, 0.0, "bf16"
    else:
        g = k if w_group == -1 else w_group
        wbytes = n * k * w_bits / 8.0
        meta = n * (k / g) * 2.0 * (1 if (sym or a_bits != 16) else 2)
        kind = "bf16" if a_bits == 16 else ("f8" if w_bits == 4 else "i8")
    abytes = m * k * (2.0 if a_bits == 16 else 1.0) + (0 if a_bits == 16 else m * max(1, k // 128) * 4.0)
    obytes = m * n * 2.0
    byt = wbytes + meta + abytes + obytes
    P = kind_peak(kind, peaks)
    t = max(flops / P, byt / (peaks["hbm_gbs"] * 1e9))
    return {"flops": flops, "bytes": byt, "t": t, "kind": kind, "t_compute": flops / P}


def layer_roofline(table, counts, hidden: int, inter: int, shared_inter: int, n_routed: int, T: int, peaks) -> Dict:
    """Sum of per-(expert, block) rooflines (seconds) + totals; shared experts see m = T."""
    tot = {"t_roof": 0.0, "flops": 0.0, "bytes": 0.0, "flops_bf16": 0.0, "flops_i8": 0.0, "flops_f8": 0.0,
           "t_compute": 0.0, "t_memory": 0.0}
    for v, row in enumerate(table):
        m = int(counts[v]) if v < n_routed else T
        if m == 0:
            continue
        f = inter if v < n_routed else shared_inter
        for j, s in enumerate(row):
            n, k = (f, hidden) if j < 2 else (hidden, f)
            r = block_roofline(m, n, k, s.w_bits, s.a_bits, s.w_group, bool(s.symmetric), peaks)
            tot["t_roof"] += r["t"]
            tot["flops"] += r["flops"]
            tot["bytes"] += r["bytes"]
            tot["flops_" + r["kind"]] += r["flops"]
            tot["t_compute"] += r["t_compute"]
            tot["t_memory"] += r["bytes"] / (peaks["hbm_gbs"] * 1e9)
    # the FLOP-mix peak: the rate at which the whole block's FLOPs would run if every block ran at its kind's peak
    tot["peak_mix"] = tot["flops"] / tot["t_compute"] if tot["t_compute"] > 0 else 0.0
    return tot
