#!/usr/bin/env python
"""bench.py — MoE-block tokens/s of the B200-native MxMoE mixed-precision group-GEMM.

Metric (BASELINE.json): MoE-block tokens/s and % of per-expert roofline, on synthetic
inputs shaped like the paper's workloads. A "step" is one
mxm_moe_group_gemm call (route-prep, act-quant + gather, plan, persistent group-GEMM,
combine) over one batch of T tokens whose inputs are resident in HBM; L2 is flushed
(256 MB memset) before every timed step, outside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config q2|dsv2|q15|mx|tiny] [--tokens T]
  python bench.py --impl reference ...   (the CPU oracle on bounded token samples)

Default workload: the BASELINE.json headline, the Qwen2-57B-A14B layer at T = 16384 tokens (the largest
single-GPU config; 64 routed + 1 shared expert, W-A mix). N > 1: when not already under torchrun, bench.py
re-executes itself under `torch.distributed.run --nproc-per-node N` (127.0.0.1); each rank then runs expert
parallelism: rank r owns routed experts [r·E/G, (r+1)·E/G) and its own batch of T tokens
(weak scaling), tokens are dispatched to / combined from the expert owners with NCCL all-to-all
(paper_2505_05799_b200/ep.py). `--replicas` instead runs N independent full replicas.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import configs as C  # noqa: E402
from synth.gen import gen_activations, gen_routing, gen_shared_weights, gen_weight, weight_seed  # noqa: E402

METRIC = "MoE-block tokens/s at 1/2/4/8 B200 and % of per-expert roofline vs bf16 & uniform"  # BASELINE.json
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--config", default="q2")
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--table", default="mixed", help="mixed | w16 | <scheme name, e.g. w2a16_g128_asym>")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=128, help="tokens of the larger cpu_baseline oracle sample")
    ap.add_argument("--no-comparators", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent full replicas instead of EP")
    ap.add_argument("--placement", default="lpt", choices=["lpt", "contiguous"],
                    help="N>1 expert parallelism: expert-to-rank placement (placement.py; LPT on the Zipf popularity)")
    return ap.parse_args()


def table_for(cfg, name, T):
    if name == "mixed":
        return C.precision_table(cfg, T)
    if name == "w16":
        return C.uniform_table(cfg, C.W16)
    for s in ([C.WO(b, g, sy) for b in (2, 3, 4, 8) for g in (64, 128, -1) for sy in (False, True)]
              + [C.WA(b, g) for b in (4, 5, 8) for g in (128, -1)] + [C.FP8(g) for g in (128, -1)]):
        if s.name() == name:
            return C.uniform_table(cfg, s)
    raise SystemExit(f"unknown table {name}")


def gen_weights(cfg):
    W = []
    for v in range(cfg.n_routed + cfg.n_shared):
        f = cfg.inter if v < cfg.n_routed else cfg.shared_inter
        W.append([gen_weight(f, cfg.hidden, weight_seed(v, 0)), gen_weight(f, cfg.hidden, weight_seed(v, 1)),
                  gen_weight(cfg.hidden, f, weight_seed(v, 2))])
    return W


def to_bf16(bits, dev):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 6 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(float(r[0]) for r in rows), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


UNIFORM_COMPARATORS = {
    "dsv2": ["w16", "w2a16_g128_asym"],      # bf16 and the equal-bits (2.25) uniform scheme
    "q15": ["w16", "w8a8_g-1_sym"],          # bf16 and uniform W8A8
    "mx": ["w16", "w8a8_g-1_sym", "w4a16_g128_asym"],
    "q2": ["w8a8_g-1_sym", "w16"],
    "tiny": ["w16"],
}


def lib_sha1() -> str:
    import hashlib
    from paper_2505_05799_b200 import _lib
    with open(os.environ.get("MXM_LIB") or _lib.LIB_PATH, "rb") as f:
        return hashlib.sha1(f.read()).hexdigest()


def time_steps(fn, steps, flush):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        ev[i][0].record()
        fn()
        ev[i][1].record()
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in ev)


def bf16_grouped_block(cfg, Wt, x, ids, w, sw, steps, flush):
    """Baseline: the bf16 MoE block with torch._grouped_mm (cuBLAS-class grouped GEMM) on the same routing.

    Stand-in for the paper's CUTLASS 16-bit Group-GEMM baseline. Returns (block ms, GEMM-only ms).
    """
    E, S, d, f = cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter
    wgu = torch.stack([torch.cat([Wt[e][0], Wt[e][1]], 0).t() for e in range(E)])  # [E, d, 2f] column-major
    wd = torch.stack([Wt[e][2].t() for e in range(E)])                            # [E, f, d]
    T, k = ids.shape
    flat = ids.reshape(-1).long()
    order = torch.argsort(flat, stable=True)
    counts = torch.bincount(flat, minlength=E)
    offs = counts.cumsum(0).to(torch.int32)
    tok = order // k
    wr = w.reshape(-1)[order].unsqueeze(1).to(torch.bfloat16)
    xs = x[tok]

    wsh = [(torch.cat([Wt[E + s][0], Wt[E + s][1]], 0).t().contiguous(), Wt[E + s][2].t().contiguous())
           for s in range(S)]  # shared experts: dense [d, 2 f_s] and [f_s, d]
    fs = cfg.shared_inter

    def routed():
        gu = torch._grouped_mm(xs, wgu, offs=offs)
        h = torch.nn.functional.silu(gu[:, :f]) * gu[:, f:]
        return torch._grouped_mm(h, wd, offs=offs)

    def shared(s):
        gu = x @ wsh[s][0]
        return (torch.nn.functional.silu(gu[:, :fs]) * gu[:, fs:]) @ wsh[s][1]

    def gemms():  # every expert GEMM of the block, routed and shared (the same FLOPs as the group-GEMM)
        o = routed()
        return o, [shared(s) for s in range(S)]

    def block():
        o, ys = gemms()
        y = torch.zeros(T, d, dtype=torch.float32, device=x.device).index_add_(0, tok, (o * wr).float())
        for s in range(S):
            y += ys[s].float() * (sw[:, s:s + 1] if sw is not None else 1.0)
        return y.to(torch.bfloat16)

    for _ in range(3):
        block()
    return time_steps(block, steps, flush), time_steps(gemms, steps, flush)


def dist_init(n):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def allmax(v, ws):
    if ws == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _oracle_block(args):
    """One block of oracle.moe.quantize_block (setup of the CPU baseline, run in a process pool)."""
    from oracle.moe import quantize_block
    wb, sch = args
    qb = quantize_block(wb, sch)
    if qb.w_bits != 16:  # same integer values in a compact dtype (the oracle casts codes to fp64 where it uses them)
        qb.codes = qb.codes.astype(np.int8 if qb.codes.min() >= -128 and qb.codes.max() <= 127 else np.int16)
    return qb


def oracle_layer(cfg, table, weights, experts=None):
    """The oracle's quantized layer (oracle.moe.QuantizedLayer), blocks quantized in parallel on the host cores.
    `experts`: routed experts to quantize (others stay None: the sample never routes to them)."""
    from concurrent.futures import ProcessPoolExecutor
    from oracle.moe import QuantizedLayer
    E, S = cfg.n_routed, cfg.n_shared
    todo = [v for v in range(E + S) if experts is None or v >= E or v in experts]
    jobs = [(weights[v][j], table[v][j]) for v in todo for j in range(3)]
    with ProcessPoolExecutor(max(1, min(len(jobs), len(os.sched_getaffinity(0))))) as ex:
        qbs = list(ex.map(_oracle_block, jobs, chunksize=1))
    blocks = [None] * (E + S)
    for i, v in enumerate(todo):
        blocks[v] = qbs[3 * i: 3 * i + 3]
    return QuantizedLayer(E, S, cfg.hidden, cfg.inter, cfg.shared_inter if S else 0, blocks)


def cpu_oracle_baseline(cfg, table, weights, x, ids, w, sw, T, n_big):
    """The oracle as it stands (oracle.moe.moe_block, fp64 NumPy) on two seeded token samples of this batch.

    Every moe_block call converts the weights of each expert it touches (dequantized / fp64 codes), a fixed
    cost per call, then spends a per-token cost; two sample sizes that touch the same experts separate the two
    and give the extrapolated full-batch rate. Setup (quantizing the layer) is untimed."""
    from oracle.moe import moe_block
    ol = oracle_layer(cfg, table, weights)
    rng = np.random.default_rng(5)
    pts = []
    for n in (max(1, n_big // 4), n_big):
        rows = np.sort(rng.choice(T, min(n, T), replace=False))
        t0 = time.perf_counter()
        moe_block(x[rows], ol, ids[rows], w[rows], None if sw is None else sw[rows])
        pts.append((len(rows), time.perf_counter() - t0, len(set(ids[rows].reshape(-1).tolist()) - {-1})))
    (n1, t1, e1), (n2, t2, e2) = pts
    per_tok = max((t2 - t1) / (n2 - n1), 1e-9) if n2 > n1 else t2 / n2
    fixed = max(t2 - per_tok * n2, 0.0)
    return {"value": n2 / t2, "unit": "tokens/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
            "sample": f"{n2} seeded random tokens of the {cfg.name} T={T} batch (oracle.moe.moe_block, fp64 NumPy): "
                      f"{t2:.1f} s, {e2}/{cfg.n_routed} routed experts + {cfg.n_shared} shared touched",
            "second_sample": {"tokens": n1, "s": t1, "experts_touched": e1},
            "per_call_weight_conversion_s": fixed, "per_token_s": per_tok,
            "extrapolated_full_batch_tokens_per_s": T / (fixed + per_tok * T),
            "note": "value = measured sample throughput; the extrapolation charges the per-call weight conversion "
                    "once per batch"}


def run_reference(args, cfg, T):
    """--impl reference: the CPU oracle on bounded token samples of the same workload (rank 0 only)."""
    ws, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return
    table = table_for(cfg, args.table, T)
    weights = gen_weights(cfg)
    x = gen_activations(T, cfg.hidden, seed=1)
    ids, w = gen_routing(T, cfg.n_routed, cfg.top_k, seed=0)
    sw = gen_shared_weights(T, cfg.n_shared) if cfg.n_shared else None
    from oracle.moe import moe_block
    ol = oracle_layer(cfg, table, weights)
    # per step: a few random tokens (each call re-converts the weights of every expert it touches, so the step
    # cost is dominated by that fixed part on the big layers; sized so K + W steps end within a few minutes)
    sample = max(1, min(T, args.cpu_sample // (64 if cfg.name == "q2" else 8)))
    rng = np.random.default_rng(5)
    times = []
    for i in range(args.warmup + args.steps):
        rows = np.sort(rng.choice(T, sample, replace=False))
        t0 = time.perf_counter()
        moe_block(x[rows], ol, ids[rows], w[rows], None if sw is None else sw[rows])
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = sample * len(times) / tot
    cores = len(os.sched_getaffinity(0))
    line = {"metric": METRIC, "value": val, "unit": "tokens/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "tokens": T, "sample_tokens_per_step": sample, "table": args.table},
            "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"{sample} random tokens of the {cfg.name} T={T} batch per step"},
            "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def maybe_spawn(args) -> bool:
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run with N local ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    maybe_spawn(args)
    cfg = C.get_config(args.config)
    T = args.tokens or cfg.tokens
    if args.impl == "reference":
        run_reference(args, cfg, T)
        return
    ws, rank, local = dist_init(args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_2505_05799_b200 as mx
    from paper_2505_05799_b200.roofline import layer_roofline, load_peaks

    table = table_for(cfg, args.table, T)
    weights = gen_weights(cfg)
    Wt = [[to_bf16(b, dev) for b in blk] for blk in weights]
    use_ep = ws > 1 and not args.replicas
    inv_place = None
    if use_ep:
        from paper_2505_05799_b200.ep import ExpertParallelMoE
        from paper_2505_05799_b200.placement import apply_placement, inverse, lpt_placement
        # expert placement: the experts are re-indexed offline (weights / table reordered; the router emits ids in
        # the new order, here the synthetic ids are mapped through the inverse permutation)
        perm = (lpt_placement(C.zipf_popularity(cfg.n_routed, 0.8, seed=0), ws) if args.placement == "lpt"
                else np.arange(cfg.n_routed))
        Wt, table = apply_placement(Wt, table, perm, cfg.n_routed)
        inv_place = inverse(perm)
        ep = ExpertParallelMoE.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, Wt,
                                            table)
        layer = ep.local  # the rank's routed experts: the dominant kernel
    else:
        layer = mx.MoELayer.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, Wt,
                                         [[mx.Scheme.of(s) for s in row] for row in table])
    del Wt
    # per-rank batch: rank r uses seeds offset by r
    x_np = gen_activations(T, cfg.hidden, seed=1 + rank)
    ids_np, w_np = gen_routing(T, cfg.n_routed, cfg.top_k, seed=rank)
    place = (lambda a: np.where(a >= 0, inv_place[np.maximum(a, 0)], -1).astype(np.int32)) if inv_place is not None \
        else (lambda a: a)
    ids_np = place(ids_np)
    sw_np = gen_shared_weights(T, cfg.n_shared, seed=2 + rank) if cfg.n_shared else None
    x = to_bf16(x_np, dev)
    ids = torch.from_numpy(ids_np).to(dev)
    w = torch.from_numpy(w_np).to(dev)
    sw = torch.from_numpy(sw_np).to(dev) if sw_np is not None else None
    k = cfg.top_k
    y = torch.empty(T, cfg.hidden, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    if use_ep:
        def step(xa, ia, wa, sa, out):
            out.copy_(ep(xa, ia, wa, sa))
        wsb = None
        # the local layer's counts: every rank's routing restricted to this rank's experts (host, seeded)
        epr = cfg.n_routed // ws
        all_ids = place(np.concatenate([gen_routing(T, cfg.n_routed, cfg.top_k, seed=r)[0] for r in range(ws)]))
        loc = all_ids[(all_ids >= rank * epr) & (all_ids < (rank + 1) * epr)] - rank * epr
        counts_local = np.bincount(loc, minlength=epr)
    else:
        wsb = layer.workspace(T, k)

        def step(xa, ia, wa, sa, out):
            layer(xa, ia, wa, sa, out=out, workspace=wsb)

    for _ in range(args.warmup):
        step(x, ids, w, sw, y)
    torch.cuda.synchronize()
    if not use_ep:
        assert layer.poll_error(wsb) == 0
        n_tasks, n_exec = layer.task_stats(T, k, wsb)
        assert n_tasks == n_exec and n_tasks > 0, (n_tasks, n_exec)
    else:
        n_tasks = None

    K = args.steps
    layer.profile(K)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clk = ClockSampler(local)
    clk.start()
    barrier(ws)
    for i in range(K):
        flush.zero_()
        ev[i][0].record()
        step(x, ids, w, sw, y)
        ev[i][1].record()
    barrier(ws)
    clocks = clk.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    stages = layer.profile_read(K)  # [K, 5]: route, gather, plan, gemm, combine
    layer.profile(0)
    ms = allmax(statistics.mean(step_ms), ws)
    gemm_ms = allmax(float(stages[:, 3].mean()), ws)
    value = ws * T / (ms / 1e3)

    # ---- e2e through the public API with pinned host buffers (H2D inputs, D2H output inside the timing)
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        idh = ids.cpu().pin_memory()
        wh = w.cpu().pin_memory()
        swh = sw.cpu().pin_memory() if sw is not None else None
        yh = torch.empty_like(y, device="cpu").pin_memory()
        xd, idd, wd = torch.empty_like(x), torch.empty_like(ids), torch.empty_like(w)
        swd = torch.empty_like(sw) if sw is not None else None
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        barrier(ws)
        for i in range(K):
            flush.zero_()
            ev2[i][0].record()
            xd.copy_(xh, non_blocking=True)
            idd.copy_(idh, non_blocking=True)
            wd.copy_(wh, non_blocking=True)
            if swd is not None:
                swd.copy_(swh, non_blocking=True)
            step(xd, idd, wd, swd, y)
            yh.copy_(y, non_blocking=True)
            ev2[i][1].record()
        barrier(ws)
        e2e_ms = allmax(statistics.mean(a.elapsed_time(b) for a, b in ev2), ws)
        h2d = x.numel() * 2 + ids.numel() * 4 + w.numel() * 4 + (sw.numel() * 4 if sw is not None else 0)
        e2e = {"value": ws * T / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(y.numel() * 2), "ms_per_step": e2e_ms}

    # ---- roofline of the dominant kernel (the persistent group-GEMM)
    peaks = load_peaks()
    if use_ep:  # the local layer: this rank's experts (no shared) on the rows it received
        rl = layer_roofline(table[rank * epr:(rank + 1) * epr], counts_local, cfg.hidden, cfg.inter, 0, epr, T, peaks)
    else:
        counts = np.bincount(ids_np[ids_np >= 0].reshape(-1), minlength=cfg.n_routed)
        rl = layer_roofline(table, counts, cfg.hidden, cfg.inter, cfg.shared_inter, cfg.n_routed, T, peaks)
    # bound of the dominant kernel from its own per-expert roofline: compute (FLOPs at each block's kind peak)
    # vs bytes over HBM; the peak is the FLOP-mix one (FLOPs / sum_kind FLOPs_kind / peak_kind)
    hbm_bound = rl["t_memory"] > rl["t_compute"]
    if hbm_bound:
        achieved = rl["bytes"] / (gemm_ms / 1e3) / 1e9
        peak, unit, alg = peaks["hbm_gbs"], "GB/s", {"algorithmic_bytes_per_launch": rl["bytes"]}
        peak_src = f"MEASURED_PEAKS.json hbm_gbs ({peaks['source']})"
    else:
        achieved = rl["flops"] / (gemm_ms / 1e3) / 1e12
        peak, unit, alg = rl["peak_mix"] / 1e12, "TFLOP/s", {"algorithmic_flops_per_launch": rl["flops"]}
        peak_src = (f"FLOP-mix of bf16 {peaks['bf16_tflops']:.0f} (MEASURED_PEAKS.json burst), i8 {peaks['i8_tops']:.0f} "
                    f"({peaks['i8_source']}), f8 {peaks['f8_tflops']:.0f} ({peaks['f8_source']}); FLOP shares bf16 "
                    f"{rl['flops_bf16'] / rl['flops']:.2f} / i8 {rl['flops_i8'] / rl['flops']:.2f} / f8 "
                    f"{rl['flops_f8'] / rl['flops']:.2f}")
    traffic, traffic_note = None, "no ncu capture of this library build for this config"
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.name}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        if tj.get("lib_sha1") == lib_sha1() and tj.get("tokens") == T:
            traffic, traffic_note = tj.get("dram_bytes_per_launch"), f"ncu --set full capture ({tp}, same library)"
        else:
            traffic_note = f"stale: {tp} was captured on another library build; not reported"
    roofline = {"bound": "hbm" if hbm_bound else "tensor", "achieved": achieved, "peak": peak, "unit": unit,
                "frac": achieved / peak, "traffic": traffic, "traffic_note": traffic_note, "kernel": "moe_gemm_kernel",
                "peak_source": peak_src, **alg, "kernel_ms": gemm_ms}
    per_expert = {"t_roof_us": rl["t_roof"] * 1e6, "frac_of_gemm": rl["t_roof"] / (gemm_ms / 1e3),
                  "frac_of_step": rl["t_roof"] / (ms / 1e3), "alg_bytes": rl["bytes"], "alg_flops": rl["flops"],
                  "t_compute_us": rl["t_compute"] * 1e6, "t_memory_us": rl["t_memory"] * 1e6}
    stage_ms = {n: float(stages[:, i].mean()) for i, n in enumerate(["route", "gather", "plan", "gemm", "combine"])}

    comparators = None
    if not args.no_comparators and args.table == "mixed" and ws == 1:
        comparators = {"note": "same routing and tokens; ms per block step, L2 flushed; tokens/s = T / time"}
        Wt = [[to_bf16(b, dev) for b in blk] for blk in weights]
        try:
            blk_ms, gemm_ms_bf16 = bf16_grouped_block(cfg, Wt, x, ids, w, sw, K, flush)
            comparators["bf16_torch_grouped_mm"] = {"block_ms": blk_ms, "gemm_ms": gemm_ms_bf16,
                                                    "tokens_per_s": T / (blk_ms / 1e3)}
        except Exception as e:  # comparator failures never fail the bench
            comparators["bf16_torch_grouped_mm"] = {"error": str(e)[:200]}
        for tb in UNIFORM_COMPARATORS.get(cfg.name, []):
            tab_u = table_for(cfg, tb, T)
            lay = mx.MoELayer.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, Wt,
                                           [[mx.Scheme.of(sc) for sc in row] for row in tab_u])
            wsu = lay.workspace(T, k)
            for _ in range(3):
                lay(x, ids, w, sw, out=y, workspace=wsu)
            lay.profile(K)
            u_ms = time_steps(lambda: lay(x, ids, w, sw, out=y, workspace=wsu), K, flush)
            u_gemm = float(lay.profile_read(K)[:, 3].mean())
            comparators["ours_uniform_" + tb] = {"block_ms": u_ms, "gemm_ms": u_gemm, "tokens_per_s": T / (u_ms / 1e3)}
            del lay, wsu
        del Wt
        comparators["ours_mixed"] = {"block_ms": ms, "gemm_ms": gemm_ms, "tokens_per_s": T / (ms / 1e3)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_baseline(cfg, table, weights, x_np, ids_np, w_np, sw_np, T, min(T, args.cpu_sample))
    launches = layer.kernels_per_call
    if use_ep:  # ep_route + ep_pack + local layer + shared layer + ep_combine (NCCL kernels not counted)
        launches += 3 + (ep.shared.kernels_per_call if ep.shared is not None else 0)
    if rank == 0:
        kinds = [k for k in ("bf16", "i8", "f8") if rl["flops_" + k] > 0]
        dt = "+".join({"bf16": "bf16", "i8": "int8", "f8": "e4m3"}[k] for k in kinds)
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dt,
                "data": "synthetic (seeded N(0,1) x, N(0,1/K) weights, Zipf-0.8 Gumbel top-k routing)",
                "config": {"workload": cfg.name, "tokens_per_gpu": T, "experts": f"{cfg.n_routed}+{cfg.n_shared}",
                           "hidden": cfg.hidden, "inter": cfg.inter, "top_k": k, "table": args.table,
                           "l2": "flushed before every timed step (256 MB memset, untimed)",
                           "parallelism": (f"ep{ws} (sync-free NCCL all-to-all dispatch/combine at fixed capacity, "
                                           f"{args.placement} expert placement, shared experts replicated)"
                                           if use_ep else f"replicas x{ws}") if ws > 1 else "single GPU"},
                "roofline": roofline, "per_expert_roofline": per_expert, "stage_ms": stage_ms,
                "cpu_baseline": cpu, "e2e": e2e, "comparators": comparators, "gpu_launches": launches * K, "clocks": clocks,
                "tasks_per_step": n_tasks}
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
