#!/usr/bin/env python
"""bench.py — MoE-block tokens/s of the B200-native MxMoE mixed-precision group-GEMM.

Metric (BASELINE.json): MoE-block tokens/s and % of per-expert roofline, on synthetic
inputs shaped like the paper's workloads. A "step" is one
mxm_moe_group_gemm call (route-prep, act-quant + gather, plan, persistent group-GEMM,
combine) over one batch of T tokens whose inputs are resident in HBM; L2 is flushed
(256 MB memset) before every timed step, outside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config dsv2|q15|mx|q2|tiny] [--tokens T]
  python bench.py --impl reference ...   (the CPU oracle on bounded token samples)

N > 1 (torchrun, one rank per GPU): expert parallelism. Rank r owns routed experts
[r·E/G, (r+1)·E/G) and its own batch of T tokens (weak scaling: per-GPU tokens and per-GPU expert work
fixed as N grows); tokens are dispatched to / combined from the expert owners with NCCL all-to-all
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
    ap.add_argument("--config", default="dsv2")
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--table", default="mixed", help="mixed | w16 | <scheme name, e.g. w2a16_g128_asym>")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=512, help="tokens in the cpu_baseline oracle sample")
    ap.add_argument("--no-comparators", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent full replicas instead of EP")
    return ap.parse_args()


def table_for(cfg, name, T):
    if name == "mixed":
        return C.precision_table(cfg, T)
    if name == "w16":
        return C.uniform_table(cfg, C.W16)
    for s in ([C.WO(b, g, sy) for b in (2, 3, 4, 8) for g in (64, 128, -1) for sy in (False, True)]
              + [C.WA(b, g) for b in (4, 5, 8) for g in (128, -1)]):
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
    "q2": ["w8a8_g-1_sym"],
    "tiny": ["w16"],
}


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

    def gemms():
        gu = torch._grouped_mm(xs, wgu, offs=offs)
        h = torch.nn.functional.silu(gu[:, :f]) * gu[:, f:]
        return torch._grouped_mm(h, wd, offs=offs)

    def block():
        o = gemms() * wr
        y = torch.zeros(T, d, dtype=torch.float32, device=x.device).index_add_(0, tok, o.float())
        for s in range(S):
            g = x @ Wt[E + s][0].t()
            u = x @ Wt[E + s][1].t()
            ys = (torch.nn.functional.silu(g) * u) @ Wt[E + s][2].t()
            y += ys.float() * (sw[:, s:s + 1] if sw is not None else 1.0)
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


def cpu_oracle_tokens_per_s(cfg, table, weights, x, ids, w, sw, sample):
    """The oracle as it stands (oracle.moe.moe_block, fp64 NumPy) on `sample` tokens; setup untimed."""
    from oracle.moe import moe_block, quantize_layer
    ol = quantize_layer(weights, table, cfg.n_routed, cfg.n_shared)
    rows = np.arange(sample)
    t0 = time.perf_counter()
    moe_block(x[rows], ol, ids[rows], w[rows], None if sw is None else sw[rows])
    dt = time.perf_counter() - t0
    return sample / dt, dt


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
    from oracle.moe import moe_block, quantize_layer
    ol = quantize_layer(weights, table, cfg.n_routed, cfg.n_shared)
    sample = max(1, min(T, args.cpu_sample // 4))
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


def main():
    args = parse()
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
    if use_ep:
        from paper_2505_05799_b200.ep import ExpertParallelMoE
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
        all_ids = np.concatenate([gen_routing(T, cfg.n_routed, cfg.top_k, seed=r)[0] for r in range(ws)])
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
    i8_dom = rl["flops_i8"] > rl["flops_bf16"]
    peak_tf = peaks["i8_tops"] if i8_dom else peaks["bf16_tflops"]
    achieved = rl["flops"] / (gemm_ms / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.name}.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s" if not i8_dom else "TOP/s",
                "frac": achieved / peak_tf, "traffic": traffic, "kernel": "moe_gemm_kernel",
                "peak_source": (peaks["i8_source"] if i8_dom else f"MEASURED_PEAKS.json bf16_tflops (burst, "
                                                                    f"{peaks['source']})"),
                "algorithmic_flops_per_launch": rl["flops"], "kernel_ms": gemm_ms}
    per_expert = {"t_roof_us": rl["t_roof"] * 1e6, "frac_of_gemm": rl["t_roof"] / (gemm_ms / 1e3),
                  "frac_of_step": rl["t_roof"] / (ms / 1e3), "alg_bytes": rl["bytes"]}
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
        samp = min(T, args.cpu_sample)
        tps, dt = cpu_oracle_tokens_per_s(cfg, table, weights, x_np, ids_np, w_np, sw_np, samp)
        cpu = {"value": tps, "unit": "tokens/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
               "sample": f"first {samp} tokens of the {cfg.name} T={T} batch (oracle.moe.moe_block, fp64), "
                         f"{dt:.1f} s"}
    launches = layer.kernels_per_call
    if use_ep:  # ep_route + ep_pack + local layer + shared layer + ep_combine (NCCL kernels not counted)
        launches += 3 + (ep.shared.kernels_per_call if ep.shared is not None else 0)
    if rank == 0:
        dt = "int8" if i8_dom else "bf16"
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dt,
                "data": "synthetic (seeded N(0,1) x, N(0,1/K) weights, Zipf-0.8 Gumbel top-k routing)",
                "config": {"workload": cfg.name, "tokens_per_gpu": T, "experts": f"{cfg.n_routed}+{cfg.n_shared}",
                           "hidden": cfg.hidden, "inter": cfg.inter, "top_k": k, "table": args.table,
                           "l2": "flushed before every timed step (256 MB memset, untimed)",
                           "parallelism": (f"ep{ws} (NCCL all-to-all dispatch/combine, shared experts replicated)"
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
