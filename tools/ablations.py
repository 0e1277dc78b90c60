"""NEXT-3 kernel ablations on this B200 (App. A.2, slice-K P:229, sequential
per-expert execution P:75 / P:131). Prints one JSON object; usage: python tools/ablations.py [out.json]

  dense_8192:      one linear-block triple (gate/up/down) of 8192 x 8192 over 8192 tokens through the unified
                   persistent kernel, per scheme -> TOP/s (the paper's specialized-vs-unified W4A4 per-channel /
                   g128 question, asked of our one unified kernel)
  split_k:         Mixtral T = 1 / 4 / 16 GEMM time with slice-K (product) vs a build without it (MXM_SPLIT_ROWS=0)
  sequential:      DSV2 / Qwen1.5 blocks: one grouped launch vs one single-expert layer call per active expert
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from synth import configs as C  # noqa: E402


def timed(fn, steps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))


def dense_8192(mx):
    n = 8192
    out = {}
    W = [[bench.to_bf16(bench.gen_weight(n, n, 9000 + j), "cuda") for j in range(3)]]
    x = bench.to_bf16(bench.gen_activations(n, n, seed=3), "cuda")
    ids = torch.zeros(n, 1, dtype=torch.int32, device="cuda")
    w = torch.ones(n, 1, dtype=torch.float32, device="cuda")
    for name, sch in [("w4a4_pc", C.WA(4, -1)), ("w4a4_g128", C.WA(4, 128)), ("w8a8_pc", C.WA(8, -1)),
                      ("w8a8_g128", C.WA(8, 128)), ("w4a16_g128", C.WO(4, 128)), ("w16", C.W16)]:
        lay = mx.MoELayer.from_weights(1, 0, n, n, 0, W, [[mx.Scheme.of(sch)] * 3])
        ws = lay.workspace(n, 1)
        y = torch.empty(n, n, dtype=torch.bfloat16, device="cuda")
        lay.profile(8)
        timed(lambda: lay(x, ids, w, out=y, workspace=ws), steps=8, warm=2)
        gemm = float(np.median(lay.profile_read(8)[:, 3]))
        out[name] = {"gemm_ms": gemm, "tops": 3 * 2 * n ** 3 / (gemm / 1e3) / 1e12}
        del lay, ws
    return out


def split_k():
    res = {}
    lib_ns = os.path.join(ROOT, "tools", "variants", "lib_nosplit.so")
    for T in (1, 4, 16):
        row = {}
        for tag, lib in (("slice_k", ""), ("no_slice_k", lib_ns)):
            env = dict(os.environ, MXM_LIB=lib)
            r = subprocess.run([sys.executable, "bench.py", "--config", "mx", "--tokens", str(T), "--steps", "10",
                                "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-comparators"],
                               cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
            d = json.loads(r.stdout.strip().splitlines()[-1])
            row[tag] = {"gemm_ms": d["roofline"]["kernel_ms"], "step_ms": d["ms_per_step"]}
        res[f"mx_T{T}"] = row
    return res


def sequential(mx, cfg_name):
    cfg = C.get_config(cfg_name)
    T = 2048
    table = C.precision_table(cfg, T)
    weights = bench.gen_weights(cfg)
    Wt = [[bench.to_bf16(b, "cuda") for b in blk] for blk in weights]
    x_np = bench.gen_activations(T, cfg.hidden, seed=1)
    ids_np, w_np = bench.gen_routing(T, cfg.n_routed, cfg.top_k, seed=0)
    x = bench.to_bf16(x_np, "cuda")
    ids = torch.from_numpy(ids_np).cuda()
    w = torch.from_numpy(w_np).cuda()
    sw = torch.from_numpy(bench.gen_shared_weights(T, cfg.n_shared)).cuda() if cfg.n_shared else None
    full = mx.MoELayer.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, Wt,
                                    [[mx.Scheme.of(s) for s in r] for r in table])
    wsf = full.workspace(T, cfg.top_k)
    y = torch.empty(T, cfg.hidden, dtype=torch.bfloat16, device="cuda")
    t_grouped = timed(lambda: full(x, ids, w, sw, out=y, workspace=wsf))
    # one single-expert layer per active expert (and per shared expert), each called on its own tokens
    calls = []
    for e in range(cfg.n_routed):
        tt, jj = np.nonzero(ids_np == e)
        if tt.size == 0:
            continue
        lay = mx.MoELayer.from_weights(1, 0, cfg.hidden, cfg.inter, 0, [Wt[e]], [[mx.Scheme.of(s) for s in table[e]]])
        xe = x[torch.from_numpy(tt).cuda()].contiguous()
        ie = torch.zeros(tt.size, 1, dtype=torch.int32, device="cuda")
        we = torch.from_numpy(w_np[tt, jj].reshape(-1, 1).copy()).cuda()
        calls.append((lay, xe, ie, we, lay.workspace(tt.size, 1), torch.empty_like(xe)))
    for s in range(cfg.n_shared):
        v = cfg.n_routed + s
        lay = mx.MoELayer.from_weights(1, 0, cfg.hidden, cfg.shared_inter, 0, [Wt[v]], [[mx.Scheme.of(q) for q in table[v]]])
        calls.append((lay, x, torch.zeros(T, 1, dtype=torch.int32, device="cuda"), sw[:, s:s + 1].contiguous(),
                      lay.workspace(T, 1), torch.empty_like(x)))

    def seq():
        for lay, xe, ie, we, wse, ye in calls:
            lay(xe, ie, we, out=ye, workspace=wse)

    t_seq = timed(seq)
    return {"tokens": T, "grouped_launch_ms": t_grouped, "sequential_per_expert_ms": t_seq, "launches": len(calls),
            "speedup_grouped": t_seq / t_grouped,
            "note": "sequential = one mxm_moe_group_gemm call per expert on its own tokens (no cross-expert combine)"}


def main():
    import paper_2505_05799_b200 as mx
    out = {"dense_8192": dense_8192(mx), "split_k": split_k(),
           "sequential": {c: sequential(mx, c) for c in ("dsv2", "q15")},
           "gpu": torch.cuda.get_device_name()}
    s = json.dumps(out, indent=1)
    print(s)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(s)


if __name__ == "__main__":
    main()
