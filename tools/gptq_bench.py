"""NEXT-4 measurement: the offline GPTQ + Hadamard pipeline of one linear block on the GPU (CUDA events per stage)
and the fp64 oracle on a row sample of the same block (rows are independent given U), as achieved fp64 FLOP/s.

usage: python tools/gptq_bench.py [--N 14336 --K 4096 --n 2048 --bits 4 --group 128] [--json out.json]
FLOPs counted: Hessian 2 n K^2; prepare K^3 / 3 (reverse Cholesky) + K^3 / 3 (triangular inverse); quantize
N K^2 (column sweep + lazy updates: one multiply-add per (row, column, later column) pair).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import configs as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=14336)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--group", type=int, default=128)
    ap.add_argument("--oracle-rows", type=int, default=16)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    import paper_2505_05799_b200 as mx
    mx.load()
    N, K, n = a.N, a.K, a.n
    g = torch.Generator().manual_seed(0)
    x = (torch.randn(n, K, generator=g) @ (torch.eye(K) + torch.randn(K, K, generator=g) * (0.5 / K ** 0.5)))
    x = x.to(torch.bfloat16).cuda()
    w = (torch.randn(N, K, generator=g) * 0.02).to(torch.bfloat16).cuda()
    signs = (torch.randint(0, 2, (K,), generator=g, dtype=torch.int8) * 2 - 1).cuda()
    sch = mx.Scheme.of(C.WO(a.bits, a.group))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for rep in range(2):  # second repetition is timed (first warms up the module / allocator)
        ev[0].record()
        wr = mx.hadamard_rotate(w, signs, 1)
        ev[1].record()
        H = mx.gptq_hessian(x)
        ev[2].record()
        U, dead = mx.gptq_prepare(H)
        ev[3].record()
        codes, scale, zero = mx.gptq_quantize(sch, wr, U, dead)
        ev[4].record()
        torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    fl = [0.0, 2.0 * n * K * K, 2.0 * K ** 3 / 3, 2.0 * N * K * K]
    res = {"shape": {"N": N, "K": K, "n": n, "bits": a.bits, "group": a.group},
           "ms": dict(zip(["rotate", "hessian", "prepare", "quantize"], ms)),
           "fp64_tflops": {k: (f / (m * 1e9) if f else None) for k, f, m in
                           zip(["rotate", "hessian", "prepare", "quantize"], fl, ms)}}
    # the oracle on a row sample (same U, i.e. the GPU's H), fp64 NumPy
    from oracle.gptq import gptq_quantize
    from oracle.bf16 import bits_to_f64
    rows = np.arange(a.oracle_rows)
    Hn = mx.gptq_hessian(x).cpu().numpy()
    wb = wr.cpu().view(torch.int16).numpy().view(np.uint16)[rows]
    t0 = time.perf_counter()
    gptq_quantize(bits_to_f64(wb), Hn, a.bits, a.group, False)
    dt = time.perf_counter() - t0
    res["oracle"] = {"rows": int(rows.size), "s": dt, "rows_per_s": rows.size / dt,
                     "gpu_rows_per_s": N / (ms[3] / 1e3), "cores": len(os.sched_getaffinity(0))}
    print(json.dumps(res, indent=1))
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
