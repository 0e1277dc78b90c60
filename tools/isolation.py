"""Isolation runs of the persistent group-GEMM per variant (SURVEY §8(d) "isolation runs"):
one single-expert layer (Mixtral-8x7B shapes, d 4096, f 14336, no shared expert) per scheme, at a memory-bound
m (tokens routed to the expert) and a compute-bound m. The fused kernel's counters are aggregate over every
block of a real layer; here each launch holds one scheme only.

usage: python tools/isolation.py [--m 8 2048] [--reps 5] [--json out.json]
Run it under ncu (tools/gpu_isolation.sh) for dram__bytes / tensor-pipe counters per launch; without ncu it
prints CUDA-event GEMM times, achieved FLOP/s and the algorithmic-bytes HBM rate per variant.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from synth import configs as C  # noqa: E402

VARIANTS = [("w16", C.W16), ("w4a16_g128", C.WO(4, 128)), ("w2a16_g128", C.WO(2, 128)),
            ("w8a8_pc", C.WA(8, -1)), ("w4a4_pc", C.WA(4, -1)), ("w4a4_g128", C.WA(4, 128)),
            ("w8a8_g128", C.WA(8, 128))]


def algorithmic_bytes(sch, d, f, m):
    """Weights (+ 16-bit group meta / W-A scales) of gate, up, down + activations in / h round trip / out."""
    def wbytes(N, K):
        if sch.w_bits == 16:
            return 2 * N * K
        meta = (2 if sch.a_bits != 16 or sch.symmetric else 4) * N * (K // (128 if sch.w_group == 128 else K))
        return N * K * sch.w_bits // 8 + meta
    wb = 2 * wbytes(f, d) + wbytes(d, f)
    ab = 1 if sch.a_bits != 16 else 2
    return wb + m * (d * ab + f * 2 + f * ab + d * 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, nargs="+", default=[8, 2048])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--f", type=int, default=14336)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    import paper_2505_05799_b200 as mx
    mx.load()
    d, f = a.d, a.f
    W = [[bench.to_bf16(bench.gen_weight(f, d, 7000), "cuda"), bench.to_bf16(bench.gen_weight(f, d, 7001), "cuda"),
          bench.to_bf16(bench.gen_weight(d, f, 7002), "cuda")]]
    peaks = bench.load_peaks() if hasattr(bench, "load_peaks") else None
    res = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, sch in VARIANTS:
        lay = mx.MoELayer.from_weights(1, 0, d, f, 0, W, [[mx.Scheme.of(sch)] * 3])
        for m in a.m:
            x = bench.to_bf16(bench.gen_activations(m, d, seed=3), "cuda")
            ids = torch.zeros(m, 1, dtype=torch.int32, device="cuda")
            w = torch.ones(m, 1, dtype=torch.float32, device="cuda")
            ws = lay.workspace(m, 1)
            y = torch.empty(m, d, dtype=torch.bfloat16, device="cuda")
            lay.profile(a.reps)
            for _ in range(2):
                lay(x, ids, w, out=y, workspace=ws)
            for _ in range(a.reps):
                flush.zero_()
                lay(x, ids, w, out=y, workspace=ws)
            torch.cuda.synchronize()
            gemm_ms = float(np.median(lay.profile_read(a.reps)[:, 3]))
            flops = 3 * 2 * m * d * f
            byts = algorithmic_bytes(sch, d, f, m)
            res[f"{name}_m{m}"] = {"gemm_ms": gemm_ms, "tflops": flops / gemm_ms / 1e9,
                                   "alg_GBps": byts / gemm_ms / 1e6, "alg_bytes": byts}
            print(f"{name:12s} m={m:5d} gemm {gemm_ms * 1e3:9.1f} us  {flops / gemm_ms / 1e9:8.1f} TFLOP/s  "
                  f"alg HBM {byts / gemm_ms / 1e6:8.1f} GB/s", flush=True)
            del ws
        del lay
    if a.json:
        with open(a.json, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
