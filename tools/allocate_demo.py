"""NEXT-2 demonstration on this B200: the Eq. 7 allocator (paper_2505_05799_b200/allocator.py) fed by MEASURED
tile costs (mxm_profile_tile_costs) and measured block perturbations Δ (Eq. 6) on the DeepSeek-V2-Lite layer
shapes, for r in {0, 0.25, 0.5, 0.75, 1} under a 4.25-bit memory budget; every resulting table is then run
through the hot path and its block time and output error (vs the all-bf16 layer) are measured -- the direction
of the paper's fig:ablation-r: larger r trades time for accuracy. Usage: python tools/allocate_demo.py [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_05799_b200 import allocator as A  # noqa: E402
from synth import configs as C  # noqa: E402


def main():
    import paper_2505_05799_b200 as mx
    cfg = C.get_config("dsv2")
    E, d, f, k, T = cfg.n_routed, cfg.hidden, cfg.inter, cfg.top_k, cfg.tokens
    schemes = [C.WO(2, 128), C.WO(3, 128), C.WO(4, 128), C.WO(8, 128), C.WA(4, 128), C.WA(4, -1), C.WA(8, -1), C.W16]
    names = [s.name() for s in schemes]
    weights = bench.gen_weights(C.LayerConfig("dsv2r", E, 0, d, f, 0, k, T))
    Wt = [[bench.to_bf16(b, "cuda") for b in blk] for blk in weights]
    ids_np, w_np = bench.gen_routing(T, E, k, seed=0)
    counts = np.bincount(ids_np.reshape(-1), minlength=E)
    freq = counts / counts.sum()
    x_cal = bench.to_bf16(bench.gen_activations(128, d, seed=77), "cuda")
    delta = A.measure_deltas(mx, Wt, schemes, x_cal, freq)                  # [E*3, K]
    cost_e = A.measure_costs(mx, d, f, schemes, counts)                     # [E, K] ms per block
    cost = np.repeat(cost_e, 3, axis=0)
    wbytes = np.array([[3 * 0 + (f * d) * mx.storage_bits_per_weight(mx.Scheme.of(s), d if j < 2 else f) / 8
                        for s in schemes] for i in range(E) for j in range(3)])
    budget = E * 3 * f * d * 4.25 / 8
    P = torch.cuda.get_device_properties(0).multi_processor_count
    prob = A.Problem(delta, cost, wbytes, budget, n_sm=P)
    x = bench.to_bf16(bench.gen_activations(T, d, seed=1), "cuda")
    ids = torch.from_numpy(ids_np).cuda()
    w = torch.from_numpy(w_np).cuda()
    ref_layer = mx.MoELayer.from_weights(E, 0, d, f, 0, Wt, [[mx.Scheme.of(C.W16)] * 3] * E)
    y_ref = ref_layer(x, ids, w).float()
    del ref_layer
    out = {"schemes": names, "budget_bits": 4.25, "runs": []}
    for r in (0.0, 0.25, 0.5, 0.75, 1.0):
        a = A.allocate(prob, r)
        table = [[schemes[a.choice[3 * i + j]] for j in range(3)] for i in range(E)]
        lay = mx.MoELayer.from_weights(E, 0, d, f, 0, Wt, [[mx.Scheme.of(s) for s in row] for row in table])
        ws = lay.workspace(T, k)
        yq = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
        for _ in range(3):
            lay(x, ids, w, out=yq, workspace=ws)
        lay.profile(10)
        for _ in range(10):
            lay(x, ids, w, out=yq, workspace=ws)
        gemm = float(np.median(lay.profile_read(10)[:, 3]))
        err = float(torch.linalg.norm(yq.float() - y_ref) / torch.linalg.norm(y_ref))
        hist = {n: int((a.choice == i).sum()) for i, n in enumerate(names)}
        avg_bits = float(sum(wbytes[b, a.choice[b]] for b in range(len(a.choice))) * 8 / (E * 3 * f * d))
        out["runs"].append({"r": r, "model_L": a.L, "model_T_ms": a.T, "avg_bits": avg_bits, "measured_gemm_ms": gemm,
                            "measured_rel_err_vs_bf16": err, "schemes": hist})
        del lay, ws
    s = json.dumps(out, indent=1)
    print(s)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            fh.write(s)


if __name__ == "__main__":
    main()
