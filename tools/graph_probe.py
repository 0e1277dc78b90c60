"""Does mxm_moe_group_gemm capture into a CUDA graph, and what does replay save at small T? (dev probe)
python tools/graph_probe.py CFG T"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import configs as C
import bench
import paper_2505_05799_b200 as mx
cfg = C.get_config(sys.argv[1]); T = int(sys.argv[2])
table = bench.table_for(cfg, "mixed", T)
W = [[bench.to_bf16(b, "cuda") for b in blk] for blk in bench.gen_weights(cfg)]
L = mx.MoELayer.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, W,
                             [[mx.Scheme.of(s) for s in r] for r in table])
x = bench.to_bf16(bench.gen_activations(T, cfg.hidden, seed=1), "cuda")
ids, w = bench.gen_routing(T, cfg.n_routed, cfg.top_k, seed=0)
ids, w = torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda()
sw = torch.from_numpy(bench.gen_shared_weights(T, cfg.n_shared)).cuda() if cfg.n_shared else None
ws = L.workspace(T, cfg.top_k)
out = torch.empty(T, cfg.hidden, dtype=torch.bfloat16, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        L(x, ids, w, sw, workspace=ws, out=out)
torch.cuda.synchronize()
ref = out.clone()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    L(x, ids, w, sw, workspace=ws, out=out)
out.zero_()
g.replay(); torch.cuda.synchronize()
print("graph replay equals eager:", torch.equal(out, ref))
def timeit(fn, n=200):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(10): fn()
    torch.cuda.synchronize(); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
with torch.cuda.stream(s):
    te = timeit(lambda: L(x, ids, w, sw, workspace=ws, out=out))
    tg = timeit(lambda: g.replay())
print(f"{cfg.name} T={T}: eager {te:.1f} us per call, graph replay {tg:.1f} us (back-to-back, L2 warm)")
