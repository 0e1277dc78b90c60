"""Per-wait-site cycle breakdown of the persistent kernel (dev tool): python tools/diag_waits.py CFG TABLE [T]."""
import os, sys
# the counters exist only in a -DMXM_DEBUG_COUNTERS build: tools/variants/lib_diag.so (built on demand)
_here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if "MXM_LIB" not in os.environ:
    os.environ["MXM_LIB"] = os.path.join(_here, "tools", "variants", "lib_diag.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import configs as C
import bench
import paper_2505_05799_b200 as mx
cfg = C.get_config(sys.argv[1]); tb = sys.argv[2] if len(sys.argv) > 2 else "mixed"
T = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.tokens
table = bench.table_for(cfg, tb, T)
W = [[bench.to_bf16(b, "cuda") for b in blk] for blk in bench.gen_weights(cfg)]
L = mx.MoELayer.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, W,
                             [[mx.Scheme.of(s) for s in r] for r in table])
x = bench.to_bf16(bench.gen_activations(T, cfg.hidden, seed=1), "cuda")
ids, w = bench.gen_routing(T, cfg.n_routed, cfg.top_k, seed=0)
ids, w = torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda()
sw = torch.from_numpy(bench.gen_shared_weights(T, cfg.n_shared)).cuda() if cfg.n_shared else None
for _ in range(3): L(x, ids, w, sw)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
buf = torch.zeros(nsm, 16, dtype=torch.int64, device="cuda")
L.debug_counters(buf); L(x, ids, w, sw); torch.cuda.synchronize(); L.debug_counters(None)
c = buf.double().cpu().numpy(); tot = c[:, 15].mean()
names = ["P ring", "P empty", "P dep", "M task", "M acce", "M full", "M aready", "X task", "X full", "E task",
         "E accf", "M issue", "E drain", "M stages", "E hq-dep", "total"]
print(f"{cfg.name} {tb} T={T}: kernel {tot:.0f} cycles (avg per CTA)")
for i, n in enumerate(names):
    if n == "-": continue
    v = c[:, i].mean()
    print(f"  {n:10s} {v:14.0f}  {100*v/tot:6.1f}%" + (f"  (stages/CTA; cycles/stage {tot/v:.0f})" if i == 13 else ""))
