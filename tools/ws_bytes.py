"""Workspace bytes of a config's layer at its token count (dev tool): python tools/ws_bytes.py CFG [TABLE]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import configs as C
import bench
import paper_2505_05799_b200 as mx
cfg = C.get_config(sys.argv[1]); tb = sys.argv[2] if len(sys.argv) > 2 else "mixed"
T = cfg.tokens
table = bench.table_for(cfg, tb, T)
W = [[bench.to_bf16(b, "cuda") for b in blk] for blk in bench.gen_weights(cfg)]
L = mx.MoELayer.from_weights(cfg.n_routed, cfg.n_shared, cfg.hidden, cfg.inter, cfg.shared_inter, W,
                             [[mx.Scheme.of(s) for s in r] for r in table])
print(f"{cfg.name} {tb} T={T} k={cfg.top_k}: workspace {L.workspace_bytes(T, cfg.top_k) / 1e9:.3f} GB "
      f"(lib {os.environ.get('MXM_LIB', 'product')})")
