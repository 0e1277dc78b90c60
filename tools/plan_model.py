"""Host replay of plan.cu's tiling for a config: padded MMA work, stages and ideal times (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import configs as C
from synth.gen import gen_routing

def pow2(m): return 16 if m <= 16 else 32 if m <= 32 else 64 if m <= 64 else 128

def model(name, T=None, table="mixed", clock=1.85e9):
    cfg = C.get_config(name); T = T or cfg.tokens
    tab = C.precision_table(cfg, T) if table == "mixed" else None
    ids, _ = gen_routing(T, cfg.n_routed, cfg.top_k, seed=0)
    cnt = np.bincount(ids.reshape(-1), minlength=cfg.n_routed).tolist() + [T] * cfg.n_shared
    mma_cyc = 0.0; real = 0.0; stages = 0; tasks = 0
    for v, m in enumerate(cnt):
        if m == 0: continue
        f = cfg.inter if v < cfg.n_routed else cfg.shared_inter
        s = tab[v] if tab else [C.W16] * 3
        i8 = s[0].a_bits != 16
        dual = (s[0].a_bits == 16 and s[1].a_bits == 16) or (s[0] == s[1])
        g128 = i8 and s[0].w_group == 128
        cap = 64 if (not dual or g128) else 128
        tiles = [cap] * (m // cap) + ([pow2(m % cap)] if m % cap else []) if m > cap else [pow2(m)]
        for nt in tiles:
            rate = 8192 if i8 else 4096
            # phase 0: f/128 tasks x (2 mats x 128 x nt x d) MACs
            mma_cyc += (f // 128) * 2 * 128 * nt * cfg.hidden / rate
            stages += (f // 128) * cfg.hidden // (128 if i8 else 64)
            i8d = s[2].a_bits != 16
            mma_cyc += (cfg.hidden // 128) * 128 * nt * f / (8192 if i8d else 4096)
            stages += (cfg.hidden // 128) * f // (128 if i8d else 64)
            tasks += f // 128 + cfg.hidden // 128
        real += 6.0 * m * cfg.hidden * f / 2
    P = 148
    print(f"{name} T={T}: tasks {tasks}, stages/CTA {stages/P:.0f}, padded MMA cycles/CTA {mma_cyc/P:.0f} "
          f"-> ideal {mma_cyc/P/clock*1e3:.3f} ms at {clock/1e9:.2f} GHz; real MAC efficiency {real/(mma_cyc*0 + 1) if False else real/ (mma_cyc * (4096)) if False else 0}")
    print(f"   padding overhead: padded/real MACs = {mma_cyc*4096/real if not any(s[0].a_bits!=16 for s in (tab or [[C.W16]])) else float('nan'):.3f}")

if __name__ == "__main__":
    model(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "mixed")
