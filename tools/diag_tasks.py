"""Per-task timeline of CTA 0 and per-CTA finish spread (dev tool; needs a -DMXM_TRACE_TASKS build):
python tools/diag_tasks.py CFG [TABLE] [T]
Splits the whole kernel into phases (gate/up, down) with the cycles per MMA stage of each for CTA 0, and shows
how far apart the CTAs finish (the tail of the dynamic queue)."""
import ctypes, os, sys
_here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("MXM_LIB", os.path.join(_here, "tools", "variants", "lib_tasks.so"))
sys.path.insert(0, _here)
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
torch.cuda.synchronize()
lib = ctypes.CDLL(os.environ["MXM_LIB"])
NT, NC = 4096, 160
tt = (ctypes.c_ulonglong * (2 * NT))()
cta = (ctypes.c_ulonglong * (NC * 4))()
assert lib.mxm_debug_trace_tasks(tt, cta) == 0
a = np.frombuffer(tt, dtype=np.uint64).reshape(2, NT).astype(np.int64)
c = np.frombuffer(cta, dtype=np.uint64).reshape(NC, 4).astype(np.int64)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
c = c[:nsm]
n = int(min(c[0, 2], NT))
clk, meta = a[0, :n], a[1, :n]
phase, nst, nt, g128 = meta & 0xFF, (meta >> 8) & 0xFFFFFF, (meta >> 32) & 0xFFFF, (meta >> 48) & 1
dur = np.diff(np.append(clk, clk[-1] + (clk[-1] - clk[-2] if n > 1 else 0)))
# the last task's duration is unknown (no next fetch): estimated from the previous one
t_ns = (c[0, 1] - c[0, 0])
total_clk = clk[-1] + dur[-1] - clk[0]
print(f"{cfg.name} {tb} T={T}: CTA 0 ran {n} MMA tasks, {nst.sum()} stages, {total_clk} cycles ({t_ns / 1e3:.1f} us)")
for ph, name in ((0, "gate/up"), (2, "down")):
    for g in (0, 1):
        m = (phase == ph) & (g128 == g)
        if m.any():
            print(f"  {name:8s} g128={g}: {m.sum():5d} tasks {nst[m].sum():6d} stages {dur[m].sum():10d} cycles "
                  f"({100 * dur[m].sum() / total_clk:5.1f} %) -> {dur[m].sum() / max(nst[m].sum(), 1):7.0f} cycles/stage"
                  f", tokens/tile median {int(np.median(nt[m]))}")
first_down = np.nonzero(phase == 2)[0]
if first_down.size:
    print(f"  first down task at {clk[first_down[0]] - clk[0]} cycles ({100 * (clk[first_down[0]] - clk[0]) / total_clk:.1f} %)")
t0 = c[:, 0].min()
start, end = (c[:, 0] - t0) / 1e3, (c[:, 1] - t0) / 1e3
print(f"CTAs: start spread {start.max() - start.min():.1f} us; end min {end.min():.1f} median {np.median(end):.1f} "
      f"max {end.max():.1f} us; stages per CTA min {c[:, 3].min()} median {int(np.median(c[:, 3]))} max {c[:, 3].max()}; "
      f"tasks per CTA min {c[:, 2].min()} max {c[:, 2].max()}")
print(f"  idle tail (sum over CTAs of end.max - end) / (CTAs x end.max): "
      f"{100 * (end.max() - end).sum() / (len(end) * end.max()):.1f} %")
