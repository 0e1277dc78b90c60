"""Per-stage event timeline of CTA 0 (dev tool; needs a -DMXM_TRACE build): python tools/diag_trace.py CFG [TABLE]
Events: 0 producer issues stage loads, 1 transform has the stage (full), 2 transform arrived aready,
3 MMA starts issuing the stage, 4 MMA finished issuing, 5 epilogue has the accumulator, 6 epilogue released it."""
import ctypes, os, sys
_here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("MXM_LIB", os.path.join(_here, "tools", "variants", "lib_trace.so"))
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
buf = (ctypes.c_ulonglong * (13 * 2048))()
lib.mxm_debug_trace(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(13, 2048).astype(np.int64)
n = int(min((a[3] > 0).sum(), (a[1] > 0).sum(), 1500))
t0 = a[0, 0]
print(f"{cfg.name} {tb}: first {n} stages of CTA 0 (cycles relative to the first load)")
print(" st   load   xf_has  xf_rdy  mma_s  mma_e | xf(has->rdy) mma(iss) wait(rdy->mma_s) gap(mma_e->next mma_s) load->has")
for i in list(range(0, 12)) + list(range(n // 2, n // 2 + 12)):
    r = a[:, i] - t0
    nx = a[3, i + 1] - t0 if i + 1 < n else r[4]
    print(f"{i:4d} {r[0]:7d} {r[1]:7d} {r[2]:7d} {r[3]:7d} {r[4]:7d} | {r[2]-r[1]:7d} {r[4]-r[3]:7d} {r[3]-r[2]:7d} {nx-r[4]:7d} {r[1]-r[0]:7d}")
d = lambda i, j: np.median(a[j, :n] - a[i, :n])
per = np.median(np.diff(a[3, :n]))
ne = int(min((a[5] > 0).sum(), (a[6] > 0).sum(), 1500))
print(" ev  epi_has  epi_done | drain  has->prev_done")
for i in list(range(0, 12)) + list(range(ne // 2, ne // 2 + 12)):
    r = a[:, i] - t0
    print(f"{i:4d} {r[5]:8d} {r[6]:8d} | {r[6]-r[5]:6d} {(r[5] - (a[6, i-1]-t0)) if i else 0:6d}")
if (a[7] > 0).sum() > 10:
    print(f"epilogue split (median): accf->sfull {np.median(a[7,:ne]-a[5,:ne]):.0f} sfull->restaged {np.median(a[8,:ne]-a[7,:ne]):.0f}"
          f" drain {np.median(a[9,:ne]-a[8,:ne]):.0f} drain_end->released {np.median(a[6,:ne]-a[9,:ne]):.0f}")
print(f"median per-event epilogue interval {np.median(np.diff(a[5, :ne])):.0f}; drain {np.median(a[6, :ne]-a[5, :ne]):.0f}")
print(f"median per-stage MMA start interval {per:.0f}; transform has->ready {d(1,2):.0f}; MMA issue {d(3,4):.0f}; "
      f"ready->MMA start {d(2,3):.0f}; load issue->transform has {d(0,1):.0f}")
if len(sys.argv) > 4 and sys.argv[4] == "full":
    print("steady-state rows (all events, same index = same stage for uniform g128 tables), cycles rel. to row 0 load")
    b = a[:, 700]
    print("  i    load  xf_has  xf_rdy   mma_s   mma_e  e_has   e_sr  e_drn0  e_drn1  e_done")
    for i in range(700, 716):
        r = a[:, i] - b[0]
        print(f"{i:4d} {r[0]:7d} {r[1]:7d} {r[2]:7d} {r[3]:7d} {r[4]:7d} {r[5]:7d} {r[7]:7d} {r[8]:7d} {r[9]:7d} {r[6]:7d}")

nm = int(min((a[12] > 0).sum(), (a[5] > 0).sum(), (a[10] > 0).sum(), 1500))
if nm > 20:
    ev = np.arange(200, min(nm, 1400))
    commit, has, done = a[12, ev], a[5, ev], a[6, ev]
    wait_s, wait_e = a[10, ev + 2], a[11, ev + 2]  # MMA of event e+2 waits for the drain of event e (same buffer)
    print("event-indexed (median over events 200..): MMA commit -> epilogue has %.0f | epilogue has -> done %.0f |"
          " done -> MMA(e+2) wait end %.0f | MMA(e+2) wait %.0f | event period %.0f" % (
          np.median(has - commit), np.median(done - has), np.median(wait_e - done), np.median(wait_e - wait_s),
          np.median(np.diff(a[12, ev]))))

if os.environ.get("TRACE_PRODUCER"):
    ev = np.arange(200, 1400)
    print("producer (median): stage start -> empty passed %.0f | empty -> before scale wait %.0f | sempty wait %.0f |"
          " stage period %.0f" % (np.median(a[0, ev] - a[7, ev]), np.median(a[8, ev] - a[0, ev]),
                                  np.median(a[9, ev] - a[8, ev]), np.median(np.diff(a[7, ev]))))
