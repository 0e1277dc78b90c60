"""Crash isolation for mixed tables (dev tool): python tools/diag_mix.py E d f T k SPEC
SPEC: comma list per expert of wo4 / wa8 / wa4g (w4a4-g128) / w16, cycled over experts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import configs as C
from synth.gen import gen_activations, gen_routing, gen_weight, weight_seed
import paper_2505_05799_b200 as mx
E, d, f, T, k = map(int, sys.argv[1:6])
spec = sys.argv[6].split(",")
M = {"wo4": C.WO(4, 128), "wa8": C.WA(8, -1), "wa4g": C.WA(4, 128), "w16": C.W16, "wo2": C.WO(2, -1)}
table = [[M[spec[e % len(spec)]]] * 3 for e in range(E)]
def bf(b): return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).cuda()
W = [[bf(gen_weight(f, d, weight_seed(e, 0))), bf(gen_weight(f, d, weight_seed(e, 1))), bf(gen_weight(d, f, weight_seed(e, 2)))]
     for e in range(E)]
L = mx.MoELayer.from_weights(E, 0, d, f, 0, W, [[mx.Scheme.of(s) for s in r] for r in table])
x = bf(gen_activations(T, d, seed=1))
ids, w = gen_routing(T, E, k, seed=0)
print("counts", np.bincount(ids.ravel(), minlength=E).tolist(), flush=True)
y = L(x, torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda(), None)
torch.cuda.synchronize()
yn = torch.isnan(y.float()).any(dim=1).cpu().numpy()
bad = np.nonzero(yn)[0]
ex_bad = np.bincount(ids[bad].ravel(), minlength=E).tolist() if bad.size else []
print("ok", L.poll_error(), L.task_stats(T, k), "nan_rows", int(bad.size), "nan_by_expert", ex_bad, "first", bad[:8].tolist())
# workspace-fill experiment: NaN that depends on the fill means reading memory the kernels did not write
if os.environ.get("FILLTEST"):
    ws = L.workspace(T, k)
    ids_d, w_d = torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda()
    outs = {}
    for name, val in (("nanfill", 0xFF), ("zerofill", 0), ("zerofill2", 0), ("nanfill2", 0xFF)):
        for rep in range(3):
            ws.view(torch.uint8).fill_(val)
            y = L(x, ids_d, w_d, None, workspace=ws)
            torch.cuda.synchronize()
            yf = y.float()
            nanr = torch.isnan(yf).any(dim=1)
            outs.setdefault(name, []).append(yf.clone())
            print(name, rep, "nan_rows", int(nanr.sum()), flush=True)
    z = outs["zerofill"][0]
    for name, ys in outs.items():
        for i, yy in enumerate(ys):
            dif = (torch.nan_to_num(yy, 1e9) - z).abs().max(dim=1).values
            print("vs zerofill0", name, i, "rows differing", int((dif > 0).sum()))
if os.environ.get("NANTEST"):
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    for rep in range(4):
        buf = torch.zeros(149 * 16, dtype=torch.int64, device="cuda")
        L.debug_counters(buf)
        y = L(x, torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda(), None)
        torch.cuda.synchronize()
        L.debug_counters(None)
        info = buf[148 * 16: 148 * 16 + 8].cpu().tolist()
        print("nan rows", int(torch.isnan(y.float()).any(dim=1).sum()), "info [site, expert, phase, ntile, ks/col, row0, block, extra]", info, hex(info[7] & 0xffffffff))

if os.environ.get("NANTEST2"):
    import ctypes
    lib = ctypes.CDLL(os.environ["MXM_LIB"])
    for rep in range(6):
        y = L(x, torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda(), None)
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * 8)()
        lib.mxm_debug_nan_info(buf)
        info = list(buf)
        print("nan rows", int(torch.isnan(y.float()).any(dim=1).sum()), "info [site, expert, phase, ntile, ks/col, row0, block, extra]", info, hex(info[7] & 0xffffffff), flush=True)
