"""Diagnostic: per-scheme parity errors on the tiny config (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from synth import configs as C
from tests.moe_cases import gpu_layer, gpu_run, make_case, oracle_layer, oracle_run, row_rel_err
import paper_2505_05799_b200 as mx

TINY = C.get_config("tiny")
ALL = ([C.W16] + [C.WO(b, g, s) for b in (2, 3, 4, 8) for g in (64, 128, -1) for s in (False, True)]
       + [C.WA(b, g) for b in (4, 5, 8) for g in (128, -1)])
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "uniform"):
    for sch in ALL:
        case = make_case(TINY, C.uniform_table(TINY, sch), 64, seed=2)
        L = gpu_layer(case); y = gpu_run(L, case); ref = oracle_run(oracle_layer(case), case)
        print(f"{sch.name():22s} err={row_rel_err(y, ref):.4g}  stats={L.task_stats(64, 2)}", flush=True)
if which in ("all", "mixed"):
    case = make_case(TINY, C.precision_table(TINY), 64)
    L = gpu_layer(case); y = gpu_run(L, case); ref = oracle_run(oracle_layer(case), case)
    print("mixed", row_rel_err(y, ref))
    # per-expert attribution: route every token only to expert e
    for e in range(4):
        ids = np.full((64, 2), -1, np.int32); ids[:, 0] = e
        w = np.zeros((64, 2), np.float32); w[:, 0] = 1
        y = gpu_run(L, case, ids=ids, w=w); ref = oracle_run(oracle_layer(case), case, ids=ids, w=w)
        print("expert", e, [s.name() for s in case["table"][e]], row_rel_err(y, ref))
