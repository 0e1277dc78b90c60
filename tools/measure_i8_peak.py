"""Measure the dense int8 tensor peak on this B200 (torch._int_mm 8192^3, best of 10 CUDA-event timings)."""
import json, os, sys
import torch
M = N = K = 8192
a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 128, (K, N), dtype=torch.int8, device="cuda")
for _ in range(3):
    torch._int_mm(a, b)
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); torch._int_mm(a, b); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
tops = 2 * M * N * K / (best / 1e3) / 1e12
x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16); y = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3): x @ y
bb = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); x @ y; e.record(); torch.cuda.synchronize(); bb = min(bb, s.elapsed_time(e))
out = {"i8_tops": tops, "bf16_tflops_same_run": 2 * M * N * K / (bb / 1e3) / 1e12, "how": "torch._int_mm / torch.matmul 8192^3 best of 10, CUDA events", "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
os.makedirs("profiles", exist_ok=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/i8_peak.json", "w"), indent=1)
