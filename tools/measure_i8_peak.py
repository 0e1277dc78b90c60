"""Measure the dense int8 and fp8 (e4m3) tensor peaks on this B200: torch._int_mm / torch._scaled_mm 8192^3, best
of 10 CUDA-event timings; bf16 torch.matmul in the same run for reference. Writes profiles/i8_peak.json (or argv[1])."""
import json, os, sys
import torch
M = N = K = 8192


def best_ms(fn, n=10):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(n):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


tflop = 2 * M * N * K / 1e12
a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 128, (K, N), dtype=torch.int8, device="cuda")
i8 = tflop / (best_ms(lambda: torch._int_mm(a, b)) / 1e3)
x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16); y = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
bf = tflop / (best_ms(lambda: x @ y) / 1e3)
f8 = None
try:
    xa = torch.randn(M, K, device="cuda").to(torch.float8_e4m3fn)
    yb = torch.randn(N, K, device="cuda").to(torch.float8_e4m3fn).t()
    one = torch.ones((), device="cuda")
    f8 = tflop / (best_ms(lambda: torch._scaled_mm(xa, yb, one, one, out_dtype=torch.bfloat16)) / 1e3)
except Exception as ex:  # noqa: BLE001
    print("fp8 measurement failed:", ex)
out = {"i8_tops": i8, "f8_tflops": f8, "bf16_tflops_same_run": bf,
       "how": "torch._int_mm / torch._scaled_mm (e4m3, bf16 out) / torch.matmul 8192^3 best of 10, CUDA events",
       "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
os.makedirs("profiles", exist_ok=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/i8_peak.json", "w"), indent=1)
