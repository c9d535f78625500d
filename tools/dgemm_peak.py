"""cuBLAS DGEMM (torch.matmul fp64) peak on this B200: burst (best of 10) and
sustained (back to back for 4 s). Prints one JSON line."""
import json, time, torch
N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda")
b = torch.randn(N, N, dtype=torch.float64, device="cuda")
c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1) * 1e-3)
t0 = time.time(); n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; n += 1
    if n % 4 == 0: torch.cuda.synchronize()
e1.record(); e1.synchronize()
sus = e0.elapsed_time(e1) * 1e-3 / n
f = 2.0 * N ** 3
print(json.dumps({"dgemm_n": N, "dgemm_burst_tflops": f / best / 1e12, "dgemm_sustained_tflops": f / sus / 1e12}))
