"""Measure the cuBLAS DGEMM ceiling (torch.matmul fp64), same method as MEASURED_PEAKS.json."""
import time, torch
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e9
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(10):
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"dgemm {n}^3 burst: {2*n**3/best/1e9:.2f} TFLOP/s ({best:.2f} ms)")
t0 = time.time(); cnt = 0
e0.record()
while time.time() - t0 < 4.0:
    c = a @ b; cnt += 1
    if cnt % 8 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(f"dgemm sustained: {2*n**3*cnt/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s over {cnt} calls")
for m, k, nn in [(69120, 128, 65408), (128, 69120, 65408), (17280, 128, 16256)]:
    x = torch.randn(m, k, dtype=torch.float64, device="cuda")
    y = torch.randn(k, nn, dtype=torch.float64, device="cuda")
    for _ in range(2): z = x @ y
    torch.cuda.synchronize()
    e0.record(); z = x @ y; e1.record(); torch.cuda.synchronize()
    print(f"dgemm {m}x{k}x{nn}: {2*m*k*nn/e0.elapsed_time(e1)/1e9:.2f} TFLOP/s")
    del x, y, z
