"""Dense TF32 tensor peak on this GPU, measured the way MEASURED_PEAKS.json measures bf16:
torch.matmul of 8192^3 fp32 operands with TF32 tensor cores allowed (2 N^3 flops), best of 10
(burst) and back to back for 4 s (sustained).  Prints one JSON line."""
import json
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    a @ b
    e.record()
    e.synchronize()
    best = min(best, s.elapsed_time(e) / 1e3)
t0 = time.perf_counter()
reps = 0
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
while time.perf_counter() - t0 < 4.0:
    a @ b
    reps += 1
e.record()
e.synchronize()
sus = s.elapsed_time(e) / 1e3 / reps
print(json.dumps({"tf32_tflops": 2 * n ** 3 / best / 1e12, "tf32_tflops_sustained": 2 * n ** 3 / sus / 1e12,
                  "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS), best of 10 / back to back 4 s"}))
