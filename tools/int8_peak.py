"""Measure the dense INT8 tensor-core throughput of this B200 with cuBLASLt
(torch._int_mm, s8 x s8 -> s32), the denominator for the prefill GEMM's
roofline (MEASURED_PEAKS.json has only bf16).  Prints one JSON line."""
import json

import torch

n = 8192
a = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda").t()   # column-major B
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
# sustained: back to back for ~3 s
it = max(1, int(3000 / best))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(it):
    torch._int_mm(a, b)
e1.record()
torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / it
fl = 2.0 * n ** 3
print(json.dumps({"int8_tops_burst": round(fl / best / 1e9, 1),
                  "int8_tops_sustained": round(fl / sus / 1e9, 1),
                  "how": "torch._int_mm (cuBLASLt IMMA) 8192^3 s8xs8->s32, best of 10 / back to back 3 s"}))
