"""Measure the dense int8 tensor-core peak on this B200 with cuBLAS (torch._int_mm), the same way
MEASURED_PEAKS.json measures bf16: 8192^3, best of 10 (burst) and back-to-back for ~3 s
(sustained).  Writes profiles/int8_peak.json, which bench.py uses as the roofline peak of
the int8 CRSS kernel."""
import json
import os
import sys
import time

import torch

n = 8192
a = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); torch._int_mm(a, b); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 1e3)
burst = 2 * n ** 3 / best / 1e12
t0 = time.perf_counter(); it = 0
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
while time.perf_counter() - t0 < 3.0:
    torch._int_mm(a, b); it += 1
e.record(); torch.cuda.synchronize()
sustained = 2 * n ** 3 * it / (s.elapsed_time(e) / 1e3) / 1e12
out = {"int8_tops_burst": burst, "int8_tops_sustained": sustained, "how": "torch._int_mm (cuBLASLt IMMA) "
       "8192^3 int8 x int8 -> int32: best of 10 (burst), back to back for 3 s (sustained)",
       "gpu": torch.cuda.get_device_name(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "int8_peak.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
