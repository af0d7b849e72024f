"""HBM write-only and read+write bandwidth on this GPU (torch fill / copy of
buffers far larger than L2), to bound output-heavy kernels (quad12 gradFD
writes 2.4 KB per knot and reads 288 B)."""
import json
import torch

n = 2_818_572_288 // 8  # quad12 gradFD fp64 at N = 2^20: bytes per launch
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for name, fn, nbytes in (("write (fill_)", lambda: a.fill_(1.0), 8 * n),
                         ("read+write (copy_)", lambda: b.copy_(a), 16 * n)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    res[name] = {"ms": ms, "GB/s": nbytes / (ms * 1e-3) / 1e9}
print(json.dumps(res))
