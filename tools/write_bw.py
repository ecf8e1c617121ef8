"""HBM write-only and read-only bandwidth on this GPU (context for K1, whose traffic is ~90% writes):
torch fill_ (write-only), sum (read-only) and copy_ (read+write, the MEASURED_PEAKS recipe) over 4 GiB,
CUDA events, best of 10. Usage: python tools/write_bw.py"""
import json
import torch

N = 1 << 30  # fp32 elements = 4 GiB
x = torch.empty(N, device="cuda", dtype=torch.float32)
y = torch.empty(N, device="cuda", dtype=torch.float32)
x.fill_(1.0)
y.fill_(2.0)
res = {}
for name, fn, nbytes in [("write_fill", lambda: x.fill_(3.0), 4 * N),
                         ("read_sum", lambda: x.sum(), 4 * N),
                         ("copy", lambda: y.copy_(x), 8 * N)]:
    best = 1e9
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    res[name] = round(nbytes / best / 1e9, 1)
print(json.dumps({"GB_per_s": res, "bytes": 4 * N}))
