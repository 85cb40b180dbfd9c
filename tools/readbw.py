"""Context measurement: achievable pure-READ HBM bandwidth on this B200 with
torch's own reduction kernel (x.sum() over a 7.55 GB fp32 tensor) and a
read+write copy, CUDA events, best of N.  Not used for any reported peak
(bench.py reports against MEASURED_PEAKS.json)."""
import json
import torch

n = 1024 * 3 * 614400
x = torch.rand(n, device="cuda", dtype=torch.float32)
y = torch.empty_like(x)
res = {}
for name, fn, nbytes in (("sum_read", lambda: x.sum(), n * 4), ("copy_rw", lambda: y.copy_(x), 2 * n * 4)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    res[name] = {"ms": best, "GB/s": nbytes / best / 1e6}
print(json.dumps(res))
