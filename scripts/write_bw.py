"""Calibration: HBM bandwidth of a pure write stream (16 GiB fill) vs the
read+write copy that MEASURED_PEAKS.json reports, on the same GPU."""
import json
import torch

n = 1 << 31  # float64 elements = 16 GiB
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n // 2, dtype=torch.float64, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for name, fn, nbytes in (("fill_16GiB", lambda: x.fill_(1.0), 8 * n),
                         ("zero_16GiB", lambda: x.zero_(), 8 * n),
                         ("copy_8GiB", lambda: y.copy_(x[: n // 2]), 2 * 8 * (n // 2))):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(10):
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    res[name] = {"ms": round(best, 3), "GBps": round(nbytes / best / 1e6, 1)}
print(json.dumps(res))
