"""Write-only and copy HBM bandwidth on this B200 (16 GiB buffers, CUDA events, best of 5)."""
import json, torch
n = 16 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda")
b = torch.empty(n, dtype=torch.uint8, device="cuda")
def best(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
tw = best(lambda: a.fill_(1))
tz = best(lambda: a.zero_())
tc = best(lambda: b.copy_(a))
print(json.dumps({"write_fill_gbs": n / tw / 1e6, "write_zero_gbs": n / tz / 1e6, "copy_rw_gbs": 2 * n / tc / 1e6,
                  "bytes": n}))
