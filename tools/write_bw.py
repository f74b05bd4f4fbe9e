"""Pure-write and read+write HBM bandwidth of this B200 at the EXP_finite output size (512^3 fine level, 1.08 GB):
torch fill_ (write only) and copy_ (read + write), CUDA events, best of 10. The realistic roofline of a
write-dominated kernel (EXP_finite writes 8 B per fine node and reads ~1.1 B)."""
import json
import torch

n = 513 ** 3
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def best(fn, reps=10):
    t = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        t = min(t, e0.elapsed_time(e1))
    return t


tf = best(lambda: a.fill_(1.5))
tc = best(lambda: b.copy_(a))
print(json.dumps({"bytes": n * 8, "fill_ms": tf, "fill_write_gbs": n * 8 / tf / 1e6,
                  "copy_ms": tc, "copy_rw_gbs": 2 * n * 8 / tc / 1e6}))
