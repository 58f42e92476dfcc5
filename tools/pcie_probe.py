"""Host<->device copy bandwidth: H2D alone, D2H alone, both at once (pinned)."""
import time
import torch
n = 335544320 // 8
a = torch.empty(n, dtype=torch.float64).pin_memory()
b = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, k=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
def h2d():
    with torch.cuda.stream(s1): d1.copy_(a, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): b.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
mb = n * 8 / 1e6
for nm, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{nm}: {ms:.2f} ms  {mb * (2 if nm == 'both' else 1) / ms:.1f} GB/s total", flush=True)
print(torch.cuda.get_device_name(), flush=True)
