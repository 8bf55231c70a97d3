"""PCIe copy bandwidth of the GPU box (pinned host memory, 1 GiB copies): the roofline of
the bench e2e keys."""
import torch, time
d = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
for name, f in (("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): f()
    torch.cuda.synchronize()
    print(name, round(10 * (1 << 30) / (time.perf_counter() - t) / 1e9, 1), "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True); d2 = torch.empty_like(d)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("duplex D2H+H2D each", round(10 * (1 << 30) / dt / 1e9, 1), "GB/s")
