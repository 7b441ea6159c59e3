"""Measure host<->device copy bandwidth with pinned buffers (e2e ceiling)."""
import time, torch
n = 1 << 30  # 4 GiB of int32
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
d = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); t = time.perf_counter() - t
    print(name, round(4 * n / t / 1e9, 1), "GB/s")
h2 = torch.empty(n, dtype=torch.int32, pin_memory=True)
d2 = torch.empty(n, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter() - t
print("bidir", round(8 * n / t / 1e9, 1), "GB/s total")
# chunked d2h 32 MiB pieces on 3 streams
ss = [torch.cuda.Stream() for _ in range(3)]
piece = 8 << 20
torch.cuda.synchronize(); t = time.perf_counter()
for i in range(0, n, piece):
    with torch.cuda.stream(ss[(i // piece) % 3]):
        h[i:i + piece].copy_(d[i:i + piece], non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter() - t
print("d2h 32MiB pieces", round(4 * n / t / 1e9, 1), "GB/s")
# the e2e pattern: D2H of 4 B/int concurrent with H2D of ~1 B/int (C5 words)
m = n // 4
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
with torch.cuda.stream(s2): d2[:m].copy_(h2[:m], non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter() - t
print("d2h 4GiB + concurrent h2d 1GiB:", round(4 * n / t / 1e9, 1), "GB/s d2h-equivalent")
