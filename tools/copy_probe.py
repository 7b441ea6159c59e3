"""Developer: device-to-device copy time at C1's traffic (read + write = 363 MB) and other sizes,
for context on small-batch roofline fractions (the measured peak is taken on a 4 GiB copy)."""
import torch
for mb in (45, 90, 181, 362, 724, 2896):
    n = mb * (1 << 20) // 4
    a = torch.empty(n, dtype=torch.int32, device="cuda"); b = torch.empty_like(a)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(12):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[len(ts) // 2]
    print(f"copy {mb} MiB (traffic {2 * mb} MiB): {t * 1e3:.1f} us, {2 * n * 4 / t / 1e6:.0f} GB/s")
