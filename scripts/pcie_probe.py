"""PCIe copy rates on this box (pinned / pageable, H2D / D2H) for the e2e budget."""
import time, torch
n = 21 * 160160
d = torch.empty(n, dtype=torch.float64, device="cuda")
for pinned in (True, False):
    h = torch.empty(n, dtype=torch.float64, pin_memory=pinned)
    h.fill_(1.0)
    for direction in ("d2h", "h2d"):
        ts = []
        for _ in range(8):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if direction == "d2h":
                h.copy_(d, non_blocking=pinned)
            else:
                d.copy_(h, non_blocking=pinned)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[len(ts) // 2]
        print(f"pinned={pinned} {direction}: {n * 8 / 1e6:.1f} MB in {t * 1e3:.3f} ms = {n * 8 / t / 1e9:.1f} GB/s", flush=True)
import os
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
# Does an idle gap slow the next copy (link power state)?
hp = torch.empty(n, dtype=torch.float64, pin_memory=True)
for gap in (0.0, 0.002, 0.005, 0.01, 0.05, 0.2):
    for direction in ("h2d", "d2h"):
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            time.sleep(gap)
            t0 = time.perf_counter()
            if direction == "d2h":
                hp.copy_(d, non_blocking=True)
            else:
                d.copy_(hp, non_blocking=True)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"gap {gap * 1e3:5.1f} ms {direction}: " + " ".join(f"{t:.3f}" for t in ts), flush=True)
# Busy GPU (kernels, no PCIe traffic) for 5 ms, then the copy.
x = torch.randn(4096, 4096, device="cuda")
for direction in ("d2h", "h2d"):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        for _ in range(20):
            x = x @ x * 1e-3
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if direction == "d2h":
            hp.copy_(d, non_blocking=True)
        else:
            d.copy_(hp, non_blocking=True)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"after compute {direction}: " + " ".join(f"{t:.3f}" for t in ts), flush=True)
