"""Does CPU access to a pinned buffer right before a DMA slow the DMA down?"""
import time, threading, torch, numpy as np
n = 21 * 160160
d = torch.empty(n, dtype=torch.float64, device="cuda")
p = torch.empty(n, dtype=torch.float64, pin_memory=True)
a = p.numpy()
store = np.empty(n)
store.fill(0)
def gpu_ms(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(); fn(); e1.record(); e1.synchronize()
    return e0.elapsed_time(e1)
def par(fn, t=16):
    th = [threading.Thread(target=fn, args=(k, t)) for k in range(t)]
    [x.start() for x in th]; [x.join() for x in th]
def read_slices(k, t):
    lo, hi = n * k // t, n * (k + 1) // t
    store[lo:hi] = a[lo:hi]
def write_slices(k, t):
    lo, hi = n * k // t, n * (k + 1) // t
    a[lo:hi] = 1.0
for label, pre in [("idle", lambda: None), ("cpu read 1 thread", lambda: store.__setitem__(slice(None), a)),
                   ("cpu read 16 threads", lambda: par(read_slices)), ("cpu write 1 thread", lambda: a.fill(2.0)),
                   ("cpu write 16 threads", lambda: par(write_slices))]:
    for direction in ("d2h", "h2d"):
        ts = []
        for _ in range(5):
            pre()
            ts.append(gpu_ms((lambda: p.copy_(d, non_blocking=True)) if direction == "d2h" else (lambda: d.copy_(p, non_blocking=True))))
        print(f"{label:22s} {direction}: " + " ".join(f"{t:.3f}" for t in ts), flush=True)
