"""H2D rate of one pinned 3.51 MB buffer over time in one process: (a) left alone,
(b) rewritten by the CPU before each measurement, (c) after GPU compute bursts."""
import time
import torch

NB = 3510000
x = torch.empty(NB // 4).pin_memory()
y = torch.empty(NB // 4).pin_memory()
d = torch.empty(NB // 4, device="cuda")
big = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()


def h2d(t, reps=5):
    with torch.cuda.stream(st):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            d.copy_(t, non_blocking=True)
        b.record(st)
        b.synchronize()
    return NB / (a.elapsed_time(b) / reps) / 1e6


t0 = time.time()
for phase, n in (("alone", 12), ("cpu-rewritten", 8), ("alone", 6), ("after memset burst", 8), ("after 50 ms sleep", 8),
                 ("single copy, sync each", 8)):
    out = []
    for i in range(n):
        if phase == "cpu-rewritten":
            x.add_(1.0)
        if phase == "after memset burst":
            big.zero_()
            torch.cuda.synchronize()
        if phase == "after 50 ms sleep":
            time.sleep(0.05)
        out.append(h2d(x, 1 if phase.startswith("single") else 5))
    print(f"t={time.time() - t0:6.3f}s {phase:24s}: " + " ".join(f"{v:5.1f}" for v in out) + " GB/s")
print("other buffer y (never DMA-read):", " ".join(f"{h2d(y):5.1f}" for _ in range(4)))
