"""H2D of config 1's V (3.51 MB, pinned) as k concurrent chunk copies on k streams:
does the box's host link read faster with more DMA streams in flight?"""
import torch

N = 3510000 // 4
x = torch.empty(N).pin_memory()
d = torch.empty(N, device="cuda")
main = torch.cuda.Stream()
for k in (1, 2, 3, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    cuts = [N * i // k for i in range(k + 1)]

    def run():
        ev = torch.cuda.Event()
        ev.record(main)
        done = []
        for i, st in enumerate(streams):
            st.wait_event(ev)
            with torch.cuda.stream(st):
                d[cuts[i]:cuts[i + 1]].copy_(x[cuts[i]:cuts[i + 1]], non_blocking=True)
                e = torch.cuda.Event()
                e.record(st)
                done.append(e)
        for e in done:
            main.wait_event(e)

    for _ in range(5):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        run()
        b.record(main)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"k={k}: median {ts[15]:.4f} ms  min {ts[0]:.4f} ms  {N * 4 / ts[15] / 1e6:.1f} GB/s")
# sizes: is it latency or bandwidth?
for mb in (0.25, 1, 3.51, 16, 64):
    n = int(mb * 1e6 / 4)
    xx = torch.empty(n).pin_memory()
    dd = torch.empty(n, device="cuda")
    for _ in range(3):
        dd.copy_(xx, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        dd.copy_(xx, non_blocking=True)
    b.record()
    b.synchronize()
    t = a.elapsed_time(b) / 10
    a.record()
    for _ in range(10):
        xx.copy_(dd, non_blocking=True)
    b.record()
    b.synchronize()
    t2 = a.elapsed_time(b) / 10
    print(f"{mb} MB: h2d {t:.4f} ms {n * 4 / t / 1e6:.1f} GB/s   d2h {t2:.4f} ms {n * 4 / t2 / 1e6:.1f} GB/s")
