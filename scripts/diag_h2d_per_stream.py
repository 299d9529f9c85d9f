"""H2D / D2H rate of a 3.51 MB pinned buffer per CUDA stream: does the copy engine a
stream is bound to decide the rate?"""
import torch

NB = 3510000
x = torch.empty(NB // 4).pin_memory()
d = torch.empty(NB // 4, device="cuda")


def rate(st, reps=10):
    with torch.cuda.stream(st):
        for _ in range(2):
            d.copy_(x, non_blocking=True)
        st.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            d.copy_(x, non_blocking=True)
        b.record(st)
        b.synchronize()
        ms = a.elapsed_time(b) / reps
        a.record(st)
        for _ in range(reps):
            x.copy_(d, non_blocking=True)
        b.record(st)
        b.synchronize()
        ms2 = a.elapsed_time(b) / reps
    return f"h2d {NB / ms / 1e6:5.1f} GB/s | d2h {NB / ms2 / 1e6:5.1f} GB/s"


for rnd in range(2):
    print("default stream:", rate(torch.cuda.default_stream()))
    for i in range(12):
        st = torch.cuda.Stream()
        print(f"round {rnd} torch.cuda.Stream() #{i} handle {st.cuda_stream:#x}:", rate(st))
