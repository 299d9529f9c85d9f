"""Copy-engine H2D vs SM loads from the same pinned buffer (UVA alias, an elementwise
kernel reading it over PCIe), sampled over time to catch the link's slow and fast
states."""
import time
import torch

NB = 3510000
x = torch.empty(NB // 4).pin_memory()
x.normal_()
d = torch.empty(NB // 4, device="cuda")


class Alias:
    def __init__(self, t):
        self.__cuda_array_interface__ = {"data": (t.data_ptr(), False), "shape": tuple(t.shape), "typestr": "<f4",
                                         "version": 2}


xa = torch.as_tensor(Alias(x), device="cuda")
st = torch.cuda.Stream()


def timed(fn):
    with torch.cuda.stream(st):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
    return NB / a.elapsed_time(b) / 1e6


torch.mul(xa, 1.0, out=d)
torch.cuda.synchronize()
assert torch.equal(d.cpu(), x)
big = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
t0 = time.time()
for i in range(40):
    if i % 10 >= 5:
        big.zero_()
        torch.cuda.synchronize()
    ce = timed(lambda: d.copy_(x, non_blocking=True))
    sm = timed(lambda: torch.mul(xa, 1.0, out=d))
    ce2 = timed(lambda: d.copy_(x, non_blocking=True))
    print(f"t={time.time() - t0:6.3f}s  CE {ce:5.1f}  SM-load {sm:5.1f}  CE {ce2:5.1f} GB/s")
    if i % 10 == 9:
        time.sleep(0.2)
