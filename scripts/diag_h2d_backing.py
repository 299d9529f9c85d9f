"""H2D rate of a 3.51 MB pinned buffer by how its pages are backed: torch's pinned
allocator (several live allocations) vs an aligned anonymous mapping with
MADV_HUGEPAGE, touched, then cudaHostRegister'ed."""
import ctypes as C
import mmap
import numpy as np
import torch

NB = 3510000
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      "| defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
d = torch.empty(NB // 4, device="cuda")
rt = torch.cuda.cudart()


def rate(t, reps=20):
    for _ in range(3):
        d.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        d.copy_(t, non_blocking=True)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    a.record()
    for _ in range(reps):
        t.copy_(d, non_blocking=True)
    b.record()
    b.synchronize()
    ms2 = a.elapsed_time(b) / reps
    return f"h2d {ms:.4f} ms {NB / ms / 1e6:5.1f} GB/s | d2h {ms2:.4f} ms {NB / ms2 / 1e6:5.1f} GB/s"


keep = []
for i in range(6):
    t = torch.empty(NB // 4).pin_memory()
    keep.append(t)
    print(f"torch pin_memory #{i} ptr%2M={t.data_ptr() % (2 << 20):#x}:", rate(t))
for i in range(3):
    t = torch.empty(NB // 4, pin_memory=True)
    keep.append(t)
    print(f"torch.empty(pin_memory=True) #{i}:", rate(t))

libc = C.CDLL(None, use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
HP = 2 << 20
for huge in (False, True):
    for i in range(3):
        size = (NB + HP - 1) // HP * HP
        raw = libc.mmap(None, size + HP, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
        base = (raw + HP - 1) // HP * HP
        if huge:
            r = libc.madvise(base, size, 14)  # MADV_HUGEPAGE
            assert r == 0, C.get_errno()
        C.memset(base, 1, size)  # touch: fault the pages in
        err = rt.cudaHostRegister(base, size, 0)
        assert int(err) == 0, err
        arr = np.ctypeslib.as_array((C.c_float * (NB // 4)).from_address(base))
        t = torch.from_numpy(arr)
        assert t.is_pinned()
        keep.append(t)
        print(f"mmap{' + MADV_HUGEPAGE' if huge else ''} + cudaHostRegister #{i}:", rate(t))
try:
    ah = [l for l in open("/proc/meminfo") if "AnonHuge" in l or "HugePages_Total" in l]
    print("".join(ah).strip())
except Exception:
    pass
