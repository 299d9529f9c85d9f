"""Per-unit timeline of CTA 0 from a WGP_TC_TRACE_DUMP file (hv_f16p stamps):
[7] Gram: before bfull wait, [0] Gram committed, [4] K.V loop top, [12] before
vfull, [13] before kfull, [3] past kfull, [5] K.V issued, [1] epilogue woke
(quarter 0), [2] epilogue kfull arrive (quarter 0), [8+q] per quarter."""
import sys

import numpy as np

h = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 16)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
t0 = h[0, 4]
d = lambda a, b: (h[8:n, b] - h[8:n, a])
print("K.V loop period      ", np.diff(h[8:n, 4]).mean())
print("loop top -> vfull    ", d(4, 12).mean(), "(odrained + gram(g+L))")
print("vfull wait           ", d(12, 13).mean())
print("kfull wait           ", d(13, 3).mean())
print("K.V issue            ", d(3, 5).mean())
print("Gram bfull wait+issue", (h[8:n, 0] - h[8:n, 7]).mean())
print("Gram commit -> epi wake (q0)", (h[8:n, 1] - h[8:n, 0]).mean())
print("epi wake -> kfull (q0)      ", (h[8:n, 2] - h[8:n, 1]).mean())
print("kfull arrive -> K.V past wait", (h[8:n, 3] - h[8:n, 2]).mean())
for q in range(4):
    print(f"epi quarter {q}", (h[8:n, 8 + q] - h[8:n, 1]).mean())
print("first units (rel clk): loop top / gram commit / epi wake / kfull / past kfull")
for u in range(0, 12):
    print(u, *(int(h[u, k] - t0) if h[u, k] else None for k in (4, 0, 1, 2, 3)))
