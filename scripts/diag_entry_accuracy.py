"""Entry-level accuracy of the tensor-core K: H e_j (one-hot V) against the
oracle's column j, so the error is the representation of single entries
(Gram + k evaluation + K.V split), free of accumulation."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402
from oracle import oracle as orc  # noqa: E402

rng = np.random.default_rng(0)
X = rng.uniform(size=(4096, 3)).astype(np.float32)
cols = [0, 17, 1000, 4095]
V = np.zeros((4096, len(cols)), np.float32)
for i, j in enumerate(cols):
    V[j, i] = 1.0
H = orc.kernel_matrices(X, np.ones(3), 1.0, 0.5)[0][:, cols]
c = wg.Context(0)
c.set_data(X)
c.set_hyper([1.0, 1.0, 1.0, 1.0, 0.5])
for impl in ("simt", "tc", "tc_bf16"):
    c.set_hv_impl(impl)
    out = c.hv(V).astype(np.float64)
    rel = np.abs(out - H) / np.abs(H)
    print(f"{impl:8s} entry rel err: max {rel.max():.3e} mean {rel.mean():.3e}  "
          f"signed mean {((out - H) / np.abs(H)).mean():+.3e}")
