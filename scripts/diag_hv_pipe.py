"""wgp_hv pipeline diagnostics: plan, accuracy vs the one-launch product, times per mode."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18328_b200 as wg  # noqa: E402

# os.environ["WGP_HV_PLAN_DEBUG"] = "1"
for n, d, impl in ((5000, 9, "tc"), (5000, 9, "tc_f16")):
    rng = np.random.default_rng(31)
    X = rng.standard_normal((n, d)).astype(np.float32)
    V = rng.standard_normal((n, 65)).astype(np.float32)
    ls = rng.uniform(0.6, 1.6, d)
    with wg.Context(0) as ctx:
        ctx.set_data(X)
        ctx.set_hyper([*ls, 1.0, 0.3])
        ctx.set_hv_impl(impl)
        os.environ["WGP_HV_PIPE"] = "1"
        one = ctx.hv(V).astype(np.float64)
        for mode in ("", "rows", "j1024", "j2048", "j3840", "j4096"):
            os.environ["WGP_HV_PIPE"] = mode
            out = ctx.hv(V)
            t0 = time.perf_counter()
            for _ in range(20):
                ctx.hv(V)
            dt = (time.perf_counter() - t0) / 20 * 1e3
            e = np.linalg.norm(out - one, axis=0) / np.linalg.norm(one, axis=0)
            rows = np.abs(out - one).max(axis=1)
            bad = np.nonzero(rows > 1e-4 * np.abs(one).max())[0]
            print(f"n={n} {impl} mode={mode or 'model'} host-timed {dt:.3f} ms rel max col {e.max():.1e}"
                  f" bad rows {len(bad)} {bad[:3]} {bad[-3:] if len(bad) else ''}", flush=True)
