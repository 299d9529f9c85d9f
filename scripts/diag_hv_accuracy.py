import numpy as np, sys
sys.path.insert(0, '.')
import paper_2405_18328_b200 as wg
from paper_2405_18328_b200 import datasets
from oracle import oracle as orc
p = datasets.config1()
ctx = wg.Context(0)
ctx.set_data(p.X); ctx.set_hyper([*p.lengthscales, p.signal, p.noise])
for impl in ("tc", "simt"):
    ctx.set_hv_impl(impl)
    out = ctx.hv(p.V)
    for r0, r1 in ((0, 384), (6000, 6200), (13300, 13500)):
        ref = orc.hv_rows(p.X, p.lengthscales, p.signal, p.noise, p.V, r0, r1)
        e = np.linalg.norm(out[r0:r1] - ref) / np.linalg.norm(ref)
        rowerr = np.linalg.norm(out[r0:r1] - ref, axis=1) / np.linalg.norm(ref, axis=1)
        print(impl, r0, "rel %.3e" % e, "worst row %.3e" % rowerr.max())
    # kernel-only part: subtract noise*V to see K V error
    ref = orc.hv_rows(p.X, p.lengthscales, p.signal, p.noise, p.V, 0, 384)
    kv_ref = ref - p.noise**2 * p.V[:384]
    print(impl, "KV part rel %.3e" % (np.linalg.norm(out[:384] - p.noise**2*p.V[:384] - kv_ref)/np.linalg.norm(kv_ref)))
rng = np.random.default_rng(3)
X = rng.standard_normal((3000, 6)).astype(np.float32); V = rng.standard_normal((3000, 33)).astype(np.float32)
ls = rng.uniform(0.6, 1.8, 6)
ctx.set_data(X); ctx.set_hyper([*ls, 1.0, 0.2])
ref = orc.hv(X, ls, 1.0, 0.2, V)
for impl in ("tc", "simt"):
    ctx.set_hv_impl(impl)
    o = ctx.hv(V)
    print(impl, "3000x6 rel %.3e" % (np.linalg.norm(o - ref)/np.linalg.norm(ref)))
