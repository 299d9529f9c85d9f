"""A/B of an hv_tc variant switch (default WGP_TC_NOPACK: packed vs hi/lo
Gram; WGP_TC_NODIRECT: direct distances vs Gram for d <= 4): entry accuracy
(H columns through identity right-hand sides vs the fp64 oracle), H.V accuracy
and kernel time at the config-2 / config-3 shapes.
usage: ab_pack.py [SWITCH [d,d,..]]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SWITCH = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "child" else os.environ.get("AB_SWITCH", "WGP_TC_NOPACK")
DIMS = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else os.environ.get("AB_DIMS", "1,3,8,9,19,20,26")).split(",")]


def child():
    import paper_2405_18328_b200 as wg
    from oracle import oracle as orc
    tag = "off" if os.environ.get(SWITCH) else "on"
    ctx = wg.Context(0, hv_impl="tc")
    for d in DIMS:
        rng = np.random.default_rng(d)
        n = 2000
        X = rng.standard_normal((n, d)).astype(np.float32)
        X[1] = X[0] + 1e-3  # a near-duplicate pair
        ls = np.exp(rng.uniform(np.log(0.5), np.log(2.0), d))
        ctx.set_data(X)
        ctx.set_hyper([*ls, 1.0, 0.1])
        E = np.zeros((n, 64), np.float32)
        E[np.arange(64), np.arange(64)] = 1.0
        Hc = ctx.hv(E)
        ref = orc.hv(X, ls, 1.0, 0.1, E)
        V = rng.standard_normal((n, 17)).astype(np.float32)
        o = ctx.hv(V)
        r = orc.hv(X, ls, 1.0, 0.1, V)
        print(f"{tag} d={d:2d} entry max abs {np.abs(Hc - ref).max():.3e}  "
              f"hv rel {np.linalg.norm(o - r) / np.linalg.norm(r):.3e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
        sys.exit(0)
    for env in ({}, {SWITCH: "1"}):
        e = dict(os.environ, AB_SWITCH=SWITCH, AB_DIMS=",".join(map(str, DIMS)), **env)
        subprocess.run([sys.executable, __file__, "child"], env=e, check=True)
        for args in (["41157", "9", "65", "20"], ["100000", "3", "65", "5"], ["100000", "1", "65", "5"],
                     ["13500", "26", "65", "30"]):
            out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts/time_hv.py"), "tc", *args], env=e,
                                 capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
            print(("off " if env else "on  ") + out, flush=True)
