"""H.V relative error vs the accumulation chunk (WGP_TC_CHUNK) on the dense
config-3-like case: separates accumulation error from representation error."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r"""
import numpy as np, sys
sys.path.insert(0, %r)
import paper_2405_18328_b200 as wg
from oracle import oracle as orc
rng = np.random.default_rng(0)
X = rng.uniform(size=(20000, 3)).astype(np.float32)
V = rng.standard_normal((20000, 65)).astype(np.float32)
ref = orc.hv_rows(X, np.ones(3), 1.0, 0.5, V, 0, 256)
c = wg.Context(0)
c.set_data(X); c.set_hyper([1.0, 1.0, 1.0, 1.0, 0.5])
for impl in ("tc", "tc_bf16"):
    c.set_hv_impl(impl)
    out = c.hv(V)[:256]
    print(impl, "%%.3e" %% (np.linalg.norm(out - ref) / np.linalg.norm(ref)), flush=True)
# Gram-only error: V = e_j columns pick single entries of K
c.set_hv_impl("tc")
""" % ROOT
for chunk in (sys.argv[1:] or ["8", "16", "32", "100000"]):
    env = dict(os.environ, WGP_TC_CHUNK=chunk, WGP_TC_SPLITS="1")
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    print("chunk", chunk, r.stdout.replace("\n", "  "), r.stderr[-300:])
