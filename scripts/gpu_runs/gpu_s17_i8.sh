export PYTHONPATH=.
echo "== i8"; timeout 300 python scripts/diag_i8.py gpurun_out/i8.npz 2>&1 | tail -12
echo "== dmma"; WGP_HV64_ENGINE=dmma timeout 300 python scripts/diag_i8.py gpurun_out/dmma.npz 2>&1 | tail -12
python - <<'PY'
import numpy as np
a, b = np.load("gpurun_out/i8.npz"), np.load("gpurun_out/dmma.npz")
for k in a.files:
    x, y = a[k], b[k]
    print(k, "i8 vs dmma max rel", float(np.abs(x - y).max() / max(np.abs(y).max(), 1e-300)))
PY
echo "== cg timing"; timeout 300 python scripts/time_cg64_c2.py; WGP_HV64_ENGINE=dmma timeout 300 python scripts/time_cg64_c2.py
