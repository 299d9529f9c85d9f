export PYTHONPATH=.
timeout 300 python scripts/diag_i8.py gpurun_out/i8.npz 2>&1 | tail -10
WGP_HV64_ENGINE=dmma timeout 300 python scripts/diag_i8.py gpurun_out/dmma.npz > /dev/null 2>&1
python - <<'PY'
import numpy as np
a, b = np.load("gpurun_out/i8.npz"), np.load("gpurun_out/dmma.npz")
for k in a.files: print(k, "i8 vs dmma max rel:", float(np.abs(a[k] - b[k]).max() / max(np.abs(b[k]).max(), 1e-300)))
PY
timeout 300 python scripts/time_cg64_c2.py
timeout 500 python scripts/diag_cg_engines.py
