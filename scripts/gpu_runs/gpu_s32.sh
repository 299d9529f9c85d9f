export PYTHONPATH=.
for r in 1 2; do for l in lib_alu lib_f2i; do
  echo "$l $(WGP_LIBRARY=$PWD/ab/$l.so timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"
done; done
timeout 300 python scripts/diag_i8.py gpurun_out/i8.npz 2>&1 | tail -3
timeout 500 python scripts/diag_cg_engines.py
